// common.cuh -- shared device helpers for the QFCA B200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define QFCA_PAD_ZERO 0
#define QFCA_PAD_REFLECT 1
#define QFCA_PAD_WRAP 2

// status codes returned through the C-ABI (include/qfca_b200.h)
#define QFCA_OK 0
#define QFCA_ERR_ARG 1
#define QFCA_ERR_CUDA 2
#define QFCA_ERR_UNSUPPORTED 3

namespace qfca {

// filter taps passed by value (kernel parameter space), at most 255 taps
constexpr int QFCA_MAX_TAPS = 255;
struct Taps {
    double k[QFCA_MAX_TAPS];
    int n;
};

// Channel groups per image for a fused scoring kernel that keeps `per_sm` CTAs
// resident per SM and scores `cpb` channels per batch: the grid is
// images x groups CTAs, each scoring batches-per-CTA (bpc) batches, so the
// run takes ceil(CTAs / resident slots) waves of bpc batch-times.  Minimise
// waves * (bpc + per-CTA setup), ties to fewer groups (fewer partial maps).
// The library's stream-ordered scratch (cudaMallocAsync, a few small buffers)
// comes from the device's default memory pool; keep its freed memory mapped
// (release threshold = max) so a synchronisation between calls does not
// return it to the driver and make the next allocation map pages again.
inline void keep_default_pool() {
    static int done_dev = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done_dev = dev;
}

inline int balanced_groups(int64_t images, int C, int cpb, int per_sm) {
    static int sms = 0;
    if (sms <= 0) {
        int dev = 0, n = 0;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0)
            sms = n;
        else
            sms = 148;
    }
    const int64_t slots = (int64_t)sms * (per_sm < 1 ? 1 : per_sm);
    const int nb = (C + cpb - 1) / cpb;
    double best = -1.0;
    int best_g = 1;
    for (int bpc = 1; bpc <= nb; ++bpc) {
        const int g = (nb + bpc - 1) / bpc;
        const int64_t waves = (images * g + slots - 1) / slots;
        const double cost = (double)waves * (bpc + 0.25);
        if (best < 0.0 || cost < best - 1e-9 || (cost < best + 1e-9 && g < best_g)) {
            best = cost;
            best_g = g;
        }
    }
    return best_g;
}

// Padded-plane coordinate -> source index, -1 for zero padding.
// Restates scoring.py:158-174 (_map_coord): reflect without edge repeat,
// repeated for large margins; n == 1 -> 0; wrap is toroidal.
__host__ __device__ __forceinline__ int map_coord(int c, int n, int pad) {
    if (c >= 0 && c < n) return c;
    if (pad == QFCA_PAD_ZERO) return -1;
    if (pad == QFCA_PAD_WRAP) {
        int m = c % n;
        return m < 0 ? m + n : m;
    }
    if (n == 1) return 0;
    while (c < 0 || c >= n) {
        if (c < 0) c = -c;
        if (c >= n) c = 2 * n - 2 - c;
    }
    return c;
}

// np.pad index as used by pooling.py:20-38 (pad_plane): identical to
// map_coord except that reflect switches to 'edge' on both axes when either
// axis has length 1 (pooling.py:31-35).  Used only by reference selection
// (quantize.py:119-132).  Zero padding returns -1 (value 0.0).
__host__ __device__ __forceinline__ int pad_plane_index(int c, int n, int pad, bool edge) {
    if (c >= 0 && c < n) return c;
    if (pad == QFCA_PAD_ZERO) return -1;
    if (pad == QFCA_PAD_WRAP) {
        int m = c % n;
        return m < 0 ? m + n : m;
    }
    if (edge || n == 1) return c < 0 ? 0 : n - 1;
    return map_coord(c, n, pad);
}

// The reference bin rule (quantize.py:79-81), evaluated exactly as NumPy does
// it: fp64 ((v - lo) * N) / safe, floor, clip to [0, N-1].
__device__ __forceinline__ int bin_of(float v, double lo, double safe, int n_bins) {
    double q = ((double)v - lo) * (double)n_bins / safe;
    double f = floor(q);
    if (!(f > 0.0)) return 0;  // also maps NaN to 0
    if (f > (double)(n_bins - 1)) return n_bins - 1;
    return (int)f;
}

__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace qfca
