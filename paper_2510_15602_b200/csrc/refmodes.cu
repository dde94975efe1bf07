// refmodes.cu -- reference histogram weights of every select_reference mode on
// the device (quantize.py:150-200), as the fp64 (planes, n_bins) array the
// reference returns:
//
//   median-quan  K3 order statistics (reference.cu) -> R_i = V_i - V_{i-1};
//   quan-median  K3 per-bin lower medians w_i of the sample histograms, then
//   quan-mean    K3 per-bin sums / S, then w * (T^2 / sum(w)) with NumPy's
//                pairwise summation order for sum(w) (k_weights_from_stats);
//   mean-quan    the per-rank MEAN of the sorted sample patches (a float mean,
//                so no integer shortcut): k_gather_patches copies every sample
//                patch (pad_plane semantics, quantize.py:119-132), a segmented
//                radix sort orders each patch (CUB, ascending float32 as
//                np.sort), k_rank_mean_bins sums each rank over the samples in
//                sample order in fp64 (ranked.mean(axis=0, dtype=float64)
//                accumulates row by row), divides by S and bins the mean with
//                the fp64 rule of _quantize_values_to_hist (quantize.py:143-147).
// Degenerate channels get [T^2, 0, ...] (quantize.py:169-171).  Every weight is
// bit-identical to the reference's.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "common.cuh"
#include "qfca_b200.h"

namespace qfca {

int launch_reference(const void*, int, const float*, const float*, int64_t, int, int, int, int,
                     int, int, int, int32_t*, cudaStream_t);
int sample_stride(int h, int w, int budget);

// numpy's pairwise_sum (numpy/_core/src/umath/loops_utils.h.src) of n contiguous
// doubles: < 8 sequential, <= 128 eight strided partial sums, else two halves
// split at a multiple of 8
__device__ double np_pairwise_sum(const double* a, int n) {
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
        return res;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; ++i) res = __dadd_rn(res, a[i]);
        return res;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(np_pairwise_sum(a, n2), np_pairwise_sum(a + n2, n - n2));
}

// weights of the median-quan / quan-median / quan-mean modes from K3's statistics
__global__ void k_weights_from_stats(const int32_t* __restrict__ stats, const float* __restrict__ lo,
                                     const float* __restrict__ hi, int64_t planes, int n_bins,
                                     int mode, int t2, int n_samples, double* __restrict__ w,
                                     double* __restrict__ tmp) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= planes) return;
    const int32_t* s = stats + p * n_bins;
    double* o = w + p * n_bins;
    if (!(hi[p] > lo[p])) {  // degenerate (quantize.py:169-171)
        for (int i = 0; i < n_bins; ++i) o[i] = i == 0 ? (double)t2 : 0.0;
        return;
    }
    if (mode == QFCA_REF_MEDIAN_QUAN) {
        int prev = 0;
        for (int i = 0; i < n_bins; ++i) {
            o[i] = (double)(s[i] - prev);
            prev = s[i];
        }
        return;
    }
    double* wv = tmp + p * n_bins;
    for (int i = 0; i < n_bins; ++i)  // quan-median: lower medians; quan-mean: sums / S
        wv[i] = mode == QFCA_REF_QUAN_MEAN ? __ddiv_rn((double)s[i], (double)n_samples)
                                           : (double)s[i];
    const double total = np_pairwise_sum(wv, n_bins);
    if (total > 0.0) {
        const double q = __ddiv_rn((double)t2, total);
        for (int i = 0; i < n_bins; ++i) o[i] = __dmul_rn(wv[i], q);
    } else {
        for (int i = 0; i < n_bins; ++i) o[i] = i == 0 ? (double)t2 : 0.0;
    }
}

// every sample patch of every plane, pad_plane index semantics (zero pad -> 0.0)
__global__ void k_gather_patches(const float* __restrict__ x, int64_t planes, int h, int w, int t,
                                 int pad, int stride, int nsy, int nsx, float* __restrict__ out) {
    const int r = t / 2, t2 = t * t;
    const int64_t S = (int64_t)nsy * nsx;
    const int64_t n = planes * S * t2;
    const bool edge = pad == QFCA_PAD_REFLECT && !(h > 1 && w > 1);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ps = i / t2;
        const int k = (int)(i - ps * t2);
        const int64_t p = ps / S;
        const int s = (int)(ps - p * S);
        const int sy = (s / nsx) * stride, sx = (s % nsx) * stride;
        const int yy = pad_plane_index(sy + k / t - r, h, pad, edge);
        const int xx = pad_plane_index(sx + k % t - r, w, pad, edge);
        out[i] = (yy < 0 || xx < 0) ? 0.0f : x[(p * h + yy) * (int64_t)w + xx];
    }
}

// per (plane, rank): fp64 sum over the samples in sample order, mean, bin, count
__global__ void k_rank_mean_bins(const float* __restrict__ sorted, int64_t planes, int S, int t2,
                                 const float* __restrict__ lo, const float* __restrict__ hi,
                                 int n_bins, double* __restrict__ w) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= planes * t2) return;
    const int64_t p = i / t2;
    const int rank = (int)(i - p * t2);
    const double l = lo[p], hh = hi[p];
    if (!(hh > l)) return;  // degenerate: set by k_degenerate_weights
    const float* col = sorted + p * (int64_t)S * t2 + rank;
    double acc = 0.0;
    for (int s = 0; s < S; ++s) acc = __dadd_rn(acc, (double)col[(int64_t)s * t2]);
    const double mean = __ddiv_rn(acc, (double)S);
    const double span = hh - l;  // quantize.py:144: hi > lo here
    double q = floor(__ddiv_rn(__dmul_rn(mean - l, (double)n_bins), span));
    q = q < 0.0 ? 0.0 : (q > (double)(n_bins - 1) ? (double)(n_bins - 1) : q);
    atomicAdd(w + p * n_bins + (int)q, 1.0);  // integer counts: exact in any order
}

__global__ void k_degenerate_weights(const float* __restrict__ lo, const float* __restrict__ hi,
                                     int64_t planes, int n_bins, int t2, double* __restrict__ w) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= planes || hi[p] > lo[p]) return;
    for (int i = 0; i < n_bins; ++i) w[p * n_bins + i] = i == 0 ? (double)t2 : 0.0;
}

struct SegOffset {  // segment k spans [k * len, (k + 1) * len)
    int len;
    __host__ __device__ int operator()(int k) const { return k * len; }
};

static constexpr int64_t MQ_CHUNK_ELEMS = 1LL << 26;  // patch values per sort chunk (256 MB)

static int64_t mq_chunk_planes(int64_t planes, int64_t per_plane) {
    int64_t c = MQ_CHUNK_ELEMS / (per_plane > 0 ? per_plane : 1);
    if (c < 1) c = 1;
    return c < planes ? c : planes;
}

static size_t mq_sort_temp(int64_t elems, int segs) {
    size_t bytes = 0;
    auto off = thrust::make_transform_iterator(thrust::make_counting_iterator(0), SegOffset{1});
    cub::DeviceSegmentedSort::SortKeys(nullptr, bytes, (const float*)nullptr, (float*)nullptr,
                                       (int)elems, segs, off, off + 1);
    return bytes;
}

static size_t align256r(size_t x) { return (x + 255) & ~(size_t)255; }

int64_t reference_weights_workspace_bytes(int64_t planes, int h, int w, int n_bins, int t,
                                          int budget, int mode) {
    if (planes <= 0 || h <= 0 || w <= 0 || n_bins < 1 || t < 1 || budget < 1) return -1;
    const size_t stats = align256r((size_t)planes * n_bins * 4) +
                         align256r((size_t)planes * n_bins * 8);
    if (mode != QFCA_REF_MEAN_QUAN) return (int64_t)stats;
    const int s = sample_stride(h, w, budget);
    const int64_t S = (int64_t)((h + s - 1) / s) * ((w + s - 1) / s);
    const int64_t per = S * t * t;
    const int64_t cp = mq_chunk_planes(planes, per);
    const int64_t elems = cp * per;
    if (elems > 0x7fffffffLL) return -1;
    return (int64_t)(stats + 2 * align256r((size_t)elems * 4) +
                     align256r(mq_sort_temp(elems, (int)(cp * S))));
}

int launch_reference_weights(const float* values, const void* bins, int bins_bytes,
                             const float* lo, const float* hi, int64_t planes, int h, int w,
                             int n_bins, int t, int pad, int budget, int mode, void* workspace,
                             int64_t workspace_bytes, double* weights, cudaStream_t st) {
    const int64_t need = reference_weights_workspace_bytes(planes, h, w, n_bins, t, budget, mode);
    if (need < 0 || !workspace || workspace_bytes < need || !weights || !lo || !hi)
        return QFCA_ERR_ARG;
    if ((t & 1) == 0) return QFCA_ERR_ARG;
    const int t2 = t * t;
    const int s = sample_stride(h, w, budget);
    const int nsy = (h + s - 1) / s, nsx = (w + s - 1) / s;
    const int S = nsy * nsx;
    uint8_t* ws = (uint8_t*)workspace;
    int32_t* stats = (int32_t*)ws;
    double* tmp = (double*)(ws + align256r((size_t)planes * n_bins * 4));
    const unsigned pb = (unsigned)((planes + 127) / 128);
    if (mode != QFCA_REF_MEAN_QUAN) {
        if (!bins) return QFCA_ERR_ARG;
        int rc = launch_reference(bins, bins_bytes, lo, hi, planes, h, w, n_bins, t, pad, budget,
                                  mode, stats, st);
        if (rc != QFCA_OK) return rc;
        k_weights_from_stats<<<pb, 128, 0, st>>>(stats, lo, hi, planes, n_bins, mode, t2, S,
                                                 weights, tmp);
        return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
    }
    if (!values) return QFCA_ERR_ARG;
    const size_t stats_b = align256r((size_t)planes * n_bins * 4) +
                           align256r((size_t)planes * n_bins * 8);
    const int64_t per = (int64_t)S * t2;
    const int64_t cp = mq_chunk_planes(planes, per);
    float* pin = (float*)(ws + stats_b);
    float* pout = (float*)(ws + stats_b + align256r((size_t)cp * per * 4));
    void* sort_tmp = ws + stats_b + 2 * align256r((size_t)cp * per * 4);
    if (cudaMemsetAsync(weights, 0, (size_t)planes * n_bins * 8, st) != cudaSuccess)
        return QFCA_ERR_CUDA;
    for (int64_t p0 = 0; p0 < planes; p0 += cp) {
        const int64_t np_ = planes - p0 < cp ? planes - p0 : cp;
        const int64_t elems = np_ * per;
        int64_t g = (elems + 255) / 256;
        if (g > 148 * 64) g = 148 * 64;
        k_gather_patches<<<(unsigned)g, 256, 0, st>>>(values + p0 * (int64_t)h * w, np_, h, w, t,
                                                      pad, s, nsy, nsx, pin);
        size_t tb = mq_sort_temp(cp * per, (int)(cp * S));
        auto off = thrust::make_transform_iterator(thrust::make_counting_iterator(0),
                                                   SegOffset{t2});
        if (cub::DeviceSegmentedSort::SortKeys(sort_tmp, tb, pin, pout, (int)elems,
                                               (int)(np_ * S), off, off + 1, st) != cudaSuccess)
            return QFCA_ERR_CUDA;
        const int64_t nr = np_ * t2;
        k_rank_mean_bins<<<(unsigned)((nr + 127) / 128), 128, 0, st>>>(
            pout, np_, S, t2, lo + p0, hi + p0, n_bins, weights + p0 * n_bins);
        if (cudaGetLastError() != cudaSuccess) return QFCA_ERR_CUDA;
    }
    k_degenerate_weights<<<pb, 128, 0, st>>>(lo, hi, planes, n_bins, t2, weights);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

}  // namespace qfca
