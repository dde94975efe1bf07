// residual.cu -- K7 v2: PCA residual r = (x - mu) - V^T V (x - mu) (features.py:183-193)
// as a persistent, tiled kernel.
//
// Each CTA owns a contiguous range of (image, 32-pixel tile) items.  A tile is
// all C channels x 32 pixels of x (C x 128 B), staged in shared memory with
// cp.async and double-buffered, so x is read from HBM exactly once and the
// next tile's load overlaps this tile's fp64 math:
//   z[p][j] = sum_c V[j][c] (x[c][p] - mu[c])      16 channel slices x 32 px,
//                                                  fixed-order slice reduction
//   r[c][p] = (x[c][p] - mu[c]) - sum_j V[j][c] z[p][j]   written as float32
// V (transposed to [c][j]) and mu are reloaded only when the image changes.
#include "common.cuh"

namespace qfca {

constexpr int RS_TP = 32;        // pixels per tile (128-byte rows)
constexpr int RS_THREADS = 512;  // 32 pixels x 16 channel slices
constexpr int RS_SLICES = RS_THREADS / RS_TP;
constexpr int RS_MAXK = 16;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <int K>
__global__ void __launch_bounds__(RS_THREADS, 1)
k_pca_residual_tiled(const float* __restrict__ x, int C, int hw, const double* __restrict__ mean,
                     const double* __restrict__ comps, int per_image_model, int64_t items,
                     int tiles_per_image, float* __restrict__ out) {
    extern __shared__ __align__(16) uint8_t rs_sm[];
    float* xs0 = reinterpret_cast<float*>(rs_sm);                        // [2][C][32]
    constexpr int KP = (K + 1) & ~1;  // even row length: V rows load as double2
    double* sV = reinterpret_cast<double*>(rs_sm + 2 * (size_t)C * RS_TP * 4);  // [C][KP]
    double* smu = sV + (size_t)C * KP;                                  // [C]
    double* zp = smu + C;                                               // [16][K][32]
    const int tid = threadIdx.x;
    const int p = tid % RS_TP, sl = tid / RS_TP;
    const int64_t w0 = (int64_t)blockIdx.x * items / gridDim.x;
    const int64_t w1 = (int64_t)(blockIdx.x + 1) * items / gridDim.x;
    if (w0 >= w1) return;

    auto load_tile = [&](int64_t w, int buf) {
        const int64_t img = w / tiles_per_image;
        const int p0 = (int)(w % tiles_per_image) * RS_TP;
        const float* src = x + img * (int64_t)C * hw + p0;
        float* dst = xs0 + (size_t)buf * C * RS_TP;
        const int valid = min(RS_TP, hw - p0);
        for (int i = tid; i < C * (RS_TP / 4); i += RS_THREADS) {
            const int c = i / (RS_TP / 4), q = i % (RS_TP / 4);
            float* d = dst + c * RS_TP + q * 4;
            if (4 * q + 4 <= valid) {
                cp_async16(d, src + (int64_t)c * hw + q * 4);
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    d[e] = 4 * q + e < valid ? src[(int64_t)c * hw + q * 4 + e] : 0.f;
            }
        }
        cp_async_commit();
    };

    int64_t cur_img = -1;
    load_tile(w0, 0);
    for (int64_t w = w0; w < w1; ++w) {
        const int buf = (int)((w - w0) & 1);
        const int64_t img = w / tiles_per_image;
        const int p0 = (int)(w % tiles_per_image) * RS_TP;
        if (img != cur_img) {  // model of this image (mean, V transposed)
            __syncthreads();
            const int64_t mi = per_image_model ? img : 0;
            for (int i = tid; i < C; i += RS_THREADS) smu[i] = mean[mi * C + i];
            for (int i = tid; i < K * C; i += RS_THREADS) {
                const int j = i / C, c = i % C;
                sV[c * KP + j] = comps[mi * (int64_t)K * C + i];
            }
            if (KP != K)
                for (int c = tid; c < C; c += RS_THREADS) sV[c * KP + K] = 0.0;
            cur_img = img;
        }
        cp_async_wait0();
        __syncthreads();  // tile w resident, previous tile's readers done
        if (w + 1 < w1) load_tile(w + 1, buf ^ 1);
        const float* xs = xs0 + (size_t)buf * C * RS_TP;

        // z partials: channel slice sl, pixel p
        double z[K];
#pragma unroll
        for (int j = 0; j < K; ++j) z[j] = 0.0;
        const int c0 = sl * C / RS_SLICES, c1 = (sl + 1) * C / RS_SLICES;
#pragma unroll 4
        for (int c = c0; c < c1; ++c) {
            const double xc = (double)xs[c * RS_TP + p] - smu[c];
            const double2* vc = reinterpret_cast<const double2*>(sV + c * KP);
#pragma unroll
            for (int j = 0; j < KP / 2; ++j) {
                const double2 v = vc[j];
                z[2 * j] = fma(v.x, xc, z[2 * j]);
                if (2 * j + 1 < K) z[2 * j + 1] = fma(v.y, xc, z[2 * j + 1]);
            }
        }
#pragma unroll
        for (int j = 0; j < K; ++j) zp[(sl * K + j) * RS_TP + p] = z[j];
        __syncthreads();
#pragma unroll
        for (int j = 0; j < K; ++j) {
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < RS_SLICES; ++q) s += zp[(q * K + j) * RS_TP + p];
            z[j] = s;
        }
        // residual rows of this slice
        const bool pin = p0 + p < hw;
        float* op = out + img * (int64_t)C * hw + p0 + p;
#pragma unroll 4
        for (int c = c0; c < c1; ++c) {
            const double xc = (double)xs[c * RS_TP + p] - smu[c];
            const double2* vc = reinterpret_cast<const double2*>(sV + c * KP);
            double proj = 0.0;
#pragma unroll
            for (int j = 0; j < KP / 2; ++j) {
                const double2 v = vc[j];
                proj = fma(v.x, z[2 * j], proj);
                if (2 * j + 1 < K) proj = fma(v.y, z[2 * j + 1], proj);
            }
            if (pin) op[(int64_t)c * hw] = (float)(xc - proj);
        }
    }
}

size_t residual_tiled_smem(int C, int K) {
    return 2 * (size_t)C * RS_TP * 4 + (size_t)C * 8 + (size_t)C * ((K + 1) & ~1) * 8 +
           (size_t)RS_SLICES * RS_TP * K * 8;
}

template <int K>
static int launch_tiled_k(const float* x, int64_t images, int C, int64_t hw, const double* mean,
                          const double* comps, int per_image_model, float* out, cudaStream_t st) {
    const size_t smem = residual_tiled_smem(C, K);
    if (smem > 227 * 1024 || hw % 4 != 0 || hw > (1 << 30) || C < RS_SLICES)
        return QFCA_ERR_UNSUPPORTED;
    if (cudaFuncSetAttribute(k_pca_residual_tiled<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return QFCA_ERR_CUDA;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int tpi = (int)((hw + RS_TP - 1) / RS_TP);
    const int64_t items = images * tpi;
    const int64_t grid = items < sms ? items : sms;
    k_pca_residual_tiled<K><<<(unsigned)grid, RS_THREADS, smem, st>>>(
        x, C, (int)hw, mean, comps, per_image_model, items, tpi, out);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

int launch_pca_residual_tiled(const float* x, int64_t images, int C, int64_t hw,
                              const double* mean, const double* comps, int k,
                              int per_image_model, float* out, cudaStream_t st) {
    switch (k) {
#define QFCA_RT_K(KK) \
    case KK: return launch_tiled_k<KK>(x, images, C, hw, mean, comps, per_image_model, out, st);
        QFCA_RT_K(1) QFCA_RT_K(2) QFCA_RT_K(3) QFCA_RT_K(4) QFCA_RT_K(5) QFCA_RT_K(6)
        QFCA_RT_K(7) QFCA_RT_K(8) QFCA_RT_K(9) QFCA_RT_K(10) QFCA_RT_K(11) QFCA_RT_K(12)
        QFCA_RT_K(13) QFCA_RT_K(14) QFCA_RT_K(15) QFCA_RT_K(16)
#undef QFCA_RT_K
    }
    return QFCA_ERR_UNSUPPORTED;
}

}  // namespace qfca
