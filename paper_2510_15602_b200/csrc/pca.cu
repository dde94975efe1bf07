// pca.cu -- K7: PCA residual r = (x - mu) - V^T V (x - mu)   (features.py:183-193)
//
// One thread per pixel: z = V (x - mu) accumulates the k projections in fp64
// (the reference computes in fp64, then casts the residual to float32), the
// second channel sweep writes the float32 residual.  mu and V (k x C, fp64)
// are staged in shared memory and broadcast.  The feature read is coalesced
// along pixels; the second read hits L2.
#include "common.cuh"

namespace qfca {

constexpr int PCA_MAXK = 32;
constexpr int PCA_THREADS = 128;

__global__ void __launch_bounds__(PCA_THREADS)
k_pca_residual(const float* __restrict__ x, int64_t images, int C, int64_t hw,
               const double* __restrict__ mean, const double* __restrict__ comps, int k,
               int64_t blocks_per_image, int per_image_model, float* __restrict__ out) {
    extern __shared__ __align__(16) double sm[];
    double* smu = sm;          // [C]
    double* sV = sm + C;       // [k][C]
    const int64_t img = blockIdx.x / blocks_per_image;
    const int64_t blk = blockIdx.x % blocks_per_image;
    const double* mu = mean + (per_image_model ? img * C : 0);
    const double* V = comps + (per_image_model ? img * (int64_t)k * C : 0);
    for (int i = threadIdx.x; i < C; i += PCA_THREADS) smu[i] = mu[i];
    for (int i = threadIdx.x; i < k * C; i += PCA_THREADS) sV[i] = V[i];
    __syncthreads();
    const int64_t px = blk * PCA_THREADS + threadIdx.x;
    if (px >= hw) return;
    const float* xp = x + img * C * hw + px;
    float* op = out + img * C * hw + px;
    double z[PCA_MAXK];
#pragma unroll
    for (int j = 0; j < PCA_MAXK; ++j) z[j] = 0.0;
    for (int c = 0; c < C; ++c) {
        const double xc = (double)__ldg(xp + (int64_t)c * hw) - smu[c];
#pragma unroll
        for (int j = 0; j < PCA_MAXK; ++j)
            if (j < k) z[j] = fma(sV[j * C + c], xc, z[j]);
    }
    for (int c = 0; c < C; ++c) {
        const double xc = (double)__ldg(xp + (int64_t)c * hw) - smu[c];
        double proj = 0.0;
#pragma unroll
        for (int j = 0; j < PCA_MAXK; ++j)
            if (j < k) proj = fma(sV[j * C + c], z[j], proj);
        op[(int64_t)c * hw] = (float)(xc - proj);
    }
}

// centred copy xc = x - mean (fp32 out) for the covariance GEMM
__global__ void k_center(const float* __restrict__ x, int64_t planes, int64_t hw,
                         const double* __restrict__ mean, float* __restrict__ out) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= planes * hw) return;
    out[gid] = (float)((double)x[gid] - mean[gid / hw]);
}

int launch_pca_residual(const float* x, int64_t images, int C, int64_t hw, const double* mean,
                        const double* comps, int k, int per_image_model, float* out,
                        cudaStream_t st) {
    if (images <= 0 || C <= 0 || hw <= 0 || k < 1 || k > PCA_MAXK) return QFCA_ERR_ARG;
    const size_t smem = (size_t)(C + (size_t)k * C) * sizeof(double);
    if (smem > 200 * 1024) return QFCA_ERR_UNSUPPORTED;
    if (cudaFuncSetAttribute(k_pca_residual, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return QFCA_ERR_CUDA;
    const int64_t bpi = (hw + PCA_THREADS - 1) / PCA_THREADS;
    k_pca_residual<<<(unsigned)(bpi * images), PCA_THREADS, smem, st>>>(
        x, images, C, hw, mean, comps, k, bpi, per_image_model, out);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

int launch_center(const float* x, int64_t planes, int64_t hw, const double* mean, float* out,
                  cudaStream_t st) {
    if (planes <= 0 || hw <= 0) return QFCA_ERR_ARG;
    k_center<<<(unsigned)((planes * hw + 255) / 256), 256, 0, st>>>(x, planes, hw, mean, out);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

}  // namespace qfca
