// pca.cu -- K7: PCA residual r = (x - mu) - V^T V (x - mu)   (features.py:183-193)
//
// z = V (x - mu) accumulates the k projections in fp64 (the reference computes
// in fp64, then casts the residual to float32); a second channel sweep writes
// the float32 residual.  Each thread owns PX consecutive pixels, so every
// broadcast of V[j][c] from shared memory feeds PX fused multiply-adds; the
// feature reads are float4-vectorised and coalesced along pixels (the second
// sweep hits L2).
#include "common.cuh"

namespace qfca {

constexpr int PCA_MAXK = 16;
constexpr int PCA_THREADS = 128;
constexpr int PCA_PX = 4;

template <int K>
__global__ void __launch_bounds__(PCA_THREADS)
k_pca_residual(const float* __restrict__ x, int C, int64_t hw,
               const double* __restrict__ mean, const double* __restrict__ comps,
               int64_t blocks_per_image, int per_image_model, float* __restrict__ out) {
    extern __shared__ __align__(16) double sm[];
    double* smu = sm;      // [C]
    double* sV = sm + C;   // [C][K]  (transposed: the K values of a channel are adjacent)
    const int64_t img = blockIdx.x / blocks_per_image;
    const int64_t blk = blockIdx.x % blocks_per_image;
    const double* mu = mean + (per_image_model ? img * C : 0);
    const double* V = comps + (per_image_model ? img * (int64_t)K * C : 0);
    for (int i = threadIdx.x; i < C; i += PCA_THREADS) smu[i] = mu[i];
    for (int i = threadIdx.x; i < K * C; i += PCA_THREADS) {
        const int j = i / C, c = i % C;
        sV[c * K + j] = V[i];
    }
    __syncthreads();
    const int64_t p0 = (blk * PCA_THREADS + threadIdx.x) * PCA_PX;
    if (p0 >= hw) return;
    const float* xp = x + img * C * hw + p0;
    float* op = out + img * C * hw + p0;
    const bool full = p0 + PCA_PX <= hw && (hw % 4) == 0;
    double z[PCA_PX][K];
#pragma unroll
    for (int q = 0; q < PCA_PX; ++q)
#pragma unroll
        for (int j = 0; j < K; ++j) z[q][j] = 0.0;
    auto load = [&](int c, double (&v)[PCA_PX]) {
        const float* src = xp + (int64_t)c * hw;
        if (full) {
            const float4 f = __ldg(reinterpret_cast<const float4*>(src));
            v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
        } else {
#pragma unroll
            for (int q = 0; q < PCA_PX; ++q) v[q] = p0 + q < hw ? (double)__ldg(src + q) : 0.0;
        }
        const double m = smu[c];
#pragma unroll
        for (int q = 0; q < PCA_PX; ++q) v[q] -= m;
    };
    for (int c = 0; c < C; ++c) {
        double xc[PCA_PX];
        load(c, xc);
        const double* vc = sV + c * K;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const double vj = vc[j];
#pragma unroll
            for (int q = 0; q < PCA_PX; ++q) z[q][j] = fma(vj, xc[q], z[q][j]);
        }
    }
    for (int c = 0; c < C; ++c) {
        double xc[PCA_PX];
        load(c, xc);
        const double* vc = sV + c * K;
        double proj[PCA_PX];
#pragma unroll
        for (int q = 0; q < PCA_PX; ++q) proj[q] = 0.0;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const double vj = vc[j];
#pragma unroll
            for (int q = 0; q < PCA_PX; ++q) proj[q] = fma(vj, z[q][j], proj[q]);
        }
        float* dst = op + (int64_t)c * hw;
        if (full) {
            float4 f;
            f.x = (float)(xc[0] - proj[0]);
            f.y = (float)(xc[1] - proj[1]);
            f.z = (float)(xc[2] - proj[2]);
            f.w = (float)(xc[3] - proj[3]);
            *reinterpret_cast<float4*>(dst) = f;
        } else {
#pragma unroll
            for (int q = 0; q < PCA_PX; ++q)
                if (p0 + q < hw) dst[q] = (float)(xc[q] - proj[q]);
        }
    }
}

// Cholesky QR of a batch of tall fp64 blocks, in place: Y (C x p, row-major)
// <- Y L^-T with L L^T = Y^T Y.  One CTA per block, the block resident in
// shared memory: Gram matrix, Cholesky factor and the triangular solve in one
// launch (the subspace iteration of features.topk_eigh re-orthonormalises
// with it after every cov @ X product).
constexpr int CQR_THREADS = 256;

__global__ void __launch_bounds__(CQR_THREADS)
k_cholqr(double* __restrict__ Y, int C, int p) {
    extern __shared__ __align__(16) double sq[];
    const int ps = p | 1;              // odd row stride: rows of a warp hit distinct banks
    double* sY = sq;                   // [C][ps]
    double* sL = sq + (size_t)C * ps;  // [p][p] Gram, then its Cholesky factor
    double* blk = Y + (size_t)blockIdx.x * C * p;
    const int tid = threadIdx.x;
    for (int i = tid; i < C * p; i += CQR_THREADS) sY[(i / p) * ps + i % p] = blk[i];
    __syncthreads();
    // Gram: G[a][b] = sum_r Y[r][a] Y[r][b], lower triangle
    for (int e = tid; e < p * p; e += CQR_THREADS) {
        const int a = e / p, b = e % p;
        if (b > a) continue;
        double s = 0.0;
        for (int r = 0; r < C; ++r) s = fma(sY[r * ps + a], sY[r * ps + b], s);
        sL[a * p + b] = s;
    }
    __syncthreads();
    // Cholesky (right-looking, one column per step)
    for (int k = 0; k < p; ++k) {
        if (tid == 0) sL[k * p + k] = sqrt(sL[k * p + k]);
        __syncthreads();
        const double dk = sL[k * p + k];
        for (int i = k + 1 + tid; i < p; i += CQR_THREADS) sL[i * p + k] /= dk;
        __syncthreads();
        for (int e = tid; e < p * p; e += CQR_THREADS) {
            const int i = e / p, j = e % p;
            if (i > k && j > k && j <= i) sL[i * p + j] -= sL[i * p + k] * sL[j * p + k];
        }
        __syncthreads();
    }
    // rows: x L^T = y  ->  forward substitution per row
    for (int r = tid; r < C; r += CQR_THREADS) {
        double* row = sY + r * ps;
        for (int k = 0; k < p; ++k) {
            double s = row[k];
            for (int j = 0; j < k; ++j) s -= row[j] * sL[k * p + j];
            row[k] = s / sL[k * p + k];
        }
    }
    __syncthreads();
    for (int i = tid; i < C * p; i += CQR_THREADS) blk[i] = sY[(i / p) * ps + i % p];
}

int launch_cqr_step(double* Y, int64_t batch, int C, int p, cudaStream_t st);

int launch_cholqr(double* Y, int64_t batch, int C, int p, cudaStream_t st) {
    if (batch <= 0 || C <= 0 || p <= 0 || p > C) return QFCA_ERR_ARG;
    // fused register-blocked step (eig.cu) for blocks up to 512 x 32
    const int rc = launch_cqr_step(Y, batch, C, p, st);
    if (rc != QFCA_ERR_UNSUPPORTED) return rc;
    const size_t smem = ((size_t)C * (p | 1) + (size_t)p * p) * sizeof(double);
    if (smem > 200 * 1024) return QFCA_ERR_UNSUPPORTED;
    if (cudaFuncSetAttribute(k_cholqr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return QFCA_ERR_CUDA;
    k_cholqr<<<(unsigned)batch, CQR_THREADS, smem, st>>>(Y, C, p);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

// centred copy xc = x - mean (fp32 out) for the covariance GEMM
__global__ void k_center(const float* __restrict__ x, int64_t planes, int64_t hw,
                         const double* __restrict__ mean, float* __restrict__ out) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= planes * hw) return;
    out[gid] = (float)((double)x[gid] - mean[gid / hw]);
}

template <int K>
static int launch_res_k(const float* x, int64_t images, int C, int64_t hw, const double* mean,
                        const double* comps, int per_image_model, float* out, cudaStream_t st) {
    const size_t smem = (size_t)(C + (size_t)K * C) * sizeof(double);
    if (smem > 200 * 1024) return QFCA_ERR_UNSUPPORTED;
    if (cudaFuncSetAttribute(k_pca_residual<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return QFCA_ERR_CUDA;
    const int64_t per_block = (int64_t)PCA_THREADS * PCA_PX;
    const int64_t bpi = (hw + per_block - 1) / per_block;
    k_pca_residual<K><<<(unsigned)(bpi * images), PCA_THREADS, smem, st>>>(
        x, C, hw, mean, comps, bpi, per_image_model, out);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

int launch_pca_residual_tiled(const float*, int64_t, int, int64_t, const double*, const double*,
                              int, int, float*, cudaStream_t);

int launch_pca_residual(const float* x, int64_t images, int C, int64_t hw, const double* mean,
                        const double* comps, int k, int per_image_model, float* out,
                        cudaStream_t st) {
    if (images <= 0 || C <= 0 || hw <= 0 || k < 1 || k > PCA_MAXK) return QFCA_ERR_ARG;
    // persistent tiled kernel (residual.cu): x read once, loads double-buffered
    const int rc = launch_pca_residual_tiled(x, images, C, hw, mean, comps, k, per_image_model,
                                             out, st);
    if (rc != QFCA_ERR_UNSUPPORTED) return rc;
    switch (k) {
#define QFCA_RES_K(KK) \
    case KK: return launch_res_k<KK>(x, images, C, hw, mean, comps, per_image_model, out, st);
        QFCA_RES_K(1) QFCA_RES_K(2) QFCA_RES_K(3) QFCA_RES_K(4) QFCA_RES_K(5) QFCA_RES_K(6)
        QFCA_RES_K(7) QFCA_RES_K(8) QFCA_RES_K(9) QFCA_RES_K(10) QFCA_RES_K(11) QFCA_RES_K(12)
        QFCA_RES_K(13) QFCA_RES_K(14) QFCA_RES_K(15) QFCA_RES_K(16)
#undef QFCA_RES_K
    }
    return QFCA_ERR_ARG;
}

int launch_center(const float* x, int64_t planes, int64_t hw, const double* mean, float* out,
                  cudaStream_t st) {
    if (planes <= 0 || hw <= 0) return QFCA_ERR_ARG;
    k_center<<<(unsigned)((planes * hw + 255) / 256), 256, 0, st>>>(x, planes, hw, mean, out);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

}  // namespace qfca
