// residual.cu -- K7 v2/v3: PCA residual r = (x - mu) - V^T V (x - mu)
// (features.py:183-193) as a persistent, tiled kernel; v3 runs the two
// contractions on the fp64 tensor cores (below), v2 on the fp64 FMA pipe.
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

// ---------------------------------------------------------------- fp64 tensor-core variant
// Same tiling, the two contractions on the fp64 tensor cores (mma.sync
// m8n8k4 f64, exact fp64 products and sums -- the reference computes in
// fp64): z (32 px x KN comps) = Xc^T V^T over the C channels, split in
// channel slices and reduced in fixed order, then r (C x 32 px) = Xc - V z^T
// with the subtraction and the float32 cast in the epilogue.  Rows of the x
// tile are padded to 40 floats and z is stored transposed with 40-double
// rows so the operand fragments load without shared-memory bank conflicts.
constexpr int RD_LDX = 40;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int K>
__global__ void __launch_bounds__(RS_THREADS, 1)
k_pca_residual_dmma(const float* __restrict__ x, int C, int hw, const double* __restrict__ mean,
                    const double* __restrict__ comps, int per_image_model, int64_t items,
                    int tiles_per_image, int c_lo, int c_hi, float* __restrict__ out) {
    constexpr int KK = (K + 3) & ~3;    // k-dim of r (multiple of 4), also V row length
    constexpr int KN = (K + 7) & ~7;    // n-dim of z (multiple of 8)
    constexpr int NZ = KN / 8;          // z n-tiles
    constexpr int NW = RS_THREADS / 32; // 16 warps
    constexpr int ZSL = NW / (4 * NZ);  // channel slices of the z contraction
    extern __shared__ __align__(16) uint8_t rd_sm[];
    float* xs0 = reinterpret_cast<float*>(rd_sm);                                    // [2][C][40]
    double* sV = reinterpret_cast<double*>(rd_sm + 2 * (size_t)C * RD_LDX * 4);      // [C][KK]
    double* smu = sV + (size_t)C * KK;                                               // [C]
    double* zp = smu + C;                                                            // [ZSL][32][KN]
    double* zt = zp + ZSL * 32 * KN;                                                 // [KN][40]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int lr = lane >> 2, lc = lane & 3;
    const int64_t w0 = (int64_t)blockIdx.x * items / gridDim.x;
    const int64_t w1 = (int64_t)(blockIdx.x + 1) * items / gridDim.x;
    if (w0 >= w1) return;

    auto load_tile = [&](int64_t w, int buf) {
        const int64_t img = w / tiles_per_image;
        const int p0 = (int)(w % tiles_per_image) * RS_TP;
        const float* src = x + img * (int64_t)C * hw + p0;
        float* dst = xs0 + (size_t)buf * C * RD_LDX;
        const int valid = min(RS_TP, hw - p0);
        for (int i = tid; i < C * (RS_TP / 4); i += RS_THREADS) {
            const int c = i / (RS_TP / 4), q = i % (RS_TP / 4);
            float* d = dst + c * RD_LDX + q * 4;
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
        if (img != cur_img) {  // model of this image: mean, V transposed to [c][j]
            __syncthreads();
            const int64_t mi = per_image_model ? img : 0;
            for (int i = tid; i < C; i += RS_THREADS) smu[i] = mean[mi * C + i];
            for (int i = tid; i < KK * C; i += RS_THREADS) {
                const int j = i / C, c = i % C;
                sV[c * KK + j] = j < K ? comps[mi * (int64_t)K * C + j * C + c] : 0.0;
            }
            cur_img = img;
        }
        cp_async_wait0();
        __syncthreads();  // tile w resident, previous tile's readers done
        if (w + 1 < w1) load_tile(w + 1, buf ^ 1);
        const float* xs = xs0 + (size_t)buf * C * RD_LDX;

        // ---- z partials: warp -> (m-tile of 8 px, n-tile of 8 comps, channel slice)
        {
            const int mt = warp & 3, nt = (warp >> 2) % NZ, sl = warp / (4 * NZ);
            const int ng = C / 4;  // slices in whole 4-channel k-steps
            const int c0 = 4 * (sl * ng / ZSL), c1 = 4 * ((sl + 1) * ng / ZSL);
            const int p = mt * 8 + lr, j = nt * 8 + lr;
            double d0 = 0.0, d1 = 0.0;
#pragma unroll 4
            for (int cb = c0; cb < c1; cb += 4) {
                const int c = cb + lc;
                const double a = (double)xs[c * RD_LDX + p] - smu[c];
                const double b = j < KK ? sV[c * KK + j] : 0.0;
                dmma(d0, d1, a, b);
            }
            double* zo = zp + (sl * 32 + mt * 8 + lr) * KN + nt * 8 + 2 * lc;
            zo[0] = d0;
            zo[1] = d1;
        }
        __syncthreads();
        for (int e = tid; e < 32 * KN; e += RS_THREADS) {
            const int pp = e / KN, j = e % KN;
            double s = 0.0;
#pragma unroll
            for (int sl = 0; sl < ZSL; ++sl) s += zp[(sl * 32 + pp) * KN + j];
            zt[j * 40 + pp] = s;
        }
        __syncthreads();

        // ---- r = xc - V z^T: warp -> output tiles (8 channels x 8 px) of the
        //      channel slice [c_lo, c_hi) (every channel unless a rank's slice)
        const bool full = p0 + RS_TP <= hw;
        const int mt0 = c_lo >> 3, nmt = ((c_hi + 7) >> 3) - mt0;
        const int cs = c_hi - c_lo;
        for (int t = warp; t < nmt * 4; t += NW) {
            const int mt = mt0 + (t >> 2), nt = t & 3;
            double d0 = 0.0, d1 = 0.0;
#pragma unroll
            for (int kb = 0; kb < KK; kb += 4) {
                const double a = sV[(mt * 8 + lr) * KK + kb + lc];
                const double b = zt[(kb + lc) * 40 + nt * 8 + lr];
                dmma(d0, d1, a, b);
            }
            const int c = mt * 8 + lr, pp = nt * 8 + 2 * lc;
            const double mu = smu[c];
            const float2 xv = *reinterpret_cast<const float2*>(xs + c * RD_LDX + pp);
            const float r0 = (float)(((double)xv.x - mu) - d0);
            const float r1 = (float)(((double)xv.y - mu) - d1);
            if (c < c_lo || c >= c_hi) continue;
            float* op = out + (img * (int64_t)cs + (c - c_lo)) * hw + p0 + pp;
            if (full) {
                *reinterpret_cast<float2*>(op) = make_float2(r0, r1);
            } else {
                if (p0 + pp < hw) op[0] = r0;
                if (p0 + pp + 1 < hw) op[1] = r1;
            }
        }
    }
}

size_t residual_dmma_smem(int C, int K) {
    const int KK = (K + 3) & ~3, KN = (K + 7) & ~7, NZ = KN / 8;
    const int ZSL = (RS_THREADS / 32) / (4 * NZ);
    return 2 * (size_t)C * RD_LDX * 4 + (size_t)C * KK * 8 + (size_t)C * 8 +
           (size_t)ZSL * 32 * KN * 8 + (size_t)KN * 40 * 8;
}

template <int K>
static int launch_dmma_k(const float* x, int64_t images, int C, int64_t hw, const double* mean,
                         const double* comps, int per_image_model, float* out, cudaStream_t st,
                         int c_lo = 0, int c_hi = -1) {
    if (c_hi < 0) c_hi = C;
    const size_t smem = residual_dmma_smem(C, K);
    if (smem > 227 * 1024 || hw % 4 != 0 || hw > (1 << 30) || C % 8 != 0 || C < 16)
        return QFCA_ERR_UNSUPPORTED;
    if (cudaFuncSetAttribute(k_pca_residual_dmma<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return QFCA_ERR_CUDA;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int tpi = (int)((hw + RS_TP - 1) / RS_TP);
    const int64_t items = images * tpi;
    const int64_t grid = items < sms ? items : sms;
    k_pca_residual_dmma<K><<<(unsigned)grid, RS_THREADS, smem, st>>>(
        x, C, (int)hw, mean, comps, per_image_model, items, tpi, c_lo, c_hi, out);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

// the residual of channels [c_lo, c_hi) only (a channel-sharded rank's slice):
// z = V (x - mu) still contracts every channel, the output is (images, c_hi -
// c_lo, hw); the fp64 tensor-core kernel only
int launch_pca_residual_slice(const float* x, int64_t images, int C, int64_t hw,
                              const double* mean, const double* comps, int k,
                              int per_image_model, int c_lo, int c_hi, float* out,
                              cudaStream_t st) {
    if (c_lo < 0 || c_hi > C || c_lo >= c_hi) return QFCA_ERR_ARG;
    switch (k) {
#define QFCA_RS_K(KK)                                                                     \
    case KK:                                                                              \
        return launch_dmma_k<KK>(x, images, C, hw, mean, comps, per_image_model, out, st, \
                                 c_lo, c_hi);
        QFCA_RS_K(1) QFCA_RS_K(2) QFCA_RS_K(3) QFCA_RS_K(4) QFCA_RS_K(5) QFCA_RS_K(6)
        QFCA_RS_K(7) QFCA_RS_K(8) QFCA_RS_K(9) QFCA_RS_K(10) QFCA_RS_K(11) QFCA_RS_K(12)
        QFCA_RS_K(13) QFCA_RS_K(14) QFCA_RS_K(15) QFCA_RS_K(16)
#undef QFCA_RS_K
    }
    return QFCA_ERR_UNSUPPORTED;
}

int launch_pca_residual_tiled(const float* x, int64_t images, int C, int64_t hw,
                              const double* mean, const double* comps, int k,
                              int per_image_model, float* out, cudaStream_t st) {
    int rc = QFCA_ERR_UNSUPPORTED;
    switch (k) {  // fp64 tensor cores first
#define QFCA_RD_K(KK) \
    case KK: rc = launch_dmma_k<KK>(x, images, C, hw, mean, comps, per_image_model, out, st); break;
        QFCA_RD_K(1) QFCA_RD_K(2) QFCA_RD_K(3) QFCA_RD_K(4) QFCA_RD_K(5) QFCA_RD_K(6)
        QFCA_RD_K(7) QFCA_RD_K(8) QFCA_RD_K(9) QFCA_RD_K(10) QFCA_RD_K(11) QFCA_RD_K(12)
        QFCA_RD_K(13) QFCA_RD_K(14) QFCA_RD_K(15) QFCA_RD_K(16)
#undef QFCA_RD_K
    }
    if (rc != QFCA_ERR_UNSUPPORTED) return rc;
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
