// cov_i8.cu -- fp64-accurate batched covariance on the int8 tensor cores.
//
// pca_fit (features.py:157-180) forms cov = xc^T xc / n in fp64, xc = x - mean.
// The QFCA+ maps depend on that covariance at the 1e-8 level (a residual bin
// flip moves a map by ~1e-4), so an fp32 GEMM is not a faithful substitute.
// Here each channel's centred values become 32-bit fixed-point integers
//
//     N_c(p) = rint(xc_c(p) * 2^(32 - e_c)),   max |xc_c| < 2^(e_c - 2),
//
// written as four balanced base-256 digits d_0..d_3 (int8, d_3 the top), and
//
//     sum_p N_c N_d = sum_{k,l} 256^(k+l) sum_p d_k,c d_l,d
//
// is evaluated with exact int8 x int8 -> int32 tcgen05 MMAs.  Pairs with
// k + l >= 2 are kept (13 of 16; the dropped ones weigh <= 2^-40 of the top
// pair), one int32 TMEM accumulator per class k + l = 2..6, and the epilogue
// combines the classes in fp64 and scales by 2^(e_c + e_d - 64) / n.  The
// result matches the fp64 reference to ~1e-11 relative (measured) at a
// fraction of an fp64 GEMM's cost.
//
// Kernel layout (one 128 x 64 output tile per CTA, lower triangle only, the
// mirror written by the same CTA):
//   warp 0   TMA producer: per K-stage of 64 pixels, the 4 digit tiles of the
//            128 A rows and of the 64 B rows (SWIZZLE_64B, 48 KB), 4 stages;
//   warp 1   MMA issuer: 13 pairs x 4 k-steps of tcgen05.mma.kind::i8
//            (M = 128, N = 64, K = 32) into 5 x 64 TMEM columns;
//   warps 2-5 epilogue: tcgen05.ld, fp64 class combine, scale, store.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace qfca {

constexpr int CV_BM = 128;   // A rows (channels) per tile
constexpr int CV_BN = 64;    // B rows (channels) per tile
constexpr int CV_BK = 64;    // K bytes (pixels) per stage = one 64-byte swizzle row
constexpr int CV_DIG = 4;    // base-256 digits
constexpr int CV_CLS = 5;    // classes k + l = 2..6
constexpr int CV_STAGES = 4;
constexpr int CV_THREADS = 192;
constexpr int CV_A_BYTES = CV_BM * CV_BK;                              // 8 KB per digit
constexpr int CV_B_BYTES = CV_BN * CV_BK;                              // 4 KB per digit
constexpr int CV_STAGE_BYTES = CV_DIG * (CV_A_BYTES + CV_B_BYTES);    // 96 KB
constexpr int CV_SMEM = CV_STAGES * CV_STAGE_BYTES + 1024 + 256;      // + align + barriers
constexpr int CV_TMEM_COLS = 512;

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
        : "memory");
}
__device__ __forceinline__ uint64_t sw64_desc(uint32_t saddr) {
    // K-major, SWIZZLE_64B: 8-row atoms of 8 x 64 B = 512 B (SBO), version 1 (sm_100)
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;                 // LBO (unused for swizzled K-major)
    d |= (uint64_t)(512 >> 4) << 32;        // SBO
    d |= (uint64_t)1 << 46;                 // descriptor version
    d |= (uint64_t)4 << 61;                 // SWIZZLE_64B
    return d;
}
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n\t}" ::"r"(
            tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(0u));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     bar)
                 : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}

// ---------------------------------------------------------------- digits
// One CTA per (image, channel row < Cp): the plane is staged in shared memory
// (one HBM read), its mean is formed there when requested (fp64, fixed
// order), then the fixed-point exponent and the four balanced base-256 digit
// planes D[((img * 4 + k) * Cp + c) * Kp + p].
constexpr int DG_THREADS = 128;

__device__ __forceinline__ double block_reduce_dg(double v, bool is_max, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double u = __shfl_xor_sync(0xffffffffu, v, o);
        v = is_max ? fmax(v, u) : v + u;
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    v = red[0];
#pragma unroll
    for (int w = 1; w < DG_THREADS / 32; ++w) v = is_max ? fmax(v, red[w]) : v + red[w];
    return v;
}

__global__ void __launch_bounds__(DG_THREADS)
k_cov_digits(const float* __restrict__ x, int C, int hw, int Cp, int Kp,
             const double* __restrict__ mean_in, double* __restrict__ mean_out,
             int8_t* __restrict__ D, int* __restrict__ expo) {
    extern __shared__ __align__(16) float xs[];  // [hw]
    __shared__ double red[DG_THREADS / 32];
    const int img = blockIdx.x / Cp, c = blockIdx.x % Cp;
    const int tid = threadIdx.x;
    int8_t* d0 = D + ((int64_t)(img * CV_DIG + 0) * Cp + c) * Kp;
    const int64_t dstep = (int64_t)Cp * Kp;
    if (c >= C) {  // padding rows: zero digits
        for (int k = 0; k < CV_DIG; ++k)
            for (int p = tid * 16; p < Kp; p += DG_THREADS * 16)
                *reinterpret_cast<uint4*>(d0 + k * dstep + p) = make_uint4(0, 0, 0, 0);
        return;
    }
    const float* xp = x + ((int64_t)img * C + c) * hw;
    double s = 0.0;
    if ((hw & 3) == 0) {
        const float4* x4 = reinterpret_cast<const float4*>(xp);
        for (int i = tid; i < hw / 4; i += DG_THREADS) {
            const float4 v = __ldg(x4 + i);
            reinterpret_cast<float4*>(xs)[i] = v;
            s += ((double)v.x + (double)v.y) + ((double)v.z + (double)v.w);
        }
    } else {
        for (int i = tid; i < hw; i += DG_THREADS) {
            const float v = __ldg(xp + i);
            xs[i] = v;
            s += (double)v;
        }
    }
    double mu;
    if (mean_out) {
        mu = block_reduce_dg(s, false, red) / (double)hw;
        if (tid == 0) mean_out[(int64_t)img * C + c] = mu;
    } else {
        mu = mean_in[(int64_t)img * C + c];
        __syncthreads();
    }
    double m = 0.0;
    for (int p = tid; p < hw; p += DG_THREADS) m = fmax(m, fabs((double)xs[p] - mu));
    m = block_reduce_dg(m, true, red);
    int e = 0;
    if (m > 0.0) {
        int E;
        frexp(m, &E);  // m < 2^E
        e = E + 2;     // max |xc| < 2^(e - 2): |N| < 2^30
    }
    if (tid == 0) expo[(int64_t)img * C + c] = e;
    const double sc = ldexp(1.0, 32 - e);
    // 16 pixels per thread per iteration: four 16-byte digit stores
    for (int p0 = tid * 16; p0 < Kp; p0 += DG_THREADS * 16) {
        uint32_t w[CV_DIG][4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            // balanced digits n = d0 + 256 (d1 + 256 (d2 + 256 d3)), d0..d2 in
            // [-128, 127]: the bytes of u = n + 0x808080 are d_k + 128 (k < 3, no
            // carries) and d3, so the two's-complement digit bytes of one pixel
            // are u ^ 0x808080; a 4 x 4 byte transpose then gives one word per digit
            uint32_t u[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int p = p0 + 4 * q + j;
                const int n = p < hw ? (int)rint(((double)xs[p] - mu) * sc) : 0;
                u[j] = ((uint32_t)n + 0x00808080u) ^ 0x00808080u;
            }
            const uint32_t t01 = __byte_perm(u[0], u[1], 0x5140);  // d0: p0 p1, d1: p0 p1
            const uint32_t t23 = __byte_perm(u[2], u[3], 0x5140);
            const uint32_t h01 = __byte_perm(u[0], u[1], 0x7362);  // d2, d3 of p0 p1
            const uint32_t h23 = __byte_perm(u[2], u[3], 0x7362);
            w[0][q] = __byte_perm(t01, t23, 0x5410);
            w[1][q] = __byte_perm(t01, t23, 0x7632);
            w[2][q] = __byte_perm(h01, h23, 0x5410);
            w[3][q] = __byte_perm(h01, h23, 0x7632);
        }
#pragma unroll
        for (int k = 0; k < CV_DIG; ++k)
            *reinterpret_cast<uint4*>(d0 + k * dstep + p0) =
                make_uint4(w[k][0], w[k][1], w[k][2], w[k][3]);
    }
}

// ---------------------------------------------------------------- GEMM
__global__ void __launch_bounds__(CV_THREADS, 1)
k_cov_i8(const __grid_constant__ CUtensorMap tmap, int C, int Cp, int Kp, int hw,
         const int* __restrict__ expo, double* __restrict__ cov) {
    extern __shared__ uint8_t cv_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>(((uintptr_t)cv_raw + 1023) & ~(uintptr_t)1023);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + CV_STAGES * CV_STAGE_BYTES);
    // bars[s] full, bars[CV_STAGES + s] empty, bars[2 CV_STAGES] tmem full; tmem base after
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * CV_STAGES + 2);

    const int nI = Cp / CV_BM;
    const int tiles = nI * (nI + 1);  // lower-triangle 128 x 64 tiles: 2I + 2 per row block
    const int img = blockIdx.x / tiles;
    int t = blockIdx.x % tiles, I = 0;
    while (t >= 2 * I + 2) { t -= 2 * I + 2; ++I; }
    const int J = t;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nkb = Kp / CV_BK;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < CV_STAGES; ++s) {
            mbar_init(smem_u32(&bars[s]), 1);
            mbar_init(smem_u32(&bars[CV_STAGES + s]), 1);
        }
        mbar_init(smem_u32(&bars[2 * CV_STAGES]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(CV_TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            const int rowA = img * CV_DIG * Cp + I * CV_BM;
            const int rowB = img * CV_DIG * Cp + J * CV_BN;
            for (int kb = 0; kb < nkb; ++kb) {
                const int s = kb % CV_STAGES;
                if (kb >= CV_STAGES) mbar_wait(smem_u32(&bars[CV_STAGES + s]), ((kb / CV_STAGES) & 1) ^ 1);
                const uint32_t full = smem_u32(&bars[s]);
                mbar_expect_tx(full, CV_STAGE_BYTES);
                const uint32_t base = smem_u32(sm + s * CV_STAGE_BYTES);
                for (int k = 0; k < CV_DIG; ++k) {
                    const uint32_t a = base + k * CV_A_BYTES;
                    tma_load_2d(a, &tmap, full, kb * CV_BK, rowA + k * Cp);
                    tma_load_2d(a + CV_A_BYTES / 2, &tmap, full, kb * CV_BK, rowA + k * Cp + 64);
                    tma_load_2d(base + CV_DIG * CV_A_BYTES + k * CV_B_BYTES, &tmap, full,
                                kb * CV_BK, rowB + k * Cp);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            // kind::i8, D s32, A/B signed, K-major, N = 64, M = 128
            const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) |
                                   ((uint32_t)(CV_BN >> 3) << 17) | ((uint32_t)(CV_BM >> 4) << 24);
            for (int kb = 0; kb < nkb; ++kb) {
                const int s = kb % CV_STAGES;
                mbar_wait(smem_u32(&bars[s]), (kb / CV_STAGES) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t base = smem_u32(sm + s * CV_STAGE_BYTES);
#pragma unroll
                for (int kk = 0; kk < CV_BK / 32; ++kk) {
                    bool first[CV_CLS] = {true, true, true, true, true};
#pragma unroll
                    for (int k = 0; k < CV_DIG; ++k)
#pragma unroll
                        for (int l = 0; l < CV_DIG; ++l) {
                            if (k + l < 2) continue;
                            const int cls = k + l - 2;
                            const uint64_t ad = sw64_desc(base + k * CV_A_BYTES + kk * 32);
                            const uint64_t bd =
                                sw64_desc(base + CV_DIG * CV_A_BYTES + l * CV_B_BYTES + kk * 32);
                            const uint32_t acc = (kb > 0 || kk > 0 || !first[cls]) ? 1u : 0u;
                            first[cls] = false;
                            mma_i8(tmem + cls * CV_BN, ad, bd, idesc, acc);
                        }
                }
                mma_commit(smem_u32(&bars[CV_STAGES + s]));  // stage free once these MMAs complete
            }
            mma_commit(smem_u32(&bars[2 * CV_STAGES]));  // accumulators complete
        }
        __syncwarp();
    } else {
        // ---- epilogue: warp w reads TMEM lanes 32 (w % 4) .. + 31
        const int q = warp & 3;
        const int r = I * CV_BM + q * 32 + lane;  // channel row
        mbar_wait(smem_u32(&bars[2 * CV_STAGES]), 0);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const int er = r < C ? expo[(int64_t)img * C + r] : 0;
        double* cimg = cov + (int64_t)img * C * C;
        const double inv_hw = 1.0 / (double)hw;  // one division per thread, not per element
        for (int cc = 0; cc < CV_BN / 16; ++cc) {
            int32_t v[CV_CLS][16];
#pragma unroll
            for (int cls = 0; cls < CV_CLS; ++cls)
                tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + cls * CV_BN + cc * 16, v[cls]);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int col = J * CV_BN + cc * 16 + j;
                if (r >= C || col >= C) continue;
                // classes from the top: each term exact, 256^(cls + 2)
                double s = (double)v[4][j] * 281474976710656.0;           // 256^6
                s += (double)v[3][j] * 1099511627776.0;                    // 256^5
                s += (double)v[2][j] * 4294967296.0;                       // 256^4
                s += (double)v[1][j] * 16777216.0;                         // 256^3
                s += (double)v[0][j] * 65536.0;                            // 256^2
                const int ec = expo[(int64_t)img * C + col];
                // exact power-of-two scale (exponent field; er + ec - 64 stays in the
                // normal range for fp32 inputs), then * 1/hw
                const double p2 = __longlong_as_double((long long)(1023 + er + ec - 64) << 52);
                const double val = (s * p2) * inv_hw;
                cimg[(int64_t)r * C + col] = val;
                cimg[(int64_t)col * C + r] = val;
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
    }
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(CV_TMEM_COLS));
    }
}

// ---------------------------------------------------------------- host
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

int64_t cov_i8_workspace(int64_t images, int C, int hw) {
    const int64_t Cp = (C + CV_BM - 1) / CV_BM * CV_BM;
    const int64_t Kp = (hw + CV_BK - 1) / CV_BK * CV_BK;
    return images * CV_DIG * Cp * Kp + ((images * C * 4 + 255) & ~255LL);
}

// cov (images, C, C) fp64 of the centred features x (images, C, hw) fp32;
// mean_out != nullptr: the plane means are formed here (and mean ignored).
int launch_cov_i8(const float* x, int64_t images, int C, int hw, const double* mean,
                  double* mean_out, void* workspace, int64_t ws_bytes, double* cov,
                  cudaStream_t st) {
    if (images <= 0 || C <= 0 || hw <= 0) return QFCA_ERR_ARG;
    const int Cp = (C + CV_BM - 1) / CV_BM * CV_BM;
    const int Kp = (hw + CV_BK - 1) / CV_BK * CV_BK;
    // int32 accumulators: a class sums <= 4 pairs of |d d'| <= 2^14 over Kp pixels,
    // Kp <= 2^14 keeps it below 2^30
    if ((int64_t)images * CV_DIG * Cp >= (1LL << 31) || Kp > (1 << 14))
        return QFCA_ERR_UNSUPPORTED;
    if (ws_bytes < cov_i8_workspace(images, C, hw)) return QFCA_ERR_ARG;
    auto enc = encode_fn();
    if (!enc) return QFCA_ERR_CUDA;
    int8_t* D = reinterpret_cast<int8_t*>(workspace);
    int* expo = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(workspace) +
                                       images * CV_DIG * (int64_t)Cp * Kp);
    const size_t dsmem = (size_t)hw * 4;
    if (dsmem > 48 * 1024 &&
        cudaFuncSetAttribute(k_cov_digits, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)dsmem) != cudaSuccess)
        return QFCA_ERR_CUDA;
    k_cov_digits<<<(unsigned)(images * Cp), DG_THREADS, dsmem, st>>>(x, C, hw, Cp, Kp, mean,
                                                                      mean_out, D, expo);
    if (cudaGetLastError() != cudaSuccess) return QFCA_ERR_CUDA;

    CUtensorMap map;
    const cuuint64_t gdim[2] = {(cuuint64_t)Kp, (cuuint64_t)(images * CV_DIG * Cp)};
    const cuuint64_t gstride[1] = {(cuuint64_t)Kp};
    const cuuint32_t box[2] = {CV_BK, 64};
    const cuuint32_t estride[2] = {1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, D, gdim, gstride, box, estride,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return QFCA_ERR_CUDA;
    if (cudaFuncSetAttribute(k_cov_i8, cudaFuncAttributeMaxDynamicSharedMemorySize, CV_SMEM) !=
        cudaSuccess)
        return QFCA_ERR_CUDA;
    const int nI = Cp / CV_BM;
    const int64_t grid = images * nI * (nI + 1);
    k_cov_i8<<<(unsigned)grid, CV_THREADS, CV_SMEM, st>>>(map, C, Cp, Kp, hw, expo, cov);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

}  // namespace qfca
