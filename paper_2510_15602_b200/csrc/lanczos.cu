// lanczos.cu -- block Lanczos stage of the top-k eigensolver (features.topk_eigh),
// which replaces np.linalg.eigh of pca_fit (features.py:173-176).
//
// pca_fit needs only the top k (= 10) eigenpairs of the C x C fp64 covariance.
// Subspace iteration pays one pass over the covariance S per iteration and
// ~30 iterations (plus a C^3 squaring); block Lanczos extracts far more from
// each pass: P passes of an 8-column block span a Krylov space of n = 8P
// vectors that contains the top-10 eigenvectors of the WRN50-2 covariances to
// ~1e-15 at P = 16 (tools/lanczos_proto.py; SURVEY H4 explains why the
// eigenvectors must be that accurate).  One CTA per image runs every pass;
// every contraction is an m8n8k4 fp64 tensor-core MMA (exact fp64 products and
// sums), and the block W (C x 8) lives in the MMA accumulators of the 8 warps
// (warp w: rows 64w .. 64w+63, eight 8 x 8 tiles):
//
//   S pass    W = S Q_j     (S symmetric, so A = S^T tiles come straight from
//             rows of S; the rows stream through a 5-stage cp.async.bulk +
//             mbarrier ring fed by a producer warp, 8 rows of S per stage,
//             further chunks prefetched into L2)
//   H column  c1 = B^T W over the basis B = [Q_0 .. Q_j], the basis blocks
//             streaming through the same ring; c1 is block column j of
//             H = B^T S B (Q_i^T S Q_j, i <= j)
//   reorth    W -= B c1, then again with c2 = B^T W (classical Gram-Schmidt
//             twice: full reorthogonalisation)
//   block QR  Cholesky QR twice on the C x 8 block (Gram on the MMAs, the 8 x 8
//             factor on one warp; a pivot below 1e-28 of the trace is a breakdown
//             and leaves a zero column) -> Q_{j+1}
//
// The start block is Q_0 = qr(S R) for a seeded R (one extra pass), so the
// basis stays in range(S).
// Outputs per image: the basis B (n vectors of C doubles, vector-contiguous)
// and the upper block triangle of H (n x n, row-major); the caller takes the
// Ritz pairs of H (topk_eigh on the small matrix) and maps them back, V = B u.
#include "common.cuh"

namespace qfca {

constexpr int LZ_BW = 8;         // block width (columns per Lanczos block)
constexpr int LZ_THREADS = 256;  // consumers: 8 warps x 64 rows: C <= 512, C % 64 == 0
constexpr int LZ_NW = LZ_THREADS / 32;
constexpr int LZ_CTA = LZ_THREADS + 32;  // + one producer warp (ring refills)
constexpr int LZ_MAXC = 64 * LZ_NW;
constexpr int LZ_KC = 8;         // rows per ring chunk
constexpr int LZ_NST = 5;        // ring stages
constexpr int LZ_MAXP = 32;      // passes (n = 8 P <= 256)
constexpr int LZ_PF = 6;         // S chunks prefetched into L2 beyond the ring

__device__ __forceinline__ uint32_t lz_smem(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void lz_mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void lz_mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void lz_mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "LZW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra LZW_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void lz_mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// consumer-only barrier (named barrier 1: the producer warp never joins)
__device__ __forceinline__ void lz_csync() {
    asm volatile("bar.sync 1, %0;" ::"n"(LZ_THREADS) : "memory");
}
__device__ __forceinline__ void lz_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void lz_bulk_load(uint32_t dst, const void* src, uint32_t bytes,
                                             uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}
// m8n8k4 fp64 tensor-core MMA, fragments as in residual.cu:
// a = A[lane>>2][lane&3], b = B[lane&3][lane>>2], d = D[lane>>2][2 (lane&3) + {0,1}]
__device__ __forceinline__ void lz_dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

struct LzSmem {
    int cp;  // padded row pitch of a ring chunk (doubles): C + 4, so both MMA
             // operand patterns on chunk rows are bank-conflict free
    int o_stage, o_w, o_cf, o_part, o_g, total;
};

__host__ __device__ inline LzSmem lz_layout(int C, int n) {
    LzSmem L;
    L.cp = C + 4;
    int off = 0;
    L.o_stage = off;
    off += LZ_NST * LZ_KC * L.cp * 8;
    L.o_w = off;  // Q_j in the S pass, W in the sweeps and the block QR
    off += C * LZ_BW * 8;
    L.o_cf = off;
    off += n * LZ_BW * 8;
    L.o_part = off;  // [2][warps][64] MMA partials, reduced over the warps per block
    off += 2 * LZ_NW * 64 * 8;
    L.o_g = off;     // Gram / L | R^-1 | 1 / diag(L)
    off += (2 * LZ_BW * LZ_BW + LZ_BW) * 8;
    L.total = off;
    return L;
}

// The ring streams 8-row chunks (8 x C doubles): rows of S in the S pass, the
// basis blocks B_i (8 vectors) in the Gram-Schmidt sweeps.  A pass is a fixed
// chunk program -- S (C/8 chunks), then for j >= 0 coefficient sweep 1 (j+1
// blocks), and unless j is the last pass projection 1, coefficient sweep 2,
// projection 2 (j+1 blocks each).  A dedicated producer warp walks the same
// program: it refills a slot as soon as all 8 consumer warps have released it
// (empty mbarrier), so the consumers never meet at a CTA barrier per chunk.
__host__ __device__ inline int lz_pass_chunks(int nS, int P, int j) {
    const int nb = j + 1;
    const int nsweep = j < 0 ? 0 : (j == P - 1 ? 1 : 4);
    return nS + nsweep * nb;  // nS: this CTA's S chunks
}

template <int NT>  // 8-row tiles per warp: C = 64 NT
__global__ void __launch_bounds__(LZ_CTA, 1)
k_lanczos(const double* __restrict__ S, int C, int P, const double* __restrict__ Q0,
          double* __restrict__ Bm, double* __restrict__ H, double* __restrict__ Bm2,
          double* __restrict__ Wx, int* __restrict__ flags, int split) {
    extern __shared__ __align__(128) uint8_t lz_sm[];
    __shared__ __align__(8) uint64_t full[LZ_NST], empty[LZ_NST];
    const int n = P * LZ_BW;
    const LzSmem L = lz_layout(C, n);
    const int CP = L.cp;
    double* const ring = reinterpret_cast<double*>(lz_sm + L.o_stage);
    double* const Ws = reinterpret_cast<double*>(lz_sm + L.o_w);
    double* const cf = reinterpret_cast<double*>(lz_sm + L.o_cf);
    double* const part = reinterpret_cast<double*>(lz_sm + L.o_part);
    double* const G = reinterpret_cast<double*>(lz_sm + L.o_g);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int lr = lane >> 2, lc = lane & 3;
    // split == 2: a cluster of two CTAs per image.  Each CTA streams half of the
    // rows of S (half the S-pass MMAs and bytes), the two partial W = S Q_j are
    // exchanged through global memory (one flag handshake per pass; the cluster
    // launch guarantees both CTAs are resident), and everything after the S
    // pass runs redundantly in both (bit-identical inputs, each CTA streams its
    // own copy of the basis); CTA 0 writes H and the output basis.
    const int img = blockIdx.x / split, half = blockIdx.x % split;
    const double* const Si = S + (size_t)img * C * C;
    double* const Bi = (half ? Bm2 : Bm) + (size_t)img * n * C;
    double* const Hi = H + (size_t)img * n * n;
    const int nS_all = C / LZ_KC;
    const int c_lo = half * (nS_all / split);
    const int nS = split == 2 ? (half ? nS_all - nS_all / 2 : nS_all / 2) : nS_all;

    if (tid == 0) {
        for (int s = 0; s < LZ_NST; ++s) {
            lz_mbar_init(lz_smem(&full[s]), 1);
            lz_mbar_init(lz_smem(&empty[s]), LZ_NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < C * LZ_BW; i += LZ_CTA) Ws[i] = Q0[i];
    if (half == 0)
        for (int i = tid; i < n * n; i += LZ_CTA) Hi[i] = 0.0;
    __syncthreads();

    if (warp == LZ_NW) {
        // ---------------- producer warp: one elected lane issues every chunk
        if (lane == 0) {
            uint32_t k = 0;  // kernel-wide chunk counter
            for (int j = -1; j < P; ++j) {
                const int nb = j + 1, nch = lz_pass_chunks(nS, P, j);
                for (int c = 0; c < nch; ++c, ++k) {
                    const int s = k % LZ_NST;
                    if (k >= LZ_NST) lz_mbar_wait(lz_smem(&empty[s]), ((k / LZ_NST) - 1) & 1u);
                    // basis chunks are written by the consumers one pass earlier; the
                    // empty-barrier wait orders their (proxy-fenced) stores before this copy
                    const double* src = c < nS ? Si + (size_t)(c_lo + c) * LZ_KC * C
                                               : Bi + (size_t)((c - nS) % nb) * LZ_KC * C;
                    const uint32_t bar = lz_smem(&full[s]);
                    lz_mbar_expect_tx(bar, (uint32_t)LZ_KC * C * 8);
                    double* dst = ring + (size_t)s * LZ_KC * CP;
                    for (int rr = 0; rr < LZ_KC; ++rr)
                        lz_bulk_load(lz_smem(dst + rr * CP), src + (size_t)rr * C, (uint32_t)C * 8,
                                     bar);
                    if (c + LZ_PF < nS)  // S rows further ahead: into L2
                        lz_prefetch_l2(Si + (size_t)(c_lo + c + LZ_PF) * LZ_KC * C,
                                       (uint32_t)LZ_KC * C * 8);
                }
            }
        }
        return;
    }

    // ---------------- consumers (8 warps)
    constexpr int ntile = NT;
    const int wrows = 8 * NT;  // rows per warp
    const int wr0 = warp * wrows;
    uint32_t consumed = 0;
    auto acquire = [&]() -> const double* {
        const int s = consumed % LZ_NST;
        lz_mbar_wait(lz_smem(&full[s]), (consumed / LZ_NST) & 1u);
        return ring + (size_t)s * LZ_KC * CP;
    };
    auto release = [&]() {  // this warp is done with the current chunk
        __syncwarp();
        if (lane == 0) lz_mbar_arrive(lz_smem(&empty[consumed % LZ_NST]));
        ++consumed;
    };

    // W tiles: acc[t] = W[wr0 + 8t + lr][2 lc + {0, 1}]
    double acc[NT][2];
    auto store_w = [&]() {  // acc -> Ws (row-major C x 8)
#pragma unroll
        for (int t = 0; t < NT; ++t)
                *reinterpret_cast<double2*>(Ws + (wr0 + 8 * t + lr) * LZ_BW + 2 * lc) =
                    make_double2(acc[t][0], acc[t][1]);
    };

    for (int j = -1; j < P; ++j) {
        const int nb = j + 1;
        // ---------------- S pass: W = S Q_j = S^T Q_j.  The start pass (j = -1)
        // turns the seeded block R into Q_0 = qr(S R), so the basis lies in
        // range(S): zero rows of S (all-zero channels) stay exact zeros in every
        // Ritz vector, as with the subspace iteration.
#pragma unroll
        for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
        for (int c = 0; c < nS; ++c) {
            const double* st = acquire();
#pragma unroll
            for (int ks = 0; ks < LZ_KC / 4; ++ks) {
                const double b = Ws[((c_lo + c) * LZ_KC + 4 * ks + lc) * LZ_BW + lr];  // Q[k][q]
                const double* arow = st + (4 * ks + lc) * CP + wr0 + lr;      // S[k][r]
#pragma unroll
                for (int t = 0; t < NT; ++t)
                    lz_dmma(acc[t][0], acc[t][1], arow[8 * t], b);
            }
            release();
        }
        if (split == 2) {
            // ---- exchange the partial W with the other CTA of the pair (buffers
            // alternate by pass parity: a buffer is rewritten only after the
            // partner has signalled the following pass, i.e. finished reading it)
            const int par = (j + 1) & 1;
            double* mine = Wx + (((size_t)img * 2 + par) * 2 + half) * C * LZ_BW;
            const double* other = Wx + (((size_t)img * 2 + par) * 2 + (1 - half)) * C * LZ_BW;
#pragma unroll
            for (int t = 0; t < NT; ++t)
                __stcg(reinterpret_cast<double2*>(mine + (wr0 + 8 * t + lr) * LZ_BW + 2 * lc),
                       make_double2(acc[t][0], acc[t][1]));
            __threadfence();
            lz_csync();
            if (tid == 0) {
                atomicAdd(flags + img, 1);
                const int target = 2 * (j + 2);
                while (atomicAdd(flags + img, 0) < target) __nanosleep(64);
                __threadfence();
            }
            lz_csync();
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const double2 o =
                    __ldcg(reinterpret_cast<const double2*>(other + (wr0 + 8 * t + lr) * LZ_BW + 2 * lc));
                acc[t][0] += o.x;  // a + b == b + a: both CTAs hold the same W
                acc[t][1] += o.y;
            }
        }

        // coefficient sweep: cf[8 i + c][q] = B_i[c] . W[:, q]; warp = row slice,
        // partials reduced over the warps in fixed order after the sweep
        auto coef_sweep = [&]() {
            lz_csync();  // every warp done reading Ws (Q_j) in the S pass
            store_w();
            lz_csync();
            for (int i = 0; i < nb; ++i) {
                const double* st = acquire();
                double d0 = 0.0, d1 = 0.0;
                for (int k = 0; k < wrows; k += 4) {
                    const int r = wr0 + k + lc;
                    lz_dmma(d0, d1, st[lr * CP + r], Ws[r * LZ_BW + lr]);
                }
                release();
                double* pp = part + ((i & 1) * LZ_NW + warp) * 64 + lr * 8 + 2 * lc;
                pp[0] = d0;
                pp[1] = d1;
                // block i's partials complete (and block i-2's reduction done, so
                // its half of the double buffer is free again)
                lz_csync();
                if (tid < 64) {
                    const double* src = part + (i & 1) * LZ_NW * 64 + tid;
                    double a = 0.0;
#pragma unroll
                    for (int ww = 0; ww < LZ_NW; ++ww) a += src[ww * 64];
                    cf[i * 64 + tid] = a;
                }
            }
            lz_csync();
        };
        // projection sweep: W -= B_i^T-tiles x cf_i over the streamed blocks
        auto proj_sweep = [&]() {
            for (int i = 0; i < nb; ++i) {
                const double* st = acquire();
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    const double b = -cf[(i * LZ_BW + 4 * ks + lc) * LZ_BW + lr];  // -cf[c][q]
                    const double* arow = st + (4 * ks + lc) * CP + wr0 + lr;       // B_i[c][r]
#pragma unroll
                    for (int t = 0; t < NT; ++t)
                        lz_dmma(acc[t][0], acc[t][1], arow[8 * t], b);
                }
                release();
            }
        };

        const int cols = nb * LZ_BW;
        if (j >= 0) {
            coef_sweep();  // block column j of H
            if (half == 0)
                for (int i = tid; i < cols * LZ_BW; i += LZ_THREADS)
                    Hi[(size_t)(i / LZ_BW) * n + j * LZ_BW + (i % LZ_BW)] = cf[i];
            if (j == P - 1) break;
            proj_sweep();
            coef_sweep();
            proj_sweep();
        }
        // ---------------- Cholesky QR, twice
        double* const Lm = G;
        double* const Ri = G + LZ_BW * LZ_BW;
        double* const dv = G + 2 * LZ_BW * LZ_BW;
        for (int rep = 0; rep < 2; ++rep) {
            lz_csync();  // (Ws / G / part free)
            store_w();
            lz_csync();
            {  // Gram W^T W (a = b = W[row][q]), warp = row slice
                double d0 = 0.0, d1 = 0.0;
                for (int k = 0; k < wrows; k += 4) {
                    const double v = Ws[(wr0 + k + lc) * LZ_BW + lr];
                    lz_dmma(d0, d1, v, v);
                }
                double* pp = part + warp * 64 + lr * 8 + 2 * lc;
                pp[0] = d0;
                pp[1] = d1;
            }
            lz_csync();
            if (warp == 0) {
                // Cholesky G = L L^T with lane i holding row i (lanes 8..31 mirror
                // 0..7), then R^-1 = L^-T: lane c forward-substitutes column c of L^-1
                const int i = lane & 7;
                double l[LZ_BW];
#pragma unroll
                for (int m = 0; m < LZ_BW; ++m) {
                    double a = 0.0;
#pragma unroll
                    for (int ww = 0; ww < LZ_NW; ++ww) a += part[ww * 64 + i * 8 + m];
                    l[m] = a;
                }
                double tr = 0.0;
#pragma unroll
                for (int m = 0; m < LZ_BW; ++m) tr += __shfl_sync(0xffffffffu, l[m], m);
                const double fl = 1e-300 + 1e-28 * tr;
                double dinv = 0.0;
#pragma unroll
                for (int k = 0; k < LZ_BW; ++k) {
                    const double d = __shfl_sync(0xffffffffu, l[k], k);
                    const double rs = d > fl ? rsqrt(d) : 0.0;
                    if (i == k) {
                        l[k] = d * rs;
                        dinv = rs;
                    } else if (i > k) {
                        l[k] *= rs;
                    }
                    const double lk = l[k];
#pragma unroll
                    for (int m = k + 1; m < LZ_BW; ++m) {
                        const double lmk = __shfl_sync(0xffffffffu, lk, m);  // L[m][k]
                        if (i > k) l[m] = fma(-lk, lmk, l[m]);
                    }
                }
                if (lane < LZ_BW) {
#pragma unroll
                    for (int m = 0; m < LZ_BW; ++m) Lm[i * LZ_BW + m] = m <= i ? l[m] : 0.0;
                    dv[i] = dinv;
                }
                __syncwarp();
                if (lane < LZ_BW) {
                    const int c = lane;
                    double x[LZ_BW];
#pragma unroll
                    for (int r = 0; r < LZ_BW; ++r) {
                        double sacc = (r == c) ? 1.0 : 0.0;
#pragma unroll
                        for (int m = 0; m < r; ++m) sacc = fma(-Lm[r * LZ_BW + m], x[m], sacc);
                        x[r] = r < c ? 0.0 : sacc * dv[r];
                    }
                    // Ri[c][r] = Linv[r][c], i.e. Ri[i][q] = (R^-1)[i][q]
#pragma unroll
                    for (int r = 0; r < LZ_BW; ++r) Ri[c * LZ_BW + r] = x[r];
                }
            }
            lz_csync();
            // W <- W R^-1 on the MMAs (A = W tiles from Ws, B = R^-1)
#pragma unroll
            for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
                const double b = Ri[(4 * ks + lc) * LZ_BW + lr];
#pragma unroll
                for (int t = 0; t < NT; ++t)
                    lz_dmma(acc[t][0], acc[t][1], Ws[(wr0 + 8 * t + lr) * LZ_BW + 4 * ks + lc], b);
            }
        }
        // ---------------- Q_{j+1} -> shared (next S pass) and global (later sweeps,
        // read back by the producer's bulk copies: proxy fence before the release
        // arrivals that order them)
        lz_csync();
        store_w();
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const int r = wr0 + 8 * t + lr;
            Bi[(size_t)(cols + 2 * lc) * C + r] = acc[t][0];
            Bi[(size_t)(cols + 2 * lc + 1) * C + r] = acc[t][1];
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");
        lz_csync();
    }
}

size_t lanczos_smem(int C, int P) { return (size_t)lz_layout(C, P * LZ_BW).total; }

int launch_lanczos(const double* S, int64_t batch, int C, int P, const double* Q0, double* Bm,
                   double* H, double* Bm2, double* Wx, int* flags, cudaStream_t st) {
    if (batch <= 0 || C <= 0 || P <= 0) return QFCA_ERR_ARG;
    if (C > LZ_MAXC || C % 64 || P > LZ_MAXP || P * LZ_BW > C) return QFCA_ERR_UNSUPPORTED;
    if (C % (2 * LZ_KC)) return QFCA_ERR_UNSUPPORTED;
    const size_t smem = lanczos_smem(C, P);
    if (smem > 227 * 1024) return QFCA_ERR_UNSUPPORTED;
    void (*kern)(const double*, int, int, const double*, double*, double*, double*, double*, int*,
                 int) = nullptr;
    switch (C / 64) {
        case 1: kern = k_lanczos<1>; break;
        case 2: kern = k_lanczos<2>; break;
        case 3: kern = k_lanczos<3>; break;
        case 4: kern = k_lanczos<4>; break;
        case 5: kern = k_lanczos<5>; break;
        case 6: kern = k_lanczos<6>; break;
        case 7: kern = k_lanczos<7>; break;
        default: kern = k_lanczos<8>; break;
    }
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return QFCA_ERR_CUDA;
    const int split = (Bm2 && Wx && flags) ? 2 : 1;
    if (split == 1) {
        kern<<<(unsigned)batch, LZ_CTA, smem, st>>>(S, C, P, Q0, Bm, H, Bm2, Wx, flags, 1);
        return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
    }
    // two-CTA clusters: the pair is co-scheduled, so the flag handshake cannot deadlock
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * batch));
    cfg.blockDim = dim3(LZ_CTA);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kern, S, C, P, Q0, Bm, H, Bm2, Wx, flags, 2) != cudaSuccess)
        return QFCA_ERR_CUDA;
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

}  // namespace qfca
