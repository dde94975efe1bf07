// eig.cu -- small dense kernels of the top-k eigensolver (features.topk_eigh),
// which replaces np.linalg.eigh of pca_fit (features.py:173-176).
//
//   k_cqr_step    one Cholesky-QR re-orthonormalisation of a subspace-iteration
//                 block Y (C x p, C <= 512, p <= 32) per CTA: Gram (register
//                 4 x 4 blocks over 8 row slices), Cholesky + R^-1 on one warp,
//                 X = Y R^-1 in place, the block resident in shared memory.
//   k_chol_rinv   the same Cholesky -> R^-1 for a batch of p x p Gram matrices
//                 (blocks too tall for k_cqr_step).
//   k_sym_eig     cyclic parallel Jacobi (round-robin pairing, all p/2
//                 rotations of a round applied at once) for the p x p
//                 Rayleigh-Ritz matrices, one warp per matrix, eigenpairs
//                 sorted by descending eigenvalue.
// They replace cuSOLVER calls whose error checks synchronise the host.
#include "common.cuh"

namespace qfca {

constexpr int EIG_MAXP = 32;
constexpr int EIG_LD = EIG_MAXP + 1;  // odd row stride: column walks hit distinct banks

// Cholesky G = L L^T and Rinv = R^-1 = (L^-1)^T on one warp, registers only:
// lane i holds row i of G / L (l[]) and column i of L^-1 (x[]); the entries a
// lane needs from another row arrive by shuffle.  A pivot below the floor
// marks a numerically rank-deficient block: that column of R^-1 is zero (the
// iteration keeps a zero vector instead of NaN).  G (row-major, ldg) is read
// from shared memory, Rinv written to shared memory (row-major, EIG_LD).
__device__ __forceinline__ double shfl_d(double v, int src) {
    return __shfl_sync(0xffffffffu, v, src);
}

__device__ void warp_chol_rinv(const double* G, int ldg, double (*Ls)[EIG_LD], double* sD,
                               double (*Ri)[EIG_LD], int p, int lane) {
    {  // Cholesky in registers: lane i holds row i
        double l[EIG_MAXP];
#pragma unroll
        for (int j = 0; j < EIG_MAXP; ++j) l[j] = (lane < p && j < p) ? G[lane * ldg + j] : 0.0;
        const double floor_ = 1e-300 + 1e-28 * fabs(shfl_d(l[0], 0));
#pragma unroll
        for (int k = 0; k < EIG_MAXP; ++k) {
            const double g = shfl_d(l[k], k);
            const bool ok = k < p && g > floor_;
            const double d = ok ? sqrt(g) : 0.0;
            const double id = ok ? 1.0 / d : 0.0;
            if (lane == 0) sD[k] = id;
            if (lane == k) l[k] = d;
            else if (lane > k) l[k] *= id;
            const double lk = l[k];  // L[lane][k]
#pragma unroll
            for (int j = k + 1; j < EIG_MAXP; ++j) {
                const double ljk = shfl_d(lk, j);  // L[j][k]
                if (lane > k) l[j] = fma(-lk, ljk, l[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < EIG_MAXP; ++j) Ls[lane][j] = l[j];
    }
    __syncwarp();
    // x[i] = (L^-1)[i][lane] by forward substitution (rows of L broadcast from smem)
    double x[EIG_MAXP];
#pragma unroll
    for (int i = 0; i < EIG_MAXP; ++i) {
        double s = i == lane ? 1.0 : 0.0;
#pragma unroll
        for (int j = 0; j < i; ++j) s = fma(-Ls[i][j], x[j], s);
        x[i] = i < lane ? 0.0 : s * sD[i];
    }
    // Rinv[lane][i] = (L^-1)[i][lane]
    if (lane < p) {
#pragma unroll
        for (int i = 0; i < EIG_MAXP; ++i)
            if (i < p) Ri[lane][i] = x[i];
    }
    __syncwarp();
}

// ---------------------------------------------------------------- fused CholQR step
constexpr int CQ_THREADS = 512;
constexpr int CQ_MAXC = 512;
constexpr int CQ_SLICES = 8;

__global__ void __launch_bounds__(CQ_THREADS, 1)
k_cqr_step(double* __restrict__ Y, int C, int p) {
    extern __shared__ __align__(16) double cq[];
    double(*sY)[EIG_LD] = reinterpret_cast<double(*)[EIG_LD]>(cq);                   // [C]
    double(*sP)[EIG_MAXP][EIG_LD] =
        reinterpret_cast<double(*)[EIG_MAXP][EIG_LD]>(cq + (size_t)C * EIG_LD);      // [8]
    double(*sR)[EIG_LD] = sP[0];     // R^-1 (slice 0 reused)
    const int tid = threadIdx.x;
    double* blk = Y + (size_t)blockIdx.x * C * p;
    for (int i = tid; i < C * EIG_MAXP; i += CQ_THREADS) {
        const int r = i / EIG_MAXP, c = i % EIG_MAXP;
        sY[r][c] = c < p ? blk[r * p + c] : 0.0;
    }
    __syncthreads();
    {  // Gram partials: slice s, 4 x 4 block (bi, bj)
        const int s = tid / 64, bidx = tid % 64, bi = bidx / 8, bj = bidx % 8;
        const int r0 = s * C / CQ_SLICES, r1 = (s + 1) * C / CQ_SLICES;
        double acc[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
        for (int r = r0; r < r1; ++r) {
            double a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                a[u] = sY[r][4 * bi + u];
                b[u] = sY[r][4 * bj + u];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
        }
        __syncthreads();  // (no reader of sP yet; keeps the slices' writes ordered)
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) sP[s][4 * bi + u][4 * bj + v] = acc[u][v];
    }
    __syncthreads();
    for (int e = tid; e < EIG_MAXP * EIG_MAXP; e += CQ_THREADS) {
        const int i = e / EIG_MAXP, j = e % EIG_MAXP;
        double g = 0.0;
#pragma unroll
        for (int s = 0; s < CQ_SLICES; ++s) g += sP[s][i][j];
        sP[CQ_SLICES - 1][i][j] = g;  // stage in the last slice (slice 0 gets reused)
    }
    __syncthreads();
    if (tid < 32)
        warp_chol_rinv(&sP[CQ_SLICES - 1][0][0], EIG_LD, sP[1], &sP[2][0][0], sR, p, tid);
    __syncthreads();
    // X = Y R^-1 row by row, in place (column j needs Y columns <= j)
    for (int r = tid; r < C; r += CQ_THREADS) {
        double y[EIG_MAXP];
#pragma unroll
        for (int i = 0; i < EIG_MAXP; ++i) y[i] = sY[r][i];
#pragma unroll
        for (int j = EIG_MAXP - 1; j >= 0; --j) {
            double s = 0.0;
#pragma unroll
            for (int i = 0; i <= j; ++i) s = fma(y[i], sR[i][j], s);
            y[j] = s;
        }
#pragma unroll
        for (int i = 0; i < EIG_MAXP; ++i) sY[r][i] = y[i];
    }
    __syncthreads();
    for (int i = tid; i < C * p; i += CQ_THREADS) blk[i] = sY[i / p][i % p];
}

size_t cqr_step_smem(int C) {
    return ((size_t)C * EIG_LD + (size_t)CQ_SLICES * EIG_MAXP * EIG_LD) * sizeof(double);
}

int launch_cqr_step(double* Y, int64_t batch, int C, int p, cudaStream_t st) {
    if (batch <= 0 || C <= 0 || p <= 0 || p > C) return QFCA_ERR_ARG;
    if (p > EIG_MAXP || C > CQ_MAXC) return QFCA_ERR_UNSUPPORTED;
    const size_t smem = cqr_step_smem(C);
    if (cudaFuncSetAttribute(k_cqr_step, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return QFCA_ERR_CUDA;
    k_cqr_step<<<(unsigned)batch, CQ_THREADS, smem, st>>>(Y, C, p);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

// ---------------------------------------------------------------- batched Gram -> R^-1
constexpr int CR_WARPS = 2;  // matrices per CTA (static shared memory)

__global__ void __launch_bounds__(CR_WARPS * 32)
k_chol_rinv(const double* __restrict__ gram, int64_t batch, int p, double* __restrict__ rinv) {
    __shared__ double sL[CR_WARPS][EIG_MAXP][EIG_LD];
    __shared__ double sI[CR_WARPS][EIG_MAXP][EIG_LD];
    __shared__ double sD[CR_WARPS][EIG_MAXP];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t m = (int64_t)blockIdx.x * CR_WARPS + w;
    if (m >= batch) return;
    const double* G = gram + m * p * p;
    for (int i = 0; i < p; ++i)
        if (lane < p) sL[w][i][lane] = G[i * p + lane];
    __syncwarp();
    warp_chol_rinv(&sL[w][0][0], EIG_LD, sL[w], sD[w], sI[w], p, lane);
    double* out = rinv + m * p * p;
    for (int i = 0; i < p; ++i)
        if (lane < p) out[i * p + lane] = sI[w][i][lane];
}

int launch_chol_rinv(const double* gram, int64_t batch, int p, double* rinv, cudaStream_t st) {
    if (batch <= 0 || p <= 0) return QFCA_ERR_ARG;
    if (p > EIG_MAXP) return QFCA_ERR_UNSUPPORTED;
    k_chol_rinv<<<(unsigned)((batch + CR_WARPS - 1) / CR_WARPS), CR_WARPS * 32, 0, st>>>(
        gram, batch, p, rinv);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

// ---------------------------------------------------------------- parallel Jacobi
// One round applies the p/2 disjoint rotations J of a round-robin pairing at
// once: A <- J^T A J acts on 2 x 2 blocks (pair I rows x pair J columns)
// independently, so each thread updates whole blocks (one barrier per phase);
// a rotated pair's own block gets the exact zero and the closed-form diagonal.
constexpr int JAC_THREADS = 256;  // one 2 x 2 block and two V row-pairs per thread
constexpr int JAC_SWEEPS = 30;

__global__ void __launch_bounds__(JAC_THREADS)
k_sym_eig(const double* __restrict__ h, int64_t batch, int p, double* __restrict__ evals,
          double* __restrict__ evecs) {
    __shared__ double A[EIG_MAXP][EIG_LD];
    __shared__ double V[EIG_MAXP][EIG_LD];
    __shared__ double sc[EIG_MAXP / 2][4];  // c, s, app', aqq'
    __shared__ int sp[EIG_MAXP / 2][2];
    __shared__ int8_t sched[EIG_MAXP - 1][EIG_MAXP];  // round -> player per position
    __shared__ int srank[EIG_MAXP];
    __shared__ int any_rot[2];  // per sweep parity: set by rotations, reset a sweep ahead
    __shared__ double s_tol;
    const int tid = threadIdx.x;
    const int64_t m = blockIdx.x;
    const int n = p + (p & 1);  // players incl. a dummy when p is odd
    const int half = n / 2;
    const double* H = h + m * p * p;
    for (int i = tid; i < p * p; i += JAC_THREADS) {
        const int r = i / p, c = i % p;
        A[r][c] = 0.5 * (H[r * p + c] + H[c * p + r]);
        V[r][c] = r == c ? 1.0 : 0.0;
    }
    if (tid == 0) any_rot[0] = 0;
    __syncthreads();
    if (tid == 0) {
        // rotations stop once an off-diagonal entry is below 1e-16 of the largest
        // |diagonal| (~lambda_1): what is left perturbs eigenvalues by < 1e-16
        // lambda_1 and the well-separated top eigenvectors by ~1e-16 lambda_1 / gap
        double md = 0.0;
        for (int i = 0; i < p; ++i) md = fmax(md, fabs(A[i][i]));
        s_tol = 1e-16 * md;
    }
    // circle method: position 0 fixed, the others rotate by one per round
    for (int i = tid; i < (n - 1) * n; i += JAC_THREADS) {
        const int rnd = i / n, pos = i % n;
        sched[rnd][pos] = (int8_t)(pos == 0 ? 0 : 1 + (pos - 1 + rnd) % (n - 1));
    }
    __syncthreads();
    for (int sweep = 0; sweep < JAC_SWEEPS; ++sweep) {
        if (tid == 0) any_rot[(sweep + 1) & 1] = 0;
        for (int rnd = 0; rnd < n - 1; ++rnd) {
            if (tid < half) {
                int a = sched[rnd][tid], b = sched[rnd][n - 1 - tid];
                if (a > b) { const int t = a; a = b; b = t; }
                double c = 1.0, s = 0.0, app = 0.0, aqq = 0.0;
                if (b < p) {
                    const double apq = A[a][b];
                    app = A[a][a];
                    aqq = A[b][b];
                    // skip entries already negligible against their diagonal pair
                    if (fabs(apq) > s_tol && fabs(apq) > 1e-17 * sqrt(fabs(app * aqq))) {
                        // t = tan(theta) = sgn(d) 2 apq / u with d = aqq - app,
                        // u = |d| + sqrt(d^2 + 4 apq^2); c = u / sqrt(u^2 + 4 apq^2),
                        // s = t c: one sqrt, then rsqrt and 1/u side by side
                        const double d = aqq - app, q2 = 4.0 * apq * apq;
                        const double u = fabs(d) + sqrt(fma(d, d, q2));
                        const double w = rsqrt(fma(u, u, q2));
                        const double sg = d >= 0.0 ? 2.0 * apq : -2.0 * apq;
                        const double tq = sg * apq / u;  // t * apq
                        c = u * w;
                        s = sg * w;
                        app -= tq;  // exact-rotation diagonal
                        aqq += tq;
                        any_rot[sweep & 1] = 1;
                    }
                }
                sc[tid][0] = c;
                sc[tid][1] = s;
                sc[tid][2] = app;
                sc[tid][3] = aqq;
                sp[tid][0] = a;
                sp[tid][1] = b < p ? b : -1;
            }
            __syncthreads();
            for (int k = tid; k < EIG_MAXP * EIG_MAXP / 4; k += JAC_THREADS) {
                const int I = k >> 4, J = k & 15;  // 16 x 16 pair grid, shifts only
                if (I >= half || J >= half) continue;
                const double c1 = sc[I][0], s1 = sc[I][1], c2 = sc[J][0], s2 = sc[J][1];
                if (s1 == 0.0 && s2 == 0.0) continue;
                const int a = sp[I][0], b = sp[I][1], a2 = sp[J][0], b2 = sp[J][1];
                if (I == J) {  // the rotated pair's own block
                    A[a][a] = sc[I][2];
                    A[b][b] = sc[I][3];
                    A[a][b] = 0.0;
                    A[b][a] = 0.0;
                    continue;
                }
                // rows (pair I, b may be the dummy), then columns (pair J)
                const double m00 = A[a][a2];
                const double m01 = b2 >= 0 ? A[a][b2] : 0.0;
                const double m10 = b >= 0 ? A[b][a2] : 0.0;
                const double m11 = (b >= 0 && b2 >= 0) ? A[b][b2] : 0.0;
                const double r00 = c1 * m00 - s1 * m10, r01 = c1 * m01 - s1 * m11;
                const double r10 = s1 * m00 + c1 * m10, r11 = s1 * m01 + c1 * m11;
                A[a][a2] = c2 * r00 - s2 * r01;
                if (b2 >= 0) A[a][b2] = s2 * r00 + c2 * r01;
                if (b >= 0) A[b][a2] = c2 * r10 - s2 * r11;
                if (b >= 0 && b2 >= 0) A[b][b2] = s2 * r10 + c2 * r11;
            }
            for (int k = tid; k < (EIG_MAXP / 2) * EIG_MAXP; k += JAC_THREADS) {  // V <- V J
                const int I = k >> 5, r = k & 31;
                if (I >= half || r >= p) continue;
                const double c = sc[I][0], s = sc[I][1];
                const int a = sp[I][0], b = sp[I][1];
                if (s == 0.0 || b < 0) continue;
                const double u = V[r][a], v = V[r][b];
                V[r][a] = c * u - s * v;
                V[r][b] = s * u + c * v;
            }
            __syncthreads();
        }
        if (!any_rot[sweep & 1]) break;
    }
    // descending order (ties: lower index first)
    if (tid < p) {
        const double li = A[tid][tid];
        int rk = 0;
        for (int j = 0; j < p; ++j) {
            const double lj = A[j][j];
            rk += (lj > li) || (lj == li && j < tid);
        }
        srank[tid] = rk;
        evals[m * p + rk] = li;
    }
    __syncthreads();
    for (int i = tid; i < p * p; i += JAC_THREADS) {
        const int r = i / p, c = i % p;  // V[r][c]: component r of vector c
        evecs[m * p * p + r * p + srank[c]] = V[r][c];
    }
}

int launch_sym_eig(const double* h, int64_t batch, int p, double* evals, double* evecs,
                   cudaStream_t st) {
    if (batch <= 0 || p <= 0) return QFCA_ERR_ARG;
    if (p > EIG_MAXP) return QFCA_ERR_UNSUPPORTED;
    k_sym_eig<<<(unsigned)batch, JAC_THREADS, 0, st>>>(h, batch, p, evals, evecs);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}


// ---------------------------------------------------------------- Ritz pairs of H
// Top-p subspace of the small Lanczos projection H = B^T S B (n <= 128, p = 32)
// in one CTA per image: X <- qr(H (H X)) for `iters` steps (m8n8k4 fp64 MMAs,
// Gram + warp Cholesky + X R^-1), then Hm = X^T H X.  Same iteration as
// features.topk_eigh on cov^2 (fifteen steps: (theta_33 / theta_10)^30 ~ 1e-16),
// fused so that the small problem costs one launch instead of ~35.  H arrives
// as lanczos.cu writes it (upper block triangle); X0 is the seeded start block.
namespace {
constexpr int RZ_P = 32;
constexpr int RZ_MAXN = 128;
constexpr int RZ_THREADS = 256;
constexpr int RZ_NW = RZ_THREADS / 32;
constexpr int RZ_XP = RZ_P + 4;  // padded pitch of the n x 32 blocks (conflict-free fragments)

__device__ __forceinline__ void rz_dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// out (n x 32) = A (n x n, pitch ha) . X (n x 32, pitch RZ_XP); warp w owns row
// tiles w and w + 8 (n = 128; fewer rows: tiles past n/8 idle) and all four
// column tiles: eight independent accumulator chains per warp
__device__ __forceinline__ void rz_mul(const double* A, int ha, const double* X, double* out,
                                       int n, int warp, int lr, int lc) {
    const int nt = n / 8;
    const int r0 = warp, r1 = warp + RZ_NW;
    const bool v0 = r0 < nt, v1 = r1 < nt;
    double d[2][4][2] = {};
    for (int k = 0; k < n; k += 4) {
        double b[4];
#pragma unroll
        for (int ct = 0; ct < 4; ++ct) b[ct] = X[(k + lc) * RZ_XP + ct * 8 + lr];
        if (v0) {
            const double a = A[(r0 * 8 + lr) * ha + k + lc];
#pragma unroll
            for (int ct = 0; ct < 4; ++ct) rz_dmma(d[0][ct][0], d[0][ct][1], a, b[ct]);
        }
        if (v1) {
            const double a = A[(r1 * 8 + lr) * ha + k + lc];
#pragma unroll
            for (int ct = 0; ct < 4; ++ct) rz_dmma(d[1][ct][0], d[1][ct][1], a, b[ct]);
        }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int rt = h ? r1 : r0;
        if (h ? !v1 : !v0) continue;
#pragma unroll
        for (int ct = 0; ct < 4; ++ct) {
            out[(rt * 8 + lr) * RZ_XP + ct * 8 + 2 * lc] = d[h][ct][0];
            out[(rt * 8 + lr) * RZ_XP + ct * 8 + 2 * lc + 1] = d[h][ct][1];
        }
    }
}

// G (32 x 32, pitch EIG_LD) = Y^T Z over n rows; warp w owns tiles 2w, 2w + 1,
// each over two interleaved k halves (four independent chains)
__device__ __forceinline__ void rz_gram(const double* Y, const double* Z, double* G, int n,
                                        int warp, int lr, int lc) {
    double d[2][2][2] = {};
    const int t0 = 2 * warp;
    for (int k = 0; k < n; k += 8) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int mt = (t0 + h) >> 2, ntl = (t0 + h) & 3;
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const int kk = k + 4 * s + lc;
                rz_dmma(d[h][s][0], d[h][s][1], Y[kk * RZ_XP + mt * 8 + lr], Z[kk * RZ_XP + ntl * 8 + lr]);
            }
        }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int mt = (t0 + h) >> 2, ntl = (t0 + h) & 3;
        G[(mt * 8 + lr) * EIG_LD + ntl * 8 + 2 * lc] = d[h][0][0] + d[h][1][0];
        G[(mt * 8 + lr) * EIG_LD + ntl * 8 + 2 * lc + 1] = d[h][0][1] + d[h][1][1];
    }
}
}  // namespace

// Cholesky G = L L^T (32 x 32, G in shared memory, pitch EIG_LD) and
// Ri = R^-1 = L^-T on one warp.  Lane i holds the trailing part of row i in
// registers (shifted left every step, so no register array is indexed at run
// time); column k of L goes through shared memory transposed (LT[k][i], rows
// contiguous: one broadcast vector load per two entries) -- LT may alias G.
// Lane c then forward-substitutes column c of L^-1, which is row c of R^-1.
// One rsqrt per pivot; a pivot below 1e-28 of the trace leaves a zero column.
__device__ __forceinline__ void rz_chol_rinv32(const double* G, double* LT, double* sD,
                                               double (*Ri)[EIG_LD], int lane) {
    double l[RZ_P];  // l[j] = G'[lane][k + j] at step k
#pragma unroll
    for (int j = 0; j < RZ_P; ++j) l[j] = G[lane * EIG_LD + j];
    double tr = G[lane * EIG_LD + lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
    const double fl = 1e-300 + 1e-28 * tr;
    __syncwarp();  // G fully read before LT overwrites it
#pragma unroll 1
    for (int k = 0; k < RZ_P; ++k) {
        const double d = __shfl_sync(0xffffffffu, l[0], k);
        const double rs = d > fl ? rsqrt(d) : 0.0;
        double lk = 0.0;  // L[lane][k] (0 above the diagonal)
        if (lane == k) {
            lk = d * rs;
            sD[k] = rs;
        } else if (lane > k) {
            lk = l[0] * rs;
        }
        LT[k * RZ_P + lane] = lk;
        __syncwarp();
        // trailing update + shift: l[j] <- G'[lane][k+1+j] - L[lane][k] L[k+1+j][k].
        // Lanes < k have lk = 0 (no change); lane k's row is final and no longer
        // read.  Entries k+1+j > 31 read on into the next LT rows / the rest of
        // the G area (finite values) and only feed columns past 31, never used.
        const double* col = LT + k * RZ_P + k + 1;
#pragma unroll
        for (int j = 0; j < RZ_P - 1; ++j) l[j] = fma(-lk, col[j], l[j + 1]);
        l[RZ_P - 1] = 0.0;
    }
    __syncwarp();
    // x = column c of L^-1: x[r] = (delta_rc - sum_{m < r} L[r][m] x[m]) / L[r][r]
    const int c = lane;
#pragma unroll
    for (int r = 0; r < RZ_P; ++r) {
        double a0 = (r == c) ? 1.0 : 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int m = 0; m < r; ++m) {
            const double t = -LT[m * RZ_P + r] * l[m];  // L[r][m] x[m]
            if ((m & 3) == 0) a0 += t;
            else if ((m & 3) == 1) a1 += t;
            else if ((m & 3) == 2) a2 += t;
            else a3 += t;
        }
        l[r] = r < c ? 0.0 : ((a0 + a1) + (a2 + a3)) * sD[r];  // (l reused as x)
    }
    // Ri[c][q] = (R^-1)[c][q] = Linv[q][c] = x[q]
#pragma unroll
    for (int q = 0; q < RZ_P; ++q) Ri[c][q] = l[q];
    __syncwarp();
}

__global__ void __launch_bounds__(RZ_THREADS, 1)
k_ritz(const double* __restrict__ h, int n, const double* __restrict__ x0, int iters,
       double* __restrict__ xout, double* __restrict__ hm) {
    extern __shared__ __align__(16) double rz[];
    const int hp = n + 4;  // Hs pitch: (4 lr + lc) mod 16 distinct -> conflict-free A fragments
    double* const Hs = rz;                                          // n x hp
    double* bufA = Hs + (size_t)n * hp;                             // n x RZ_XP
    double* bufB = bufA + (size_t)n * RZ_XP;                        // n x RZ_XP
    double(*G)[EIG_LD] = reinterpret_cast<double(*)[EIG_LD]>(bufB + (size_t)n * RZ_XP);
    double(*Ri)[EIG_LD] = G + RZ_P;
    double* sD = &Ri[RZ_P][0];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int lr = lane >> 2, lc = lane & 3;
    const int64_t m = blockIdx.x;
    const double* H = h + m * n * n;
    for (int e = tid; e < n * n; e += RZ_THREADS) {
        const int i = e / n, j = e % n;
        Hs[i * hp + j] = i <= j ? H[i * n + j] : H[j * n + i];
    }
    for (int e = tid; e < n * RZ_P; e += RZ_THREADS) bufA[(e / RZ_P) * RZ_XP + e % RZ_P] = x0[e];
    __syncthreads();
    for (int it = 0; it < iters; ++it) {
        rz_mul(Hs, hp, bufA, bufB, n, warp, lr, lc);  // T = H X
        __syncthreads();
        rz_mul(Hs, hp, bufB, bufA, n, warp, lr, lc);  // Y = H T
        __syncthreads();
        rz_gram(bufA, bufA, &G[0][0], n, warp, lr, lc);
        __syncthreads();
        if (warp == 0) rz_chol_rinv32(&G[0][0], &G[0][0], sD, Ri, lane);
        __syncthreads();
        // X = Y R^-1 -> bufB
        for (int rt = warp; rt < n / 8; rt += RZ_NW) {
            double d[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
#pragma unroll
            for (int k = 0; k < RZ_P; k += 4) {
                const double a = bufA[(rt * 8 + lr) * RZ_XP + k + lc];
#pragma unroll
                for (int ct = 0; ct < 4; ++ct) rz_dmma(d[ct][0], d[ct][1], a, Ri[k + lc][ct * 8 + lr]);
            }
#pragma unroll
            for (int ct = 0; ct < 4; ++ct) {
                bufB[(rt * 8 + lr) * RZ_XP + ct * 8 + 2 * lc] = d[ct][0];
                bufB[(rt * 8 + lr) * RZ_XP + ct * 8 + 2 * lc + 1] = d[ct][1];
            }
        }
        __syncthreads();
        double* t = bufA;
        bufA = bufB;
        bufB = t;
    }
    // Rayleigh-Ritz matrix Hm = X^T (H X)
    rz_mul(Hs, hp, bufA, bufB, n, warp, lr, lc);
    __syncthreads();
    rz_gram(bufA, bufB, &G[0][0], n, warp, lr, lc);
    __syncthreads();
    for (int e = tid; e < RZ_P * RZ_P; e += RZ_THREADS) {
        const int i = e / RZ_P, j = e % RZ_P;
        hm[m * RZ_P * RZ_P + e] = 0.5 * (G[i][j] + G[j][i]);
    }
    for (int e = tid; e < n * RZ_P; e += RZ_THREADS)
        xout[m * n * RZ_P + e] = bufA[(e / RZ_P) * RZ_XP + e % RZ_P];
}

size_t ritz_smem(int n) {
    return ((size_t)n * (n + 4) + 2 * (size_t)n * RZ_XP + 2 * (size_t)RZ_P * EIG_LD + RZ_P) *
           sizeof(double);
}

int launch_ritz(const double* h, int64_t batch, int n, const double* x0, int iters, double* xout,
                double* hm, cudaStream_t st) {
    if (batch <= 0 || n <= 0 || iters < 0) return QFCA_ERR_ARG;
    if (n > RZ_MAXN || n % 8 || n < RZ_P) return QFCA_ERR_UNSUPPORTED;  // (n % 8: k steps of 8 in rz_gram)
    const size_t smem = ritz_smem(n);
    if (cudaFuncSetAttribute(k_ritz, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return QFCA_ERR_CUDA;
    k_ritz<<<(unsigned)batch, RZ_THREADS, smem, st>>>(h, n, x0, iters, xout, hm);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}
}  // namespace qfca
