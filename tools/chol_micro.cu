// Latency of the one-warp 32 x 32 Cholesky + R^-1 used by k_ritz (eig.cu).
#include <cstdio>
#include "../paper_2510_15602_b200/csrc/eig.cu"
using namespace qfca;
namespace qfca {
__device__ __forceinline__ void rz_chol_t(const double* G, double* LT, double* sD,
                                               double (*Ri)[EIG_LD], int lane, long long* ph) {
    ph[0] -= clock64();
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
    ph[0] += clock64();
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

}

__global__ void k_chol_bench(double* out, int reps) {
    __shared__ double G[32][EIG_LD], Ri[32][EIG_LD], sD[32], G0[32][EIG_LD];
    const int lane = threadIdx.x;
    for (int j = 0; j < 32; ++j) G0[lane][j] = (lane == j ? 64.0 : 0.0) + 1.0 / (1 + lane + j);
    __syncwarp();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        for (int j = 0; j < 32; ++j) G[lane][j] = G0[lane][j];
        __syncwarp();
        rz_chol_rinv32(&G[0][0], &G[0][0], sD, Ri, lane);
        __syncwarp();
    }
    long long t1 = clock64();
    long long t2 = clock64();
    for (int r = 0; r < reps; ++r) {
        for (int j = 0; j < 32; ++j) G[lane][j] = G0[lane][j];
        __syncwarp();
        warp_chol_rinv(&G[0][0], EIG_LD, G, sD, Ri, 32, lane);
        __syncwarp();
    }
    long long t3 = clock64();
    long long ph = 0;
    for (int r = 0; r < reps; ++r) {
        for (int j = 0; j < 32; ++j) G[lane][j] = G0[lane][j];
        __syncwarp();
        rz_chol_t(&G[0][0], &G[0][0], sD, Ri, lane, &ph);
        __syncwarp();
    }
    if (lane == 0) out[3] = (double)ph / reps;
    if (lane == 0) { out[0] = (double)(t1 - t0) / reps; out[1] = (double)(t3 - t2) / reps; out[2] = Ri[3][5]; }
}
int main() {
    double* d; cudaMalloc(&d, 64);
    k_chol_bench<<<1, 32>>>(d, 10);
    double h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("rz_chol_rinv32 %.0f clk (factor %.0f), warp_chol_rinv %.0f clk (%g)\n", h[0], h[3], h[1], h[2]);
    return 0;
}
