// Microbenchmark: per-CTA streaming of a 2 MiB matrix through a cp.async.bulk +
// mbarrier ring (the block-Lanczos S pass), with and without the DFMA work.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
__device__ __forceinline__ uint32_t sm32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint32_t b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c)); }
__device__ __forceinline__ void mb_tx(uint32_t b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(n) : "memory"); }
__device__ __forceinline__ void mb_wait(uint32_t b, uint32_t ph) {
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(b), "r"(ph) : "memory"); }
__device__ __forceinline__ void bulk(uint32_t d, const void* s, uint32_t n, uint32_t b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d), "l"(s), "r"(n), "r"(b) : "memory"); }
template <int NST, int KC, int SPLIT, bool COMPUTE>
__global__ void __launch_bounds__(256, 1) k_ring(const double* S, int C, int passes, double* out) {
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t mbar[NST];
    const int tid = threadIdx.x;
    const double* Si = S + (size_t)blockIdx.x * C * C;
    double* Qs = sm + NST * KC * C;
    if (tid == 0) { for (int s = 0; s < NST; ++s) mb_init(sm32(&mbar[s]), 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    for (int i = tid; i < C * 8; i += 256) Qs[i] = 1e-3 * (i % 7);
    __syncthreads();
    uint32_t issued = 0, consumed = 0;
    const int nS = C / KC;
    double w[2][8] = {};
    for (int p = 0; p < passes; ++p) {
        auto issue = [&](int c) {
            const int s = issued % NST; ++issued;
            const uint32_t b = sm32(&mbar[s]);
            mb_tx(b, KC * C * 8);
            const uint32_t bytes = KC * C * 8 / SPLIT;
            for (int k = 0; k < SPLIT; ++k)
                bulk(sm32(sm + (size_t)s * KC * C) + k * bytes, (const char*)(Si + (size_t)c * KC * C) + k * bytes, bytes, b);
        };
        if (tid == 0) for (int c = 0; c < NST && c < nS; ++c) issue(c);
        for (int c = 0; c < nS; ++c) {
            const int s = consumed % NST;
            mb_wait(sm32(&mbar[s]), (consumed / NST) & 1u); ++consumed;
            const double* st = sm + (size_t)s * KC * C;
            if (COMPUTE) {
#pragma unroll
                for (int kk = 0; kk < KC; ++kk) {
                    const double2 sv = *reinterpret_cast<const double2*>(st + kk * C + 2 * tid);
                    const double* qk = Qs + (c * KC + kk) * 8;
#pragma unroll
                    for (int q = 0; q < 8; ++q) { w[0][q] = fma(sv.x, qk[q], w[0][q]); w[1][q] = fma(sv.y, qk[q], w[1][q]); }
                }
            } else if (tid < 8) w[0][0] += st[tid];
            __syncthreads();
            if (tid == 0 && c + NST < nS) issue(c + NST);
        }
        __syncthreads();
    }
    double a = 0; for (int q = 0; q < 8; ++q) a += w[0][q] + w[1][q];
    out[blockIdx.x * 256 + tid] = a;
}
template <int NST, int KC, int SPLIT, bool COMPUTE>
void run(const double* S, double* out, int B, int C, int passes, const char* name) {
    size_t smem = (size_t)NST * KC * C * 8 + C * 8 * 8;
    cudaFuncSetAttribute(k_ring<NST, KC, SPLIT, COMPUTE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    k_ring<NST, KC, SPLIT, COMPUTE><<<B, 256, smem>>>(S, C, passes, out);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) k_ring<NST, KC, SPLIT, COMPUTE><<<B, 256, smem>>>(S, C, passes, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 3;
    printf("%-34s B=%3d %.3f ms  %.0f GB/s  %s\n", name, B, ms, (double)B * C * C * 8 * passes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    const int C = 512, passes = 17;
    double *S, *out; cudaMalloc(&S, (size_t)148 * C * C * 8); cudaMalloc(&out, 148 * 256 * 8);
    cudaMemset(S, 0, (size_t)148 * C * C * 8);
    for (int B : {64, 148}) {
        run<3, 8, 8, false>(S, out, B, C, passes, "nst3 kc8 split8 nocompute");
        run<3, 8, 1, false>(S, out, B, C, passes, "nst3 kc8 split1 nocompute");
        run<6, 8, 1, false>(S, out, B, C, passes, "nst6 kc8 split1 nocompute");
        run<12, 4, 1, false>(S, out, B, C, passes, "nst12 kc4 split1 nocompute");
        run<3, 8, 8, true>(S, out, B, C, passes, "nst3 kc8 split8 compute");
        run<6, 8, 1, true>(S, out, B, C, passes, "nst6 kc8 split1 compute");
        run<12, 4, 1, true>(S, out, B, C, passes, "nst12 kc4 split1 compute");
    }
    return 0;
}
