#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, int iters, double a) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
        x0 = fma(x0, a, 1.0); x1 = fma(x1, a, 1.0); x2 = fma(x2, a, 1.0); x3 = fma(x3, a, 1.0);
        x4 = fma(x4, a, 1.0); x5 = fma(x5, a, 1.0); x6 = fma(x6, a, 1.0); x7 = fma(x7, a, 1.0);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void kf(float* out, int iters, float a) {
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
        x0 = fmaf(x0, a, 1.0f); x1 = fmaf(x1, a, 1.0f); x2 = fmaf(x2, a, 1.0f); x3 = fmaf(x3, a, 1.0f);
        x4 = fmaf(x4, a, 1.0f); x5 = fmaf(x5, a, 1.0f); x6 = fmaf(x6, a, 1.0f); x7 = fmaf(x7, a, 1.0f);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void klat(double* out, int iters, double a) {
    double x0 = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) x0 = fma(x0, a, 1.0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (double)(t1 - t0) / iters;
    out[1 + threadIdx.x] = x0;
}
__global__ void kdiv(double* out, int iters, double a) {
    double x0 = threadIdx.x + 1.5;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) x0 = a / x0 + 1.0;
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (double)(t1 - t0) / iters;
    out[1 + threadIdx.x] = x0;
}
__global__ void ksqrt(double* out, int iters) {
    double x0 = threadIdx.x + 1.5;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) x0 = sqrt(x0) + 1.0;
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (double)(t1 - t0) / iters;
    out[1 + threadIdx.x] = x0;
}
template <int NACC>
__global__ void kdmma(double* out, int iters, double a) {
    double d[NACC][2];
    for (int t = 0; t < NACC; ++t) d[t][0] = d[t][1] = threadIdx.x + t;
    double b = a * threadIdx.x;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int t = 0; t < NACC; ++t)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(d[t][0]), "+d"(d[t][1]) : "d"(a), "d"(b));
    }
    double s = 0; for (int t = 0; t < NACC; ++t) s += d[t][0] + d[t][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int NACC>
void run_dmma(double* d, int sms, int th, int per_sm) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int iters = 1 << 12, blocks = sms * per_sm;
    kdmma<NACC><<<blocks, th>>>(d, 10, 1.0000001); cudaDeviceSynchronize();
    cudaEventRecord(e0); kdmma<NACC><<<blocks, th>>>(d, iters, 1.0000001); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 256 * NACC * iters * (double)blocks * th / 32;
    printf("DMMA m8n8k4 acc=%d warps/SM=%d: %.1f TFLOPS (%.1f FMA/clk/SM)\n", NACC, per_sm * th / 32, fl / ms / 1e9, fl / 2 / (ms * 1e-3) / sms / 1.965e9);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d; cudaMalloc(&d, 1 << 26); float* f = (float*)d;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int iters = 1 << 14, blocks = sms * 8, th = 256;
    k<<<blocks, th>>>(d, 10, 1.0000001); cudaDeviceSynchronize();
    cudaEventRecord(e0); k<<<blocks, th>>>(d, iters, 1.0000001); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * (double)blocks * th;
    printf("fp64 FMA: %.1f TFLOPS (%.1f DFMA/clk/SM at 1.965GHz)\n", fl / ms / 1e9, fl / 2 / (ms * 1e-3) / sms / 1.965e9);
    cudaEventRecord(e0); kf<<<blocks, th>>>(f, iters, 1.0000001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("fp32 FMA: %.1f TFLOPS\n", fl / ms / 1e9);
    double h[2];
    klat<<<1, 32>>>(d, 4096, 1.0000001); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); printf("DFMA latency %.1f clk\n", h[0]);
    kdiv<<<1, 32>>>(d, 4096, 1.0000001); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); printf("fp64 div+add latency %.1f clk\n", h[0]);
    ksqrt<<<1, 32>>>(d, 4096); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); printf("fp64 sqrt+add latency %.1f clk\n", h[0]);
    run_dmma<1>(d, sms, 256, 1); run_dmma<4>(d, sms, 256, 1); run_dmma<8>(d, sms, 256, 1);
    run_dmma<8>(d, sms, 512, 1); run_dmma<8>(d, sms, 256, 4); run_dmma<16>(d, sms, 256, 2);
    return 0;
}
