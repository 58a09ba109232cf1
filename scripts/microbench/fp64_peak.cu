// Microbenchmark: FP64 DFMA and DMMA (mma.sync m8n8k4 f64) throughput on B200.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters) {
    double a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
    const double b = 1.0000001, c = 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += a[i];
    if (s == 1.2345) out[0] = s;
}

__global__ void k_dmma(double* out, int iters) {
    double acc[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { acc[i][0] = threadIdx.x; acc[i][1] = 1.0; }
    double a = 1.0 + threadIdx.x * 1e-6, b = 0.999;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
    if (s == 1.2345) out[0] = s;
}

int main() {
    double* d; cudaMalloc(&d, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int threads : {128, 256, 512, 1024}) {
        int iters = 4096, blocks = sms * (2048 / threads);
        k_dfma<<<blocks, threads>>>(d, 16);
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(d, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 16 * iters * (double)blocks * threads;
        printf("DFMA threads/blk %4d: %.2f TFLOP/s\n", threads, flops / ms / 1e9);
        k_dmma<<<blocks, threads>>>(d, 16);
        cudaEventRecord(e0);
        k_dmma<<<blocks, threads>>>(d, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        flops = 2.0 * 256 * 8 * iters * (double)blocks * (threads / 32);
        printf("DMMA threads/blk %4d: %.2f TFLOP/s\n", threads, flops / ms / 1e9);
    }
    return 0;
}
