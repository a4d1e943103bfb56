// FP64 peak microbenchmark ("FP64 peak is not in
// MEASURED_PEAKS.json; measure it before quoting FP64 fractions").
//   dfma: independent DFMA chains, 148*k blocks of 256 threads
//   dmma: mma.sync.aligned.m8n8k4.row.col.f64 (FP64 tensor core), 8 chains
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void dfma_kernel(double* out, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
        x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i)
            x[i] = fma(x[i], a, b);
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
        s += x[i];
    if (s == 1234.5)
        out[threadIdx.x] = s;
}

__global__ void dmma_kernel(double* out, double a) {
    double acc[8][2];
    double fa = a * threadIdx.x, fb = a + threadIdx.x;
#pragma unroll
    for (int i = 0; i < 8; ++i)
        acc[i][0] = acc[i][1] = 0.0;
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(acc[i][0]), "+d"(acc[i][1])
                         : "d"(fa), "d"(fb));
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
        s += acc[i][0] + acc[i][1];
    if (s == 1234.5)
        out[threadIdx.x] = s;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 1024 * sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int bps : {2, 4, 8}) {
        const int blocks = sms * bps, threads = 256;
        dfma_kernel<<<blocks, threads>>>(out, 1.0000001, 1e-9);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r)
            dfma_kernel<<<blocks, threads>>>(out, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 5.0 * blocks * threads * kIters * 8 * 2;
        printf("dfma blocks/SM=%d  %.2f TFLOP/s\n", bps, flops / (ms / 1e3) / 1e12);
        dmma_kernel<<<blocks, threads>>>(out, 1.0);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r)
            dmma_kernel<<<blocks, threads>>>(out, 1.0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double mflops = 5.0 * blocks * (threads / 32) * kIters * 8 * (8.0 * 8 * 4 * 2);
        printf("dmma blocks/SM=%d  %.2f TFLOP/s (%s)\n", bps, mflops / (ms / 1e3) / 1e12,
               cudaGetErrorString(cudaGetLastError()));
    }
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("SMs=%d clock(attr)=%d kHz\n", sms, clk);
    return 0;
}
