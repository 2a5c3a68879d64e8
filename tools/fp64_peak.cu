// fp64_peak.cu — measured FP64 DFMA throughput of this B200 (the "alu" roofline denominator
// of bench.py; VERDICT r1 asked for a measured, not derived, FP64 peak).
//
// Every thread runs 8 independent DFMA chains (enough ILP to cover the pipe latency) for
// `iters` iterations; 148 × 8 blocks of 256 threads keep every SM's FP64 pipe busy.  Flops =
// 2 × threads × 8 × iters; timed with CUDA events after a warm-up launch; best of 10.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) dfma_kernel(double *out, int iters, double a, double b)
{
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;     // never true: keeps the chains live
}

int main()
{
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double *out;
    cudaMalloc(&out, 8);
    const int blocks = sms * 8, threads = 256, iters = 1 << 14;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
        cudaEventRecord(e0);
        dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double flops = 2.0 * blocks * threads * 8.0 * iters;
    const double tf = flops / (best * 1e-3) / 1e12;
    const double per_sm_clk = flops / 2.0 / (best * 1e-3) / sms / (clk * 1e3);
    printf("{\"fp64_dfma_tflops\": %.3f, \"dfma_per_sm_per_clk_at_attr_clock\": %.2f, \"sms\": %d, "
           "\"attr_clock_mhz\": %.0f, \"best_ms\": %.4f, \"how\": \"%d blocks x %d threads x 8 independent DFMA "
           "chains x %d iters, CUDA events, best of 10\"}\n",
           tf, per_sm_clk, sms, clk / 1e3, best, blocks, threads, iters);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
