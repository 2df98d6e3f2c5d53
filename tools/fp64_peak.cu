// fp64_peak.cu -- FP64 DFMA throughput microbenchmark (the roofline denominator for
// the FP64-ALU-bound kernels; MEASURED_PEAKS.json carries no FP64 figure).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/fp64_peak tools/fp64_peak.cu
//   ./build/fp64_peak > profiles/fp64_peak.json
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CHAINS = 8;
__global__ void k_dfma(double* out, int iters, double a, double b)
{
    double x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;
}

int main()
{
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double* out;
    cudaMalloc(&out, 8);
    const int threads = 256, blocks = sms * 8, iters = 1 << 16;
    k_dfma<<<blocks, threads>>>(out, 1024, 0.999999, 1e-7);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        double tf = 2.0 * CHAINS * (double)iters * threads * blocks / (ms * 1e-3) / 1e12;
        if (tf > best) best = tf;
    }
    cudaError_t e = cudaGetLastError();
    printf("{\"dfma_tflops\": %.3f, \"sms\": %d, \"max_clock_mhz\": %d, \"how\": \"%d independent DFMA chains x %d iters, "
           "%d blocks x %d threads, best of 5, CUDA events\", \"cuda\": \"%s\"}\n",
           best, sms, clk / 1000, CHAINS, iters, blocks, threads, cudaGetErrorString(e));
    return e != cudaSuccess;
}
