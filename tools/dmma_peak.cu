// dmma_peak.cu -- does the FP64 tensor-core MMA (DMMA, mma.sync m8n8k4 f64) add throughput
// on top of the FP64 DFMA pipe on B200?  Three kernels, best of 5 each (CUDA events):
//   dfma  : 8 independent DFMA chains per thread
//   dmma  : 4 independent m8n8k4 f64 accumulator chains per warp (512 flop per instruction)
//   mixed : both in the same loop (if the pipes are separate, the sum exceeds either alone)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/dmma_peak tools/dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int DCH = 8, MCH = 4;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int MODE>   // 0 dfma, 1 dmma, 2 both
__global__ void k_bench(double* out, int iters, double a, double b)
{
    double x[DCH], d[MCH][2];
#pragma unroll
    for (int c = 0; c < DCH; ++c) x[c] = threadIdx.x * 1e-9 + c;
#pragma unroll
    for (int c = 0; c < MCH; ++c) d[c][0] = d[c][1] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < iters; ++i) {
        if (MODE != 1) {
#pragma unroll
            for (int c = 0; c < DCH; ++c) x[c] = fma(x[c], a, b);
        }
        if (MODE != 0) {
#pragma unroll
            for (int c = 0; c < MCH; ++c) dmma(d[c][0], d[c][1], a, b);
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < DCH; ++c) s += x[c];
#pragma unroll
    for (int c = 0; c < MCH; ++c) s += d[c][0] + d[c][1];
    if (s == 12345.678) out[0] = s;
}

template <int MODE>
static double run(double* out, int blocks, int threads, int iters)
{
    k_bench<MODE><<<blocks, threads>>>(out, 256, 0.999999, 1e-7);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_bench<MODE><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double warps = (double)blocks * threads / 32;
        double flop = 0;
        if (MODE != 1) flop += 2.0 * DCH * iters * (double)blocks * threads;
        if (MODE != 0) flop += 512.0 * MCH * iters * warps;
        const double tf = flop / (ms * 1e-3) / 1e12;
        if (tf > best) best = tf;
    }
    return best;
}

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    const int threads = 256, blocks = sms * 8, iters = 1 << 14;
    const double a = run<0>(out, blocks, threads, iters);
    const double b = run<1>(out, blocks, threads, iters);
    const double c = run<2>(out, blocks, threads, iters);
    cudaError_t e = cudaGetLastError();
    printf("{\"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, \"mixed_tflops\": %.3f, \"how\": \"%d blocks x %d threads, "
           "%d DFMA chains/thread, %d m8n8k4 f64 chains/warp, %d iters, best of 5\", \"cuda\": \"%s\"}\n",
           a, b, c, blocks, threads, DCH, MCH, iters, cudaGetErrorString(e));
    return e != cudaSuccess;
}
