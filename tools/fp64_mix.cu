// fp64_mix.cu -- how the FP64 pipe of one SM sub-partition shares issue with other instruction
// classes (the question behind k_near's 62-70 % FP64-pipe ceiling).
// Every kernel runs CHAINS independent DFMA chains per thread at k_near's occupancy (8 blocks of
// 128 threads per SM) and adds, per DFMA, E extra instructions of one class that do not depend
// on the FP64 results.  Reported: DFMA rate as a fraction of the nominal FP64 peak
// (SMs x 64 lanes x clock), per mode.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/fp64_mix tools/fp64_mix.cu
//   ./build/fp64_mix > profiles/r02/fp64_mix.json
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CHAINS = 8;
enum Mode { PURE = 0, DISTINCT, ALU1, ALU2, IMAD1, IMAD2, FSEL2, LDS1, LDSR, MUFU8, MIXOPS, KNEARMIX, NMODES };
static const char* kNames[NMODES] = {"dfma_shared_operands", "dfma_distinct_operands", "dfma+1alu", "dfma+2alu",
                                     "dfma+1imad", "dfma+2imad", "dfma+2fsel", "dfma+1lds_broadcast",
                                     "dfma+1lds128_random", "dfma+mufu_per_8", "dadd_dmul_dfma_mix", "k_near_like_mix"};

template <int MODE>
__global__ void __launch_bounds__(128, 8) k_mix(double* out, int iters, double a, double b, unsigned seed)
{
    __shared__ double2 tab[512];
    for (int i = threadIdx.x; i < 512; i += blockDim.x) tab[i] = make_double2(1.0 + i * 1e-9, 1e-9 * i);
    __syncthreads();
    double x[CHAINS], e[CHAINS], f[CHAINS];
    unsigned u[CHAINS];
    float g[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
        x[c] = threadIdx.x * 1e-9 + c;
        e[c] = a + c * 1e-12;
        f[c] = b + c * 1e-13;
        u[c] = seed * (threadIdx.x + 1) + c * 2654435761u;
        g[c] = (float)c;
    }
    double acc = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
            if (MODE == DISTINCT) x[c] = fma(x[c], e[c], f[c]);
            else if (MODE == MIXOPS) {
                x[c] = (c % 3 == 0) ? fma(x[c], a, b) : ((c % 3 == 1) ? x[c] + b : x[c] * a);
            } else x[c] = fma(x[c], a, b);
            if (MODE == ALU1 || MODE == ALU2 || MODE == KNEARMIX) u[c] = (u[c] ^ seed) + 0x9E3779B9u;       // LOP3 + IADD
            if (MODE == ALU2) u[c] = (u[c] >> 3) | (u[c] << 7);
            if (MODE == IMAD1 || MODE == IMAD2) u[c] = u[c] * seed + 12345u;
            if (MODE == IMAD2) u[c] = u[c] * 3u + seed;
            if (MODE == FSEL2) {
                g[c] = (u[c] & 1) ? g[c] : (float)x[c & 1];
                u[c] += 1;
            }
            if (MODE == LDS1) acc += tab[(i + c) & 511].x;
            if (MODE == LDSR || (MODE == KNEARMIX && (c & 3) == 0)) {
                u[c] = u[c] * 1664525u + 1013904223u;
                const double2 t = tab[(u[c] >> 12) & 511];
                acc += t.x;
            }
            if ((MODE == MUFU8 && c == 0) || (MODE == KNEARMIX && c == 1)) {
                double r;
                asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(e[c]));
                e[c] = r + 1.0;
            }
        }
    }
    double s = acc;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += x[c] + e[c] + (double)u[c] + (double)g[c];
    if (s == 12345.678) out[0] = s;
}

template <int MODE>
static double run(double* out, int sms, double peak_tf)
{
    const int threads = 128, blocks = sms * 8, iters = 1 << 14;
    k_mix<MODE><<<blocks, threads>>>(out, 256, 0.999999, 1e-7, 12345u);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        k_mix<MODE><<<blocks, threads>>>(out, iters, 0.999999, 1e-7, 12345u + r);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double tf = 2.0 * CHAINS * (double)iters * threads * blocks / (ms * 1e-3) / 1e12;
        if (tf > best) best = tf;
    }
    return best / peak_tf;
}

int main()
{
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double* out;
    cudaMalloc(&out, 8);
    const double peak = sms * 64.0 * 2.0 * clk * 1e3 / 1e12;
    double fr[NMODES];
    fr[PURE] = run<PURE>(out, sms, peak);
    fr[DISTINCT] = run<DISTINCT>(out, sms, peak);
    fr[ALU1] = run<ALU1>(out, sms, peak);
    fr[ALU2] = run<ALU2>(out, sms, peak);
    fr[IMAD1] = run<IMAD1>(out, sms, peak);
    fr[IMAD2] = run<IMAD2>(out, sms, peak);
    fr[FSEL2] = run<FSEL2>(out, sms, peak);
    fr[LDS1] = run<LDS1>(out, sms, peak);
    fr[LDSR] = run<LDSR>(out, sms, peak);
    fr[MUFU8] = run<MUFU8>(out, sms, peak);
    fr[MIXOPS] = run<MIXOPS>(out, sms, peak);
    fr[KNEARMIX] = run<KNEARMIX>(out, sms, peak);
    cudaError_t e = cudaGetLastError();
    printf("{\"nominal_fp64_tflops\": %.2f, \"occupancy\": \"8 blocks x 128 threads per SM, %d independent chains per thread\", "
           "\"fp64_rate_fraction_of_nominal\": {", peak, CHAINS);
    for (int m = 0; m < NMODES; ++m) printf("\"%s\": %.3f%s", kNames[m], fr[m], m + 1 < NMODES ? ", " : "");
    printf("}, \"cuda\": \"%s\"}\n", cudaGetErrorString(e));
    return e != cudaSuccess;
}
