// p2p_census.cu -- the FP64 cost of ONE ordered P2P pair when written with the CUDA math
// library (libdevice: log, atan2, IEEE division), i.e. SURVEY 8(d)'s convention "count each
// transcendental at its libdevice FP64 instruction cost, measured once by ncu on a
// microbenchmark".  The pair body is Eq. 1's summand and its derivative:
//     dz = z_i - z_j;  Phi_i += m_j Log(dz) = m_j (0.5 log|dz|^2 + i atan2(dy, dx));
//     Phi'_i += m_j / dz = m_j conj(dz) / |dz|^2            (real m_j, the C5 workload)
// Sources and targets are drawn like one C5 leaf neighbourhood (|dz| ~ 1e-4 .. 1e-3).
// Run under ncu for the executed DFMA / DADD / DMUL counts (flop = 2 DFMA + DADD + DMUL per
// thread instruction), and alone for the pair rate of the library-math kernel:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o build/p2p_census tools/p2p_census.cu
//   ./build/p2p_census                       # timing (JSON)
//   ncu --metrics sm__sass_thread_inst_executed_op_dfma_pred_on.sum,... ./build/p2p_census 1
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int NS = 256;              // sources staged per CTA (one chunk of a near list)

__global__ void k_pair_libdevice(const double4* __restrict__ src, const double2* __restrict__ tgt, int ns_total,
                                 double4* __restrict__ out)
{
    __shared__ double4 s[NS];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const double2 t = tgt[i];
    double f_re = 0, f_im = 0, d_re = 0, d_im = 0;
    for (int c = 0; c < ns_total; c += NS) {
        __syncthreads();
        for (int k = threadIdx.x; k < NS; k += blockDim.x) s[k] = src[(c + k) % ns_total];
        __syncthreads();
#pragma unroll 1
        for (int j = 0; j < NS; ++j) {
            const double4 q = s[j];
            const double dx = t.x - q.x, dy = t.y - q.y;
            const double r2 = dx * dx + dy * dy;
            const double lg = 0.5 * log(r2);              // Log|dz|
            const double ar = atan2(dy, dx);              // Arg dz
            const double inv = 1.0 / r2;                  // IEEE division
            f_re += q.z * lg;
            f_im += q.z * ar;
            d_re += q.z * dx * inv;
            d_im -= q.z * dy * inv;
        }
    }
    out[i] = make_double4(f_re, f_im, d_re, d_im);
}

int main(int argc, char** argv)
{
    const bool census = argc > 1;                          // one small launch for ncu
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int threads = 128;
    const int blocks = census ? sms : sms * 64;
    const int nt = threads * blocks;
    const int ns = census ? NS : 4 * NS;
    std::vector<double4> hs(ns);
    std::vector<double2> ht(nt);
    srand(12345);
    auto u = [] { return (double)rand() / RAND_MAX; };
    for (auto& q : hs) q = make_double4(1e-3 * u(), 1e-3 * u(), 2 * u() - 1, 0);
    for (auto& t : ht) t = make_double2(1e-3 * u() + 1e-7, 1e-3 * u() + 3e-7);
    double4 *ds, *dout;
    double2* dt;
    cudaMalloc(&ds, sizeof(double4) * ns);
    cudaMalloc(&dt, sizeof(double2) * nt);
    cudaMalloc(&dout, sizeof(double4) * nt);
    cudaMemcpy(ds, hs.data(), sizeof(double4) * ns, cudaMemcpyHostToDevice);
    cudaMemcpy(dt, ht.data(), sizeof(double2) * nt, cudaMemcpyHostToDevice);
    k_pair_libdevice<<<blocks, threads>>>(ds, dt, ns, dout);
    if (census) {
        cudaDeviceSynchronize();
        printf("{\"pairs\": %.0f}\n", (double)nt * ns);
        return cudaGetLastError() != cudaSuccess;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_pair_libdevice<<<blocks, threads>>>(ds, dt, ns, dout);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double pairs = (double)nt * ns;
    printf("{\"kernel\": \"k_pair_libdevice\", \"pairs_per_launch\": %.0f, \"ms\": %.4f, \"pairs_per_s\": %.4e, "
           "\"cuda\": \"%s\"}\n", pairs, best, pairs / (best * 1e-3), cudaGetErrorString(cudaGetLastError()));
    return 0;
}
