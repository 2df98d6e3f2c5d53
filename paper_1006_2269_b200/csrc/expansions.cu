// expansions.cu -- A4-A8: P2M, M2M, M2L and L2L as sm_100a FP64 kernels.
//
// Paper: "In the downward/upward phases the expansions are shifted as usual
// according to parent/child relations.  The critical far-to-local shift follows
// the weak connectivity pattern", in "the classical complex
// polynomial/multipole representation".  Forms:
//   P2M  a_0 = sum m_j,  a_k = -sum m_j (z_j - c)^k / k
//   M2M  b_l = -a_0 z0^l / l + sum_{k=1..l} a_k z0^{l-k} C(l-1,k-1),  z0 = c - c'
//   M2L  b_0 = a_0 Log(c_t - c_s) + sum_k (-1)^k a_k z0^-k
//        b_l = z0^-l ( sum_k C(l+k-1,k-1) (-1)^k a_k z0^-k  -  a_0 / l ),  z0 = c_s - c_t
//   L2L  d_k = sum_{l>=k} b_l C(l,k) h^{l-k},  h = c' - c  (Horner/Taylor shift)
// M2L is organised as the paper's "constant transition matrices with pre- and
// post-scaling according to the local geometry": pre-scale
// alpha_k = a_k (-1/z0)^k, apply the constant (p+1) x p matrix C(l+k-1,k-1)
// (held in __constant__ memory, a warp-uniform operand of every DFMA), post-scale
// by z0^-l -- fused per pair in registers (no HBM staging: 2.25 flop/B would be
// below the machine balance).  Every kernel is templated on p so the coefficient
// vectors live in registers.
#include <mutex>
#include "fmm2d_internal.cuh"

namespace fmm2d {

// M2L transition matrix C(l+k-1, k-1), l = 0..p, k = 1..p, at [l * M2L_CS + k - 1 + M2L_KOFF]
// (the layout changes which uniform constant loads the compiler emits: measured per layout)
#ifndef FMM2D_M2L_CS
#define FMM2D_M2L_CS 33
#endif
#ifndef FMM2D_M2L_KOFF
#define FMM2D_M2L_KOFF 1
#endif
constexpr int M2L_CS = FMM2D_M2L_CS, M2L_KOFF = FMM2D_M2L_KOFF;
#ifndef FMM2D_M2L_CT
#define FMM2D_M2L_CT 0            // 1: the matrix transposed, C(l+k-1, k-1) at [(k-1) M2L_CS + l + M2L_KOFF]
#endif
// index of C(l+k-1, k-1)
__host__ __device__ constexpr int m2l_ci(int l, int k)
{
    return FMM2D_M2L_CT ? (k - 1) * M2L_CS + l + M2L_KOFF : l * M2L_CS + k - 1 + M2L_KOFF;
}
static_assert(M2L_CS + M2L_KOFF >= FMM2D_PMAX + 1, "row stride of the M2L matrix");
__constant__ double c_m2l[(FMM2D_PMAX + 1) * M2L_CS + M2L_KOFF];

__constant__ double c_pas[(FMM2D_PMAX + 1) * (FMM2D_PMAX + 1)];   // [a][b] = C(a, b)

// exact binomials in 64-bit integers (C(63,31) < 2^64), correctly rounded to double
static uint64_t binom_u64(int a, int b)
{
    if (b < 0 || b > a) return 0;
    if (b > a - b) b = a - b;
    unsigned __int128 v = 1;
    for (int i = 1; i <= b; ++i) v = v * (unsigned __int128)(a - b + i) / (unsigned __int128)i;
    return (uint64_t)v;
}

int upload_binomials(int p)
{
    static bool uploaded[64] = {false};           // per device (__constant__ data is per device)
    static std::mutex mu;
    int dev = 0;
    FMM2D_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (dev >= 0 && dev < 64 && uploaded[dev]) return 0;
    (void)p;
    const int S = FMM2D_PMAX + 1;
    std::vector<double> m2l(S * M2L_CS + M2L_KOFF, 0.0), pas(S * S, 0.0);
    for (int l = 0; l <= FMM2D_PMAX; ++l)
        for (int k = 1; k <= FMM2D_PMAX; ++k)
            m2l[m2l_ci(l, k)] = (double)binom_u64(l + k - 1, k - 1);
    for (int a = 0; a <= FMM2D_PMAX; ++a)
        for (int b = 0; b <= a; ++b) pas[a * S + b] = (double)binom_u64(a, b);
    FMM2D_CUDA_TRY(cudaMemcpyToSymbol(c_m2l, m2l.data(), sizeof(double) * m2l.size()));

    FMM2D_CUDA_TRY(cudaMemcpyToSymbol(c_pas, pas.data(), sizeof(double) * S * S));
    if (dev >= 0 && dev < 64) uploaded[dev] = true;
    return 0;
}

namespace {

constexpr int S1 = FMM2D_PMAX + 1;

__device__ __forceinline__ double2 cmul(double2 a, double2 b)
{
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }

// children per block of k_m2m / k_l2l (their expansions staged in shared memory, <= 48 KB)
#ifndef FMM2D_L2L_BLOCK
#define FMM2D_L2L_BLOCK 128
#endif
template <int P>
__host__ __device__ constexpr int l2l_block() { return (P + 2) * 16 * FMM2D_L2L_BLOCK <= 48 * 1024 ? FMM2D_L2L_BLOCK : 64; }

// ---------------------------------------------------------------- P2M (A4)
template <int P>
// m != nullptr: the strengths are gathered here (m[perm[j]], input order) and written into
// the rows' (z, w) halves for the near field -- the rows' sectors are in cache from the
// coordinate read, so the 16-byte writes merge there
__global__ void __launch_bounds__(128) k_p2m(int64_t b0, int64_t b1, const uint32_t* __restrict__ off,
                                             double4* __restrict__ src, const double* __restrict__ cx,
                                             const double* __restrict__ cy, double2* __restrict__ mp,
                                             const double2* __restrict__ mg, const uint32_t* __restrict__ perm)
{
    int64_t b = b0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= b1) return;
    double2 a[P + 1];
#pragma unroll
    for (int k = 0; k <= P; ++k) a[k] = make_double2(0.0, 0.0);
    const double c0 = cx[b], c1 = cy[b];
    for (uint32_t j = off[b]; j < off[b + 1]; ++j) {
        double4 s = src[j];
        double2 w = make_double2(s.x - c0, s.y - c1);
        double2 m = make_double2(s.z, s.w);
        if (mg) {
            m = mg[perm[j]];
            reinterpret_cast<double2*>(src + j)[1] = m;
        }
        a[0] = cadd(a[0], m);
        double2 wk = m;                                 // m w^k, k = 1..P
#pragma unroll
        for (int k = 1; k <= P; ++k) {
            wk = cmul(wk, w);
            a[k] = csub(a[k], cscale(wk, 1.0 / k));
        }
    }
    double2* out = mp + b * (P + 1);
#pragma unroll
    for (int k = 0; k <= P; ++k) out[k] = a[k];
}

// ---------------------------------------------------------------- M2M (A5)
template <int P>
__global__ void __launch_bounds__(128) k_m2m(int64_t b0, int64_t b1, const double* __restrict__ cxp,
                                             const double* __restrict__ cyp, const double* __restrict__ cxc,
                                             const double* __restrict__ cyc, const double2* __restrict__ mc,
                                             double2* __restrict__ mpar)
{
    // one thread per CHILD (32 parents per block): the children's multipoles in and the
    // parents' out through shared memory with coalesced accesses; the four shifted children
    // are added by the parent's lane in child order 0, 1, 2, 3 (the sequential order)
    constexpr int W = P + 2, NB = l2l_block<P>();
    __shared__ double2 sm[NB * W];
    const int64_t cb = 4 * b0 + (int64_t)blockIdx.x * NB;               // first child of the block
    const int nc = (int)min((int64_t)NB, 4 * b1 - cb);
    const double2* g = mc + cb * (P + 1);
    for (int e = threadIdx.x; e < nc * (P + 1); e += NB) {
        const int i = e / (P + 1), k = e - i * (P + 1);
        sm[i * W + k] = g[e];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, q = threadIdx.x & 3;
    const int64_t c = cb + threadIdx.x, b = c >> 2;
    const bool act = threadIdx.x < nc;
    double2 t[P + 1];
#pragma unroll
    for (int k = 0; k <= P; ++k) t[k] = make_double2(0.0, 0.0);
    if (act) {
        const double2* a = sm + threadIdx.x * W;
        const double2 z0 = make_double2(cxc[c] - cxp[b], cyc[c] - cyp[b]);
        const double2 a0 = a[0];
        t[0] = a0;
        double2 zl = make_double2(1.0, 0.0);
#pragma unroll
        for (int l = 1; l <= P; ++l) {
            zl = cmul(zl, z0);                          // z0^l
            // Horner in z0: sum_{k=1..l} C(l-1,k-1) a_k z0^{l-k}
            double2 u = cscale(a[1], c_pas[(l - 1) * S1 + 0]);
#pragma unroll
            for (int k = 2; k <= l; ++k) u = cadd(cmul(u, z0), cscale(a[k], c_pas[(l - 1) * S1 + (k - 1)]));
            t[l] = csub(u, cscale(cmul(a0, zl), 1.0 / l));
        }
    }
    __syncthreads();                                 // children consumed: sm reused for parents
    const int base = lane & ~3;
#pragma unroll
    for (int k = 0; k <= P; ++k) {
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const double x = __shfl_sync(0xffffffffu, t[k].x, base + j);
            const double y = __shfl_sync(0xffffffffu, t[k].y, base + j);
            acc = cadd(acc, make_double2(x, y));
        }
        if (q == 0 && act) sm[(threadIdx.x >> 2) * W + k] = acc;
    }
    __syncthreads();
    const int np = (nc + 3) >> 2;
    double2* o = mpar + (cb >> 2) * (P + 1);
    for (int e = threadIdx.x; e < np * (P + 1); e += NB) {
        const int i = e / (P + 1), k = e - i * (P + 1);
        o[e] = sm[i * W + k];
    }
}

// ---------------------------------------------------------------- M2L (A6/A7)
// compile-time options of the M2L pair body (defaults: measured best at C5)
#ifndef FMM2D_M2L_LOGSPLIT
#define FMM2D_M2L_LOGSPLIT 0       // 1: the a_0 Log term of coefficient 0 in its own kernel (rr.cu: k_m2l_log) -- measured: k_m2l without the term compiles to 242 registers, no spills, and runs 31 ms instead of 15.8
#endif
#ifndef FMM2D_M2L_RCP
#define FMM2D_M2L_RCP 1            // 1 / r2 by MUFU + one cubic Newton step (C5 M2L 16.53 -> 15.84 ms)
#endif
#ifndef FMM2D_M2L_POW2
#define FMM2D_M2L_POW2 0          // bit 0: pre-scale powers by doubling, bit 1: post-scale powers
#endif
#ifndef FMM2D_M2L_LB
#define FMM2D_M2L_LB 18           // 0: one output coefficient at a time; 18: C5 M2L 19.26 -> 17.40 ms
#endif
#ifndef FMM2D_M2L_PREFETCH
#define FMM2D_M2L_PREFETCH 1   // next entry's box index loaded one pair ahead (M2L 19.26 -> 19.02 ms at C5)
#endif
// (struct M2LArgs: fmm2d_internal.cuh -- shared with the log-term kernel in rr.cu)

// One weak pair: the multipole M of source box s (global id, for its centre) into
// coefficients l in [L0, L1) of the local about (ctx, cty), accumulated into acc.
// LOGT = false leaves out the a_0 Log(c_t - c_s) term of coefficient 0 (k_m2l_log adds it).
template <int P, int L0, int L1, bool LOGT = true>
__device__ __forceinline__ void m2l_pair(const M2LArgs& A, int64_t s, const double2* __restrict__ M, double ctx,
                                         double cty, double2 (&acc)[L1 - L0])
{
    const double csx = A.cx[s], csy = A.cy[s];
    // z0 = c_s - c_t and 1/z0
    const double dx = csx - ctx, dy = csy - cty;
    const double r2 = dx * dx + dy * dy;
#if FMM2D_M2L_RCP
    // 1 / r2 by the reciprocal estimate and one cubic Newton step (~1 ulp) instead of the IEEE
    // division's longer dependent chain: everything in the pair waits for it
    double ir2;
    {
        double r0;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r0) : "d"(r2));
        const double e = fma(-r2, r0, 1.0);
        ir2 = fma(r0, fma(e, e, e), r0);
    }
#else
    const double ir2 = 1.0 / r2;
#endif
    const double2 iz = make_double2(dx * ir2, -dy * ir2);
    const double2 w = make_double2(-iz.x, -iz.y);
    // pre-scale: alpha_k = a_k (-1/z0)^k
    double2 al[P + 1];
#if FMM2D_M2L_POW2 & 1
    {   // powers by doubling: w^k = w^h w^(k-h), h the largest power of two below k -- a
        // dependent chain of <= 5 complex products instead of P - 1 (the FP64 pipe's
        // dependent-issue latency is ~28 cycles)
        double2 pw[P + 1];
        pw[1] = w;
#pragma unroll
        for (int k = 2; k <= P; ++k) {
            int h = 1;
            while (2 * h < k) h *= 2;
            pw[k] = cmul(pw[h], pw[k - h]);
        }
#pragma unroll
        for (int k = 1; k <= P; ++k) al[k] = cmul(M[k], pw[k]);
    }
#else
    double2 wk = w;
#pragma unroll
    for (int k = 1; k <= P; ++k) {
        al[k] = cmul(M[k], wk);
        if (k < P) wk = cmul(wk, w);
    }
#endif
    const double2 a0 = M[0];
#if FMM2D_M2L_LB > 0
    // The contraction in blocks of FMM2D_M2L_LB output coefficients, k outermost inside a block:
    // 2 LB independent FMA chains, so consecutive FMAs of one chain are 2 LB instructions apart
    // (the shared FP64 pipe's dependent-issue latency is ~28 cycles).
    double2 beta[L1 - L0];
#pragma unroll
    for (int lb = L0; lb < L1; lb += FMM2D_M2L_LB) {
#pragma unroll
        for (int l = lb; l < lb + FMM2D_M2L_LB && l < L1; ++l) beta[l - L0] = make_double2(0.0, 0.0);
#pragma unroll
        for (int k = 1; k <= P; ++k) {
#pragma unroll
            for (int l = lb; l < lb + FMM2D_M2L_LB && l < L1; ++l) {
                const double c = c_m2l[m2l_ci(l, k)];
                beta[l - L0].x = fma(c, al[k].x, beta[l - L0].x);
                beta[l - L0].y = fma(c, al[k].y, beta[l - L0].y);
            }
        }
    }
#endif
#if FMM2D_M2L_POW2 & 2
    double2 ipw[L1 > 2 ? L1 : 2];
    ipw[0] = make_double2(1.0, 0.0);
    ipw[1] = iz;
#pragma unroll
    for (int l = 2; l < L1; ++l) {
        int h = 1;
        while (2 * h < l) h *= 2;
        ipw[l] = cmul(ipw[h], ipw[l - h]);
    }
#endif
    double2 izl = make_double2(1.0, 0.0);
#pragma unroll
    for (int l = 0; l < L1; ++l) {
#if FMM2D_M2L_POW2 & 2
        izl = ipw[l];
#else
        if (l >= 1) izl = cmul(izl, iz);            // z0^-l
#endif
        if (l < L0) continue;
#if FMM2D_M2L_LB > 0
        const double2 bl = beta[l - L0];
#else
        double2 bl = make_double2(0.0, 0.0);
#pragma unroll
        for (int k = 1; k <= P; ++k) {
            const double c = c_m2l[m2l_ci(l, k)];
            bl.x = fma(c, al[k].x, bl.x);
            bl.y = fma(c, al[k].y, bl.y);
        }
#endif
        double2 v;
        if (l == 0) {
            if (LOGT) {
                // a_0 Log(c_t - c_s), componentwise difference (DESIGN R2)
                const double tx = ctx - csx, ty = cty - csy;
                const double2 lg = make_double2(0.5 * log(r2), atan2(ty, tx));
                v = cadd(cmul(a0, lg), bl);
            } else {
                v = bl;
            }
        } else {
            const double2 t = csub(bl, cscale(a0, 1.0 / l));
            v = cmul(t, izl);
        }
        acc[l - L0] = cadd(acc[l - L0], v);
    }
}

// Output coefficients l in [L0, L1) of target box g (level lev, level-local b), summed
// over the entries j = ja, ja + js, ... < jb of its weak list followed by its cross-level
// (parent merge) list.
template <int P, int L0, int L1, bool LOGT = true>
__device__ __forceinline__ void m2l_accum(const M2LArgs& A, int64_t g, int lev, int64_t b, int64_t ja, int64_t js,
                                          double2 (&acc)[L1 - L0])
{
    const int64_t w0 = A.woff[lev][b], nw = A.woff[lev][b + 1] - w0;
    const int64_t x0 = A.xoff[lev] ? A.xoff[lev][b] : 0;
    const int64_t jb = nw + (A.xoff[lev] ? A.xoff[lev][b + 1] - x0 : 0);
    const uint32_t* __restrict__ widx = A.widx[lev];
    const uint32_t* __restrict__ xidx = A.xidx[lev];
    const int64_t wbase = A.base[lev], xbase = lev > 0 ? A.base[lev - 1] : 0;
    const double ctx = A.cx[g], cty = A.cy[g];
#if FMM2D_M2L_PREFETCH
    // the NEXT entry's box index is loaded one pair ahead, so a pair's centre and multipole
    // loads (which depend on it) start at once instead of behind the index load's latency
    auto entry = [&](int64_t j) -> uint32_t {
        return (j >= nw) ? xidx[x0 + (j - nw)] : widx[w0 + j];
    };
    uint32_t bnext = (ja < jb) ? entry(ja) : 0u;
#endif
    for (int64_t j = ja; j < jb; j += js) {
        const bool cross = j >= nw;
        const int sl = cross ? lev - 1 : lev;                       // the source's level
#if FMM2D_M2L_PREFETCH
        const uint32_t bs = bnext;
        if (j + js < jb) bnext = entry(j + js);
#else
        const uint32_t bs = cross ? xidx[x0 + (j - nw)] : widx[w0 + j];
#endif
        const int64_t s = (cross ? xbase : wbase) + bs;
        // stored multipole (own / replicated box), or an imported one (sharded plans' halo)
        const double2* M = (bs >= A.slo[sl] && bs < A.shi[sl]) ? A.mpl[sl] + (int64_t)bs * (P + 1)
                                                              : A.mhalo + (int64_t)A.hmap[s] * (P + 1);
        m2l_pair<P, L0, L1, LOGT>(A, s, M, ctx, cty, acc);
    }
}

// One thread computes output coefficients l in [L0, L1) of one target box.
template <int P, int L0, int L1, bool LOGT = true>
__device__ __forceinline__ void m2l_target(const M2LArgs& A, int64_t g, int lev)
{
    const int64_t b = g - A.base[lev];
    double2 acc[L1 - L0];
#pragma unroll
    for (int l = 0; l < L1 - L0; ++l) acc[l] = make_double2(0.0, 0.0);
    m2l_accum<P, L0, L1, LOGT>(A, g, lev, b, 0, 1, acc);
    double2* out = A.lcl[lev] + b * (P + 1);
#pragma unroll
    for (int l = L0; l < L1; ++l) out[l] = acc[l - L0];
}

// Long weak lists (non-uniform inputs): one warp per target, lanes over the pairs, a
// fixed-order shuffle reduction -- so one box's list no longer serialises on one thread.
template <int P, int L0, int L1>
__device__ __forceinline__ void m2l_target_warp(const M2LArgs& A, int64_t g, int lev, int lane)
{
    const int64_t b = g - A.base[lev];
    double2 acc[L1 - L0];
#pragma unroll
    for (int l = 0; l < L1 - L0; ++l) acc[l] = make_double2(0.0, 0.0);
    m2l_accum<P, L0, L1>(A, g, lev, b, lane, 32, acc);
#pragma unroll
    for (int l = 0; l < L1 - L0; ++l) {
        for (int o = 16; o; o >>= 1) {
            acc[l].x += __shfl_xor_sync(0xffffffffu, acc[l].x, o);
            acc[l].y += __shfl_xor_sync(0xffffffffu, acc[l].y, o);
        }
    }
    if (lane == 0) {
        double2* out = A.lcl[lev] + b * (P + 1);
#pragma unroll
        for (int l = L0; l < L1; ++l) out[l] = acc[l - L0];
    }
}

#ifndef FMM2D_M2L_MINB
#define FMM2D_M2L_MINB 1
#endif
#ifndef FMM2D_M2L_T
#define FMM2D_M2L_T 256              // one block of 8 warps per SM (255 registers): C5 M2L 15.84 -> 15.25 ms (128 x 2 blocks: 15.84, 64 x 4: 15.74)
#endif
constexpr int M2L_T = FMM2D_M2L_T;
constexpr int M2L_LONG_T = 128;     // k_m2l_long (warp per long-list target): 2 blocks of 128 (C4: 6.7 ms vs 7.4 at 256)

// threads: NS consecutive warps share 32 target boxes; warp-uniform part index.
// (Tried and measured slower at p = 17 on B200: accumulators in shared memory, and a
// k-outer contraction with beta in registers.)
template <int P, int NS>
__global__ void __launch_bounds__(M2L_T, FMM2D_M2L_MINB) k_m2l(M2LArgs A)
{
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int lane = threadIdx.x & 31;
    int64_t warp = t >> 5;
    int part = (int)(warp % NS);
    int64_t w = (warp / NS) * 32 + lane;         // work item: one target box
    if (w >= A.pre[A.L + 1]) return;
    int lev = 1;
    while (lev < A.L && w >= A.pre[lev + 1]) ++lev;
    const int64_t g = A.base[lev] + A.order[w];
    {   // long lists are done by k_m2l_long
        const int64_t b = g - A.base[lev];
        const int64_t len = A.woff[lev][b + 1] - A.woff[lev][b] + (A.xoff[lev] ? A.xoff[lev][b + 1] - A.xoff[lev][b] : 0);
        if (len > FMM2D_M2L_LONG) return;
    }
    // part q computes coefficients [q H, min((q+1) H, P+1)), H = ceil((P+1)/NS)
    constexpr int H = (P + NS) / NS;
    constexpr int E1 = (2 * H < P + 1) ? 2 * H : P + 1;
    constexpr int E2 = (3 * H < P + 1) ? 3 * H : P + 1;
    if constexpr (NS == 1) {
        m2l_target<P, 0, P + 1, !FMM2D_M2L_LOGSPLIT>(A, g, lev);     // (k_m2l_log adds the log terms)
    } else if constexpr (NS == 2) {
        if (part == 0) m2l_target<P, 0, H>(A, g, lev);
        else           m2l_target<P, H, P + 1>(A, g, lev);
    } else {
        static_assert(NS == 3, "M2L split into 1..3 parts");
        if (part == 0)      m2l_target<P, 0, H>(A, g, lev);
        else if (part == 1) m2l_target<P, H, E1>(A, g, lev);
        else                m2l_target<P, E1, E2>(A, g, lev);
    }
}

// The same work as k_m2l from a CAPPED grid of single-warp blocks, grid-stride over the warp
// rounds: used when the expansions run concurrently with the near field (FMM2D_OVERLAP), so
// that M2L keeps only a few warps per SM and the P2P CTAs fill the rest of each SM.
template <int P, int NS>
__global__ void __launch_bounds__(32, 1) k_m2l_gs(M2LArgs A, int64_t nwarps)
{
    const int lane = threadIdx.x & 31;
    constexpr int H = (P + NS) / NS;
    constexpr int E1 = (2 * H < P + 1) ? 2 * H : P + 1;
    constexpr int E2 = (3 * H < P + 1) ? 3 * H : P + 1;
    for (int64_t warp = blockIdx.x; warp < nwarps; warp += gridDim.x) {
        const int part = (int)(warp % NS);
        const int64_t w = (warp / NS) * 32 + lane;
        if (w >= A.pre[A.L + 1]) continue;
        int lev = 1;
        while (lev < A.L && w >= A.pre[lev + 1]) ++lev;
        const int64_t g = A.base[lev] + A.order[w];
        const int64_t b = g - A.base[lev];
        const int64_t len = A.woff[lev][b + 1] - A.woff[lev][b] + (A.xoff[lev] ? A.xoff[lev][b + 1] - A.xoff[lev][b] : 0);
        if (len > FMM2D_M2L_LONG) continue;
        if constexpr (NS == 1) {
            m2l_target<P, 0, P + 1>(A, g, lev);
        } else if constexpr (NS == 2) {
            if (part == 0) m2l_target<P, 0, H>(A, g, lev);
            else           m2l_target<P, H, P + 1>(A, g, lev);
        } else {
            if (part == 0)      m2l_target<P, 0, H>(A, g, lev);
            else if (part == 1) m2l_target<P, H, E1>(A, g, lev);
            else                m2l_target<P, E1, E2>(A, g, lev);
        }
    }
}

// one warp (per coefficient part) per long-list target; long[] holds global box ids
template <int P, int NS>
__global__ void __launch_bounds__(M2L_LONG_T, 2) k_m2l_long(M2LArgs A, const uint32_t* __restrict__ longs,
                                                                   int64_t nlong)
{
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int part = (int)(warp % NS);
    const int64_t w = warp / NS;
    if (w >= nlong) return;
    const int64_t g = longs[w];
    int lev = 1;
    while (lev < A.L && g >= A.base[lev + 1]) ++lev;
    constexpr int H = (P + NS) / NS;
    constexpr int E1 = (2 * H < P + 1) ? 2 * H : P + 1;
    constexpr int E2 = (3 * H < P + 1) ? 3 * H : P + 1;
    if constexpr (NS == 1) {
        m2l_target_warp<P, 0, P + 1>(A, g, lev, lane);
    } else if constexpr (NS == 2) {
        if (part == 0) m2l_target_warp<P, 0, H>(A, g, lev, lane);
        else           m2l_target_warp<P, H, P + 1>(A, g, lev, lane);
    } else {
        if (part == 0)      m2l_target_warp<P, 0, H>(A, g, lev, lane);
        else if (part == 1) m2l_target_warp<P, H, E1>(A, g, lev, lane);
        else                m2l_target_warp<P, E1, E2>(A, g, lev, lane);
    }
}

// ---------------------------------------------------------------- L2L (A8)
template <int P>
__global__ void __launch_bounds__(128) k_l2l(int64_t c0, int64_t c1, const double* __restrict__ cxp,
                                             const double* __restrict__ cyp, const double* __restrict__ cxc,
                                             const double* __restrict__ cyc, const double2* __restrict__ lpar,
                                             double2* __restrict__ lch)
{
    // the block's children's locals (contiguous) move through shared memory with coalesced
    // 16-byte accesses; each thread's row is padded by one entry (bank spread)
    constexpr int W = P + 2, NB = l2l_block<P>();
    __shared__ double2 sl[NB * W];
    const int64_t cb = c0 + (int64_t)blockIdx.x * NB;
    const int nc = (int)min((int64_t)NB, c1 - cb);
    double2* g = lch + cb * (P + 1);
    for (int e = threadIdx.x; e < nc * (P + 1); e += NB) {
        const int i = e / (P + 1), k = e - i * (P + 1);
        sl[i * W + k] = g[e];
    }
    __syncthreads();
    const int64_t c = cb + threadIdx.x;
    if (threadIdx.x < nc) {
        const int64_t b = c >> 2;
        const double2* B = lpar + b * (P + 1);
        double2 d[P + 1];
#pragma unroll
        for (int k = 0; k <= P; ++k) d[k] = B[k];
        const double2 h = make_double2(cxc[c] - cxp[b], cyc[c] - cyp[b]);
        // Taylor shift: d_k = sum_{l>=k} b_l C(l,k) h^{l-k}
#pragma unroll
        for (int i = 0; i < P; ++i) {
#pragma unroll
            for (int j = P - 1; j >= i; --j) d[j] = cadd(d[j], cmul(h, d[j + 1]));
        }
        double2* out = sl + threadIdx.x * W;
#pragma unroll
        for (int k = 0; k <= P; ++k) out[k] = cadd(out[k], d[k]);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nc * (P + 1); e += NB) {
        const int i = e / (P + 1), k = e - i * (P + 1);
        g[e] = sl[i * W + k];
    }
}

inline unsigned grid_for(int64_t n, int bs) { return (unsigned)((n + bs - 1) / bs); }

// P2M of the own leaves, then M2M for parent levels L-1 .. lstop (own parents; the
// replicated levels above the partition level are done by upward_top_p)
template <int P>
int upward_p(fmm2d_plan* Pl)
{
    cudaStream_t st = Pl->stream;
    const int L = Pl->L;
    const int64_t l0 = Pl->box_lo(L), l1 = Pl->box_hi(L);
    k_p2m<P><<<grid_for(l1 - l0, 128), 128, 0, st>>>(l0, l1, Pl->boff + Pl->obase[L], Pl->src, Pl->cx + Pl->base[L],
                                                    Pl->cy + Pl->base[L], Pl->mpl[L],
                                                    Pl->m_fused, Pl->perm);
    Pl->m_fused = nullptr;
    fmm2d::note_launch();
    FMM2D_CUDA_TRY(cudaGetLastError());
    for (int l = L - 1; l >= Pl->kpart; --l) {
        const int64_t b0 = Pl->own_lo(l), b1 = Pl->own_hi(l);
        k_m2m<P><<<grid_for(4 * (b1 - b0), l2l_block<P>()), l2l_block<P>(), 0, st>>>(
            b0, b1, Pl->cx + Pl->base[l], Pl->cy + Pl->base[l], Pl->cx + Pl->base[l + 1], Pl->cy + Pl->base[l + 1],
            Pl->mpl[l + 1], Pl->mpl[l]); fmm2d::note_launch();
        FMM2D_CUDA_TRY(cudaGetLastError());
    }
    return 0;
}

// M2M of the replicated levels kpart-1 .. 0 (every box; after the level-kpart
// multipoles have been all-gathered)
template <int P>
int upward_top_p(fmm2d_plan* Pl)
{
    cudaStream_t st = Pl->stream;
    for (int l = Pl->kpart - 1; l >= 0; --l) {
        const int64_t nb = nboxes(l);
        k_m2m<P><<<grid_for(4 * nb, l2l_block<P>()), l2l_block<P>(), 0, st>>>(
            0, nb, Pl->cx + Pl->base[l], Pl->cy + Pl->base[l], Pl->cx + Pl->base[l + 1], Pl->cy + Pl->base[l + 1],
            Pl->mpl[l + 1], Pl->mpl[l]); fmm2d::note_launch();
        FMM2D_CUDA_TRY(cudaGetLastError());
    }
    return 0;
}

template <int P>
#ifndef FMM2D_M2L_SPLIT_P
#define FMM2D_M2L_SPLIT_P 20      // p above this: the output coefficients over 2-3 threads
#endif
constexpr int m2l_split() { return P <= FMM2D_M2L_SPLIT_P ? 1 : (P <= 26 ? 2 : 3); }

template <int P, int NS>
int m2l_long_p(fmm2d_plan* Pl, const M2LArgs& A)
{
    k_m2l_long<P, NS><<<grid_for(Pl->m2l_nlong * NS * 32, M2L_LONG_T), M2L_LONG_T, 0, Pl->stream>>>(A, Pl->m2l_long,
                                                                                        Pl->m2l_nlong);
    fmm2d::note_launch();
    FMM2D_CUDA_TRY(cudaGetLastError());
    return 0;
}

template <int P>
int m2l_p(fmm2d_plan* Pl)
{
    cudaStream_t st = Pl->stream;
    const int L = Pl->L;
    if (L < 1) {
        FMM2D_CUDA_TRY(cudaMemsetAsync(Pl->local, 0, sizeof(double2) * (P + 1), st));
        return 0;
    }
    M2LArgs A;
    for (int l = 0; l <= L; ++l) {
        A.woff[l] = Pl->weak[l].off;
        A.widx[l] = Pl->weak[l].idx;
        A.xoff[l] = Pl->xweak[l].off;
        A.xidx[l] = Pl->xweak[l].idx;
    }
    for (int l = 0; l <= L + 1; ++l) A.base[l] = Pl->base[l];
    A.pre[0] = A.pre[1] = 0;
    A.lo[0] = 0;
    for (int l = 1; l <= L; ++l) {
        A.lo[l] = Pl->box_lo(l);
        A.pre[l + 1] = A.pre[l] + (Pl->box_hi(l) - Pl->box_lo(l));
    }
    A.order = Pl->m2l_order;
    A.L = L;
    A.cx = Pl->cx;
    A.cy = Pl->cy;
    for (int l = 0; l <= L; ++l) {
        A.mpl[l] = Pl->mpl[l];
        A.lcl[l] = Pl->lcl[l];
        A.slo[l] = Pl->box_lo(l);
        A.shi[l] = Pl->box_hi(l);
    }
    A.mhalo = Pl->mhalo;
    A.hmap = Pl->hmap;
    // level-0 local is zero (no M2L at the root)
    FMM2D_CUDA_TRY(cudaMemsetAsync(Pl->local, 0, sizeof(double2) * (P + 1), st));
    constexpr int NS = m2l_split<P>();
    const int64_t work = A.pre[L + 1];
    int64_t nthreads = ((work + 31) / 32) * 32 * NS;
    if (Pl->m2l_cap > 0) {                      // concurrent with the near field: a capped grid
        const int64_t nwarps = nthreads / 32;
        k_m2l_gs<P, NS><<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(Pl->m2l_cap, nwarps)), 32, 0, st>>>(A, nwarps);
    } else {
        k_m2l<P, NS><<<grid_for(nthreads, M2L_T), M2L_T, 0, st>>>(A);
        fmm2d::note_launch();
        FMM2D_CUDA_TRY(cudaGetLastError());
        if (NS == 1 && FMM2D_M2L_LOGSPLIT) FMM2D_TRY(m2l_log_terms(Pl, A, P + 1));
        return Pl->m2l_nlong > 0 ? m2l_long_p<P, NS>(Pl, A) : 0;
    }
    fmm2d::note_launch();
    FMM2D_CUDA_TRY(cudaGetLastError());
    return Pl->m2l_nlong > 0 ? m2l_long_p<P, NS>(Pl, A) : 0;
}

template <int P>
int downward_p(fmm2d_plan* Pl)
{
    cudaStream_t st = Pl->stream;
    for (int l = 2; l <= Pl->L; ++l) {
        const int64_t c0 = Pl->box_lo(l), c1 = Pl->box_hi(l);
        k_l2l<P><<<grid_for(c1 - c0, l2l_block<P>()), l2l_block<P>(), 0, st>>>(
            c0, c1, Pl->cx + Pl->base[l - 1], Pl->cy + Pl->base[l - 1], Pl->cx + Pl->base[l], Pl->cy + Pl->base[l],
            Pl->lcl[l - 1], Pl->lcl[l]); fmm2d::note_launch();
        FMM2D_CUDA_TRY(cudaGetLastError());
    }
    return 0;
}

}  // namespace

#define FMM2D_P_CASES(F)                                                                      \
    case 1: return F<1>(P); case 2: return F<2>(P); case 3: return F<3>(P);                   \
    case 4: return F<4>(P); case 5: return F<5>(P); case 6: return F<6>(P);                   \
    case 7: return F<7>(P); case 8: return F<8>(P); case 9: return F<9>(P);                   \
    case 10: return F<10>(P); case 11: return F<11>(P); case 12: return F<12>(P);             \
    case 13: return F<13>(P); case 14: return F<14>(P); case 15: return F<15>(P);             \
    case 16: return F<16>(P); case 17: return F<17>(P); case 18: return F<18>(P);             \
    case 19: return F<19>(P); case 20: return F<20>(P); case 21: return F<21>(P);             \
    case 22: return F<22>(P); case 23: return F<23>(P); case 24: return F<24>(P);             \
    case 25: return F<25>(P); case 26: return F<26>(P); case 27: return F<27>(P);             \
    case 28: return F<28>(P); case 29: return F<29>(P); case 30: return F<30>(P);             \
    case 31: return F<31>(P); case 32: return F<32>(P);

int run_upward(fmm2d_plan* P)
{
    switch (P->p) { FMM2D_P_CASES(upward_p) default: return FMM2D_EINVAL; }
}

int run_upward_top(fmm2d_plan* P)
{
    switch (P->p) { FMM2D_P_CASES(upward_top_p) default: return FMM2D_EINVAL; }
}


int run_m2l(fmm2d_plan* P)
{
    switch (P->p) { FMM2D_P_CASES(m2l_p) default: return FMM2D_EINVAL; }
}

int run_downward(fmm2d_plan* P)
{
    switch (P->p) { FMM2D_P_CASES(downward_p) default: return FMM2D_EINVAL; }
}

}  // namespace fmm2d
