// near.cu -- A9-A11: L2P + P2P over the strong leaf lists, written back in input order.
//
// Paper: "at the finest level, the remaining strong connections are evaluated
// directly"; the pairwise term is m_j log(z_i - z_j) of Eq. 1
// with j != i by index; the result is returned in input order.
//
// GPU formulation: one CTA of 128 threads per target leaf t.
// The sources of t's strong list are staged through shared memory in chunks of up
// to NEAR_CHUNK 32-byte rows {x, y, Re m, Im m} (whole leaves, at most 32 per chunk;
// warp 0 scans the leaf sizes, all four warps copy).  Each thread owns TWO targets
// (register blocking: every source row loaded from shared memory feeds two pairs)
// and one of G source groups; group g walks chunk rows g, g+G, ...  Rows of t's own
// leaf are walked in a separate short range where the self pair j == i is neutralised
// (dz := 1, m := 0), so the main loop carries no per-pair test.  Log(dz) and 1/dz use
// the table-driven FP64 routines of fastmath.cuh (tables in shared memory).  The G
// partial sums per target are reduced in shared memory in fixed group order
// (deterministic), the L2P Horner evaluation of t's local expansion is added, and the
// result is stored at the input position perm[i].
// Leaves larger than NEAR_CHUNK (only when nlevels forces a shallow tree) take
// k_near_wide, which reads sources straight from global memory.
#include <cstdlib>
#include <mutex>
#include <cub/cub.cuh>

#include "fastmath.cuh"
#include "fmm2d_internal.cuh"

namespace fmm2d {

namespace {

constexpr int NEAR_T = 128;
#ifndef FMM2D_NEAR_MINB
#define FMM2D_NEAR_MINB 8
#endif
#ifndef FMM2D_NEAR_SKIPBAR
#define FMM2D_NEAR_SKIPBAR 1      // no barrier before the first chunk of a pass
#endif
#ifndef FMM2D_NEAR_TMA_TABLES
#define FMM2D_NEAR_TMA_TABLES 1       // k_near: tables by one cp.async.bulk + mbarrier
#endif
#ifndef FMM2D_NEAR_TMA_ROWS
#define FMM2D_NEAR_TMA_ROWS 1         // k_near: the chunk's source rows by per-leaf cp.async.bulk
#endif
#ifndef FMM2D_NEAR_TPT
#define FMM2D_NEAR_TPT 2          // targets per thread (register blocking)
#endif
#ifndef FMM2D_NEAR_UNROLL
#define FMM2D_NEAR_UNROLL 1       // source rows per unrolled iteration (1: measured best at C5)
#endif
constexpr int NEAR_TPT = FMM2D_NEAR_TPT;
constexpr int NEAR_UNROLL = FMM2D_NEAR_UNROLL;
#ifndef FMM2D_NEAR_LOG5
#define FMM2D_NEAR_LOG5 1         // degree-5 log1p (absolute error < 2^-52: tests/test_fastmath.py)
#endif
constexpr int NEAR_CHUNK = FMM2D_NEAR_CHUNK;    // >= 256: the chunk buffer doubles as reduction space
static_assert(NEAR_CHUNK >= 2 * NEAR_T, "chunk buffer too small for the reduction");

// the strengths into the source rows' (z, w) halves (16-byte stores; the coordinates in
// (x, y) are not read); GM rows per thread with the random gathers of m in flight together
constexpr int GM = 4;
__global__ void __launch_bounds__(256) k_gather_m(const double2* __restrict__ m, const uint32_t* __restrict__ perm,
                                                  int64_t k0, int64_t k1, double4* __restrict__ src)
{
    const int64_t kb = k0 + (int64_t)blockIdx.x * (256 * GM) + threadIdx.x;
    uint32_t j[GM];
    double2 v[GM];
#pragma unroll
    for (int u = 0; u < GM; ++u) j[u] = (kb + u * 256 < k1) ? perm[kb + u * 256] : 0u;
#pragma unroll
    for (int u = 0; u < GM; ++u)
        if (kb + u * 256 < k1) v[u] = m[j[u]];
#pragma unroll
    for (int u = 0; u < GM; ++u)
        if (kb + u * 256 < k1) reinterpret_cast<double2*>(src + kb + u * 256)[1] = v[u];
}

// Sums of one target: A = sum m log|dz|^2, B = sum m Arg dz, D = sum m conj(dz)/|dz|^2,
// so that Phi = A/2 + i B and Phi' = D (the halving is done once, at the end).
struct PairAcc {
    double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0, dr = 0.0, di = 0.0;
    __device__ __forceinline__ double2 phi() const { return make_double2(0.5 * ar - bi, 0.5 * ai + br); }
    __device__ __forceinline__ double2 dphi() const { return make_double2(dr, di); }
};

// one ordered pair: Phi_i += m Log(dz), Phi'_i += m / dz  (REAL: Im m = 0)
// the lane's view of the near-field tables (fm::TablesN in shared memory): its copy of each
struct NearTab {
    const double2* lg;
    const double* th;
    const double2* oct;
    __device__ __forceinline__ NearTab(const fm::TablesN& N, int lane)
        : lg(N.lg + (lane & (fm::NRL - 1))), th(N.th + (lane & (fm::NRA - 1))), oct(N.oct) {}
};

template <bool REAL>
__device__ __forceinline__ void pair(PairAcc& a, double dx, double dy, double mr, double mi,
                                     const NearTab& T)
{
    const double r2 = fma(dx, dx, dy * dy);
    const double l2 = fm::log_pos5<fm::LRL>(r2, T.lg);                // log |dz|^2 (absolute error < 2^-52)
    const double th = fm::arg_n(dx, dy, T.th, T.oct);                 // Arg dz (absolute error < 2^-51)
    const double ir2 = fm::rcp(r2);
    const double mr2 = mr * ir2;
    a.ar = fma(mr, l2, a.ar);
    a.br = fma(mr, th, a.br);
    a.dr = fma(mr2, dx, a.dr);                                        // m conj(dz) / |dz|^2
    a.di = fma(-mr2, dy, a.di);
    if (!REAL) {
        const double mi2 = mi * ir2;
        a.ai = fma(mi, l2, a.ai);
        a.bi = fma(mi, th, a.bi);
        a.dr = fma(mi2, dy, a.dr);
        a.di = fma(mi2, dx, a.di);
    }
}

// the same with the general-purpose routines on fm::Tables (symmetric kernel's own leaf)
template <bool REAL>
__device__ __forceinline__ void pair_t(PairAcc& a, double dx, double dy, double mr, double mi, const fm::Tables& T)
{
    const double r2 = fma(dx, dx, dy * dy);
    const double l2 = fm::log_pos5(r2, T.lg);
    const double th = fm::arg_t(dx, dy, T.at);
    const double ir2 = fm::rcp(r2);
    const double mr2 = mr * ir2;
    a.ar = fma(mr, l2, a.ar);
    a.br = fma(mr, th, a.br);
    a.dr = fma(mr2, dx, a.dr);
    a.di = fma(-mr2, dy, a.di);
    if (!REAL) {
        const double mi2 = mi * ir2;
        a.ai = fma(mi, l2, a.ai);
        a.bi = fma(mi, th, a.bi);
        a.dr = fma(mi2, dy, a.dr);
        a.di = fma(mi2, dx, a.di);
    }
}

__device__ __forceinline__ double4 pack(const PairAcc& a)
{
    const double2 f = a.phi(), g = a.dphi();
    return make_double4(f.x, f.y, g.x, g.y);
}

// L2P (Horner): Phi = sum b_l w^l, Phi' = sum l b_l w^{l-1}, w = z_i - c
__device__ __forceinline__ void l2p(const double2* __restrict__ B, int p, double wx, double wy, double& fr,
                                    double& fi, double& gr, double& gi)
{
    fr = B[p].x;
    fi = B[p].y;
    gr = p * B[p].x;
    gi = p * B[p].y;
    for (int l = p - 1; l >= 0; --l) {
        const double2 b = B[l];
        double nr = fr * wx - fi * wy + b.x;
        double ni = fr * wy + fi * wx + b.y;
        fr = nr;
        fi = ni;
        if (l >= 1) {
            nr = gr * wx - gi * wy + l * b.x;
            ni = gr * wy + gi * wx + l * b.y;
            gr = nr;
            gi = ni;
        }
    }
}

template <class TT>
__device__ __forceinline__ void load_tables(TT& T, const TT* __restrict__ g)
{
    static_assert(sizeof(TT) % 16 == 0, "tables are copied in 16-byte pieces");
    const double2* gs = (const double2*)g;
    double2* ss = (double2*)&T;
    for (int k = threadIdx.x; k < (int)(sizeof(TT) / 16); k += blockDim.x) ss[k] = gs[k];
}

// first k >= b with k == g (mod G)
__device__ __forceinline__ int first_in_class(int b, int g, int G)
{
    int r = (g - b) % G;
    return b + (r < 0 ? r + G : r);
}

// Work items: blockIdx.x < nmain is target leaf t0 + blockIdx.x over its whole list
// (skipped if the leaf is split: seg_off[t+1] > seg_off[t]); the items after it are the
// segments of split leaves (long strong lists of non-uniform inputs), each over a part of
// the list, writing partial sums to part[] (k_near_combine finishes those leaves).
template <bool REAL>
__global__ void __launch_bounds__(NEAR_T, FMM2D_NEAR_MINB) k_near(int G, int p, int64_t t0, int64_t nmain,
                                                 const int64_t* __restrict__ seg_off, const NearSeg* __restrict__ segs,
                                                 double4* __restrict__ part, int part_w,
                                                 const uint32_t* __restrict__ off,
                                                 const int64_t* __restrict__ soff, const uint32_t* __restrict__ sidx,
                                                 const double4* __restrict__ src, const double* __restrict__ cx,
                                                 const double* __restrict__ cy, const double2* __restrict__ loc,
                                                 const uint32_t* __restrict__ perm, const fm::TablesN* __restrict__ gtab,
                                                 double2* __restrict__ phi, double2* __restrict__ dphi,
                                                 const int64_t* __restrict__ m2p_off, const double4* __restrict__ m2p_acc,
                                                 double4* __restrict__ nacc, const uint32_t* __restrict__ lmap,
                                                 const double4* __restrict__ hsrc)
{
    __shared__ double4 S[(NEAR_CHUNK > NEAR_TPT * NEAR_T) ? NEAR_CHUNK : NEAR_TPT * NEAR_T];
    __shared__ fm::TablesN T;
    double4(*red)[NEAR_T] = reinterpret_cast<double4(*)[NEAR_T]>(S);   // after the last chunk
    __shared__ int cstart[33];
    __shared__ int cinfo[2];                 // [0] leaves in chunk, [1] chunk row of leaf t (-1)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const NearTab NT(T, lane);
    int64_t t, q0, q1, segi = -1;
    if ((int64_t)blockIdx.x < nmain) {
        t = t0 + blockIdx.x;
        if (seg_off && seg_off[t + 1] > seg_off[t]) return;      // split leaf: segments + combine
        q0 = soff[t];
        q1 = soff[t + 1];
    } else {
        segi = (int64_t)blockIdx.x - nmain;
        const NearSeg sg = segs[segi];
        t = sg.t;
        q0 = sg.qa;
        q1 = sg.qb;
    }
#if FMM2D_NEAR_TMA_TABLES
    // the tables by ONE bulk asynchronous copy (TMA engine, completion on an mbarrier) instead
    // of a copy loop through every thread's registers; waited for just before the first pair
    __shared__ __align__(8) unsigned long long tbar;
    const uint32_t tbar_s = (uint32_t)__cvta_generic_to_shared(&tbar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tbar_s) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tbar_s),
                     "r"((uint32_t)sizeof(fm::TablesN)) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"((uint32_t)__cvta_generic_to_shared(&T)), "l"(gtab), "r"((uint32_t)sizeof(fm::TablesN)),
                     "r"(tbar_s) : "memory");
    }
    bool tables_ready = false;              // (the mbarrier's init is ordered by the chunk barriers)
#if FMM2D_NEAR_TMA_ROWS
    // the chunk's source rows: one bulk copy per leaf (its rows are contiguous), issued by warp 0
    // right after its scan, completing on rbar (one phase per chunk)
    __shared__ __align__(8) unsigned long long rbar;
    const uint32_t rbar_s = (uint32_t)__cvta_generic_to_shared(&rbar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(rbar_s) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    uint32_t rphase = 0;
#endif
#else
    load_tables(T, gtab);                    // (the first chunk's barriers cover it)
#endif
    const uint32_t ts = off[t], te = off[t + 1];
    const int nt = (int)(te - ts);
    const int tile = (int)blockDim.x / G;        // target tuples per pass (the launch picks the block size)
    for (int i0 = 0; i0 < nt; i0 += NEAR_TPT * tile) {
        const int tp = tid % tile;
        const int g = tid / tile;
        const int ni = min(NEAR_TPT * tile, nt - i0);   // targets in this pass
        const bool active = (g < G) && (NEAR_TPT * tp < ni);
        int la[NEAR_TPT];
        double4 A[NEAR_TPT];
        PairAcc acc[NEAR_TPT];
#pragma unroll
        for (int u = 0; u < NEAR_TPT; ++u) {
            la[u] = min(NEAR_TPT * tp + u, ni - 1);
            A[u] = src[ts + i0 + la[u]];
        }
        for (int64_t q = q0; q < q1;) {
            if (q != q0 || !FMM2D_NEAR_SKIPBAR) __syncthreads();   // previous chunk consumed
            if (warp == 0) {
                const int64_t qq = q + lane;
                int sz = 0;
                uint32_t lf = 0;
                if (qq < q1) {
                    lf = sidx[qq];
                    sz = (int)(off[lf + 1] - off[lf]);
                }
                int incl = sz;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    int v = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += v;
                }
                const unsigned fit = __ballot_sync(0xffffffffu, qq < q1 && incl <= NEAR_CHUNK);
                const int nl = __popc(fit);       // leaves in this chunk (prefix property)
                if (lane < nl) cstart[lane + 1] = incl;
                if (lane == 0) {
                    cstart[0] = 0;
                    cinfo[0] = nl;
                    cinfo[1] = -1;
                }
                __syncwarp();
                if (lane < nl && lf == (uint32_t)t) cinfo[1] = incl - sz;
#if FMM2D_NEAR_TMA_TABLES && FMM2D_NEAR_TMA_ROWS
                const int rows = __shfl_sync(0xffffffffu, incl, nl - 1);
                if (lane == 0) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // after the generic reads of S
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(rbar_s),
                                 "r"((uint32_t)(rows * sizeof(double4))) : "memory");
                }
                __syncwarp();
                if (lane < nl) {
                    // own / replicated leaf: rows at its position; halo leaf (sharded plans): in hsrc
                    const uint32_t hm = lmap ? lmap[lf] : 0xFFFFFFFFu;
                    const double4* sp = (hm != 0xFFFFFFFFu) ? hsrc + hm : src + off[lf];
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                 ::"r"((uint32_t)__cvta_generic_to_shared(&S[incl - sz])), "l"(sp),
                                 "r"((uint32_t)(sz * sizeof(double4))), "r"(rbar_s) : "memory");
                }
#endif
            }
            __syncthreads();
            const int nl = cinfo[0];
#if FMM2D_NEAR_TMA_TABLES && FMM2D_NEAR_TMA_ROWS
            {
                uint32_t done = 0;
                while (!done)
                    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                                 : "=r"(done) : "r"(rbar_s), "r"(rphase) : "memory");
                rphase ^= 1u;
            }
            if (false)
#endif
            for (int l = warp; l < nl; l += (int)blockDim.x / 32) {
                const uint32_t lf = sidx[q + l];
                // own / replicated leaf: rows at its position; halo leaf (sharded plans): in hsrc
                const uint32_t hm = lmap ? lmap[lf] : 0xFFFFFFFFu;
                const double4* __restrict__ sp = (hm != 0xFFFFFFFFu) ? hsrc + hm : src + off[lf];
                const int c0 = cstart[l], sz = cstart[l + 1] - c0;
#ifndef FMM2D_NEAR_EXP_NOSTAGE
                for (int e = lane; e < sz; e += 32) S[c0 + e] = sp[e];
#else
                (void)sp; (void)c0; (void)sz;              // timing experiment only: rows not staged
#endif
            }
#if !(FMM2D_NEAR_TMA_TABLES && FMM2D_NEAR_TMA_ROWS)
            __syncthreads();
#endif
            const int total = cstart[nl];
#if FMM2D_NEAR_TMA_TABLES
            if (!tables_ready) {                 // first chunk: the tables' bulk copy has landed
                uint32_t done = 0;
                while (!done)
                    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                                 : "=r"(done) : "r"(tbar_s) : "memory");
                tables_ready = true;
            }
#endif
            const int kown = (cinfo[1] >= 0) ? cinfo[1] : total;       // own leaf rows [kown, kown+nt)
            const int kend = min(total, kown + nt);
            if (active) {
                // rows before the own leaf, then after it: no self pair possible
#pragma unroll NEAR_UNROLL
                for (int k = g; k < kown; k += G) {
                    const double4 s = S[k];
#pragma unroll
                    for (int u = 0; u < NEAR_TPT; ++u) pair<REAL>(acc[u], A[u].x - s.x, A[u].y - s.y, s.z, s.w, NT);
                }
#pragma unroll NEAR_UNROLL
                for (int k = first_in_class(kend, g, G); k < total; k += G) {
                    const double4 s = S[k];
#pragma unroll
                    for (int u = 0; u < NEAR_TPT; ++u) pair<REAL>(acc[u], A[u].x - s.x, A[u].y - s.y, s.z, s.w, NT);
                }
                // own leaf: neutralise j == i
                for (int k = first_in_class(kown, g, G); k < kend; k += G) {
                    const double4 s = S[k];
#pragma unroll
                    for (int u = 0; u < NEAR_TPT; ++u) {
                        const bool x = (k == kown + i0 + la[u]);
                        pair<REAL>(acc[u], x ? 1.0 : A[u].x - s.x, x ? 0.0 : A[u].y - s.y, x ? 0.0 : s.z,
                                   x ? 0.0 : s.w, NT);
                    }
                }
            }
            q += nl;
        }
        __syncthreads();                          // chunk buffer free: reuse it for partial sums
#pragma unroll
        for (int u = 0; u < NEAR_TPT; ++u) red[u][tid] = pack(acc[u]);
        __syncthreads();
        // finalize: NEAR_TPT*tile targets, thread k < ni handles target k (tuple k/TPT, slot k%TPT)
        for (int kk = tid; kk < ni; kk += (int)blockDim.x) {
            const int ptp = kk / NEAR_TPT, slot = kk % NEAR_TPT;
            double4 acc = red[slot][ptp];
            for (int gg = 1; gg < G; ++gg) {
                const double4 v = red[slot][gg * tile + ptp];
                acc.x += v.x;
                acc.y += v.y;
                acc.z += v.z;
                acc.w += v.w;
            }
            if (segi >= 0) {                      // a segment of a split leaf: partial sums only
                part[segi * part_w + i0 + kk] = acc;
                continue;
            }
            if (nacc) {                           // overlapped eval: P2P sums only (k_near_final adds L2P)
                nacc[ts + i0 + kk] = acc;
                continue;
            }
            double4 f;                            // L2P (Horner) of the target
#ifndef FMM2D_NEAR_EXP_NOL2P
            {
                const double4 me = src[ts + i0 + kk];
                l2p(loc + t * (p + 1), p, me.x - cx[t], me.y - cy[t], f.x, f.y, f.z, f.w);
            }
#else
            f = make_double4(0.0, 0.0, 0.0, 0.0);    // timing experiment only
#endif
            if (m2p_off && m2p_off[t + 1] > m2p_off[t]) {      // r/R exchange: M2P sums
                const double4 g = m2p_acc[ts + i0 + kk];
                f.x += g.x;
                f.y += g.y;
                f.z += g.z;
                f.w += g.w;
            }
#ifndef FMM2D_NEAR_EXP_NOSTORE
            const uint32_t o = perm[ts + i0 + kk];
#else
            const uint32_t o = ts + i0 + kk;         // timing experiment only: leaf order, no scatter
#endif
            if (phi) phi[o] = make_double2(acc.x + f.x, acc.y + f.y);
            if (dphi) dphi[o] = make_double2(acc.z + f.z, acc.w + f.w);
        }
        __syncthreads();
    }
}

// Split leaves: the partial sums of their segments (in segment order) + L2P + M2P.
__global__ void __launch_bounds__(NEAR_T) k_near_combine(const uint32_t* __restrict__ leaves,
                                                         const int64_t* __restrict__ seg_off, const double4* __restrict__ part,
                                                         int part_w, int p, const uint32_t* __restrict__ off,
                                                         const double4* __restrict__ src, const double* __restrict__ cx,
                                                         const double* __restrict__ cy, const double2* __restrict__ loc,
                                                         const uint32_t* __restrict__ perm, double2* __restrict__ phi,
                                                         double2* __restrict__ dphi, const int64_t* __restrict__ m2p_off,
                                                         const double4* __restrict__ m2p_acc, double4* __restrict__ nacc)
{
    const uint32_t t = leaves[blockIdx.x];
    const uint32_t ts = off[t], te = off[t + 1];
    for (uint32_t i = ts + threadIdx.x; i < te; i += NEAR_T) {
        double4 acc = part[seg_off[t] * part_w + (i - ts)];
        for (int64_t sg = seg_off[t] + 1; sg < seg_off[t + 1]; ++sg) {
            const double4 v = part[sg * part_w + (i - ts)];
            acc.x += v.x;
            acc.y += v.y;
            acc.z += v.z;
            acc.w += v.w;
        }
        if (nacc) {                               // overlapped eval: P2P sums only
            nacc[i] = acc;
            continue;
        }
        const double4 me = src[i];
        double4 f;
        l2p(loc + (int64_t)t * (p + 1), p, me.x - cx[t], me.y - cy[t], f.x, f.y, f.z, f.w);
        if (m2p_off && m2p_off[t + 1] > m2p_off[t]) {
            const double4 g = m2p_acc[i];
            f.x += g.x;
            f.y += g.y;
            f.z += g.z;
            f.w += g.w;
        }
        const uint32_t o = perm[i];
        if (phi) phi[o] = make_double2(acc.x + f.x, acc.y + f.y);
        if (dphi) dphi[o] = make_double2(acc.z + f.z, acc.w + f.w);
    }
}

// Overlapped evaluation (DESIGN 6.4): the P2P sums nacc (leaf order) + L2P + M2P, written
// at the input positions.  One warp per target leaf, lanes over its points.
__global__ void __launch_bounds__(NEAR_T) k_near_final(int64_t t0, int64_t nl, int p, const uint32_t* __restrict__ off,
                                                       const double4* __restrict__ nacc, const double4* __restrict__ src,
                                                       const double* __restrict__ cx, const double* __restrict__ cy,
                                                       const double2* __restrict__ loc, const uint32_t* __restrict__ perm,
                                                       double2* __restrict__ phi, double2* __restrict__ dphi,
                                                       const int64_t* __restrict__ m2p_off,
                                                       const double4* __restrict__ m2p_acc)
{
    const int64_t w = ((int64_t)blockIdx.x * NEAR_T + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= nl) return;
    const int64_t t = t0 + w;
    const uint32_t ts = off[t], te = off[t + 1];
    const bool m2p = m2p_off && m2p_off[t + 1] > m2p_off[t];
    for (uint32_t i = ts + lane; i < te; i += 32) {
        const double4 acc = nacc[i];
        const double4 me = src[i];
        double4 f;
        l2p(loc + t * (p + 1), p, me.x - cx[t], me.y - cy[t], f.x, f.y, f.z, f.w);
        if (m2p) {
            const double4 g = m2p_acc[i];
            f.x += g.x;
            f.y += g.y;
            f.z += g.z;
            f.w += g.w;
        }
        const uint32_t o = perm[i];
        if (phi) phi[o] = make_double2(acc.x + f.x, acc.y + f.y);
        if (dphi) dphi[o] = make_double2(acc.z + f.z, acc.w + f.w);
    }
}

// Wide leaves (> NEAR_CHUNK points): sources straight from global memory.
template <bool REAL>
__global__ void __launch_bounds__(NEAR_T) k_near_wide(int p, int64_t t0, const uint32_t* __restrict__ off,
                                                      const int64_t* __restrict__ soff,
                                                      const uint32_t* __restrict__ sidx,
                                                      const double4* __restrict__ src, const double* __restrict__ cx,
                                                      const double* __restrict__ cy, const double2* __restrict__ loc,
                                                      const uint32_t* __restrict__ perm,
                                                      const fm::TablesN* __restrict__ gtab, double2* __restrict__ phi,
                                                      double2* __restrict__ dphi, const int64_t* __restrict__ m2p_off,
                                                      const double4* __restrict__ m2p_acc,
                                                      const uint32_t* __restrict__ lmap,
                                                      const double4* __restrict__ hsrc)
{
    __shared__ fm::TablesN T;
    load_tables(T, gtab);
    __syncthreads();
    const NearTab NT(T, threadIdx.x & 31);
    const int64_t t = t0 + blockIdx.x;
    const uint32_t ts = off[t], te = off[t + 1];
    for (uint32_t i = ts + threadIdx.x; i < te; i += NEAR_T) {
        const double4 me = src[i];
        PairAcc acc;
        for (int64_t q = soff[t]; q < soff[t + 1]; ++q) {
            const uint32_t lf = sidx[q];
            const uint32_t hm = lmap ? lmap[lf] : 0xFFFFFFFFu;
            const double4* __restrict__ sp = (hm != 0xFFFFFFFFu) ? hsrc + hm - off[lf] : src;   // indexed by position
            for (uint32_t j = off[lf]; j < off[lf + 1]; ++j) {
                const double4 s = sp[j];
                const bool self = (j == i) && (hm == 0xFFFFFFFFu);
                pair<REAL>(acc, self ? 1.0 : me.x - s.x, self ? 0.0 : me.y - s.y, self ? 0.0 : s.z,
                           self ? 0.0 : s.w, NT);
            }
        }
        double fr, fi, gr, gi;
        l2p(loc + t * (p + 1), p, me.x - cx[t], me.y - cy[t], fr, fi, gr, gi);
        if (m2p_off && m2p_off[t + 1] > m2p_off[t]) {          // r/R exchange: M2P sums
            const double4 g = m2p_acc[i];
            fr += g.x;
            fi += g.y;
            gr += g.z;
            gi += g.w;
        }
        const uint32_t o = perm[i];
        const double2 f = acc.phi(), d = acc.dphi();
        if (phi) phi[o] = make_double2(f.x + fr, f.y + fi);
        if (dphi) dphi[o] = make_double2(d.x + gr, d.y + gi);
    }
}

// ---------------------------------------------------------------------------------
// Symmetric near field.  The strong relation is symmetric, so every
// unordered pair of distinct leaves (t, s), s > t, is evaluated ONCE by the CTA of t:
// the shared part of the pair (|dz|^2, log|dz|^2, Arg dz and Arg of the reversed
// componentwise difference, 1/|dz|^2) feeds both Phi_i (t side, registers) and Phi_j
// (s side).  The s-side partial sums of a chunk are reduced over the CTA's target
// threads in shared memory in fixed order and written to the slot of (s, t): slot row
// lower[s] + (position of t in s's list).  k_near_gather then adds, per point, its own
// CTA's sum and its slots in ascending order -- deterministic, no atomics.
// Own-leaf pairs (t, t) are evaluated one-sided (ordered, self pair neutralised).
template <bool REAL>
__device__ __forceinline__ void pair_sym(PairAcc& at, PairAcc& as, double dx, double dy, double mt_r, double mt_i,
                                         double ms_r, double ms_i, const fm::Tables& T)
{
    // at: target i gets m_s Log(dz) and m_s/dz;  as: source j gets m_t Log(-dz) and -m_t/dz
    const double r2 = fma(dx, dx, dy * dy);
    const double l2 = fm::log_pos(r2, T.lg);
    double th, thn;
    fm::arg_pair(dx, dy, T.at, th, thn);
    const double ir2 = fm::rcp(r2);
    const double a2 = ms_r * ir2, b2 = mt_r * ir2;
    at.ar = fma(ms_r, l2, at.ar);
    at.br = fma(ms_r, th, at.br);
    at.dr = fma(a2, dx, at.dr);
    at.di = fma(-a2, dy, at.di);
    as.ar = fma(mt_r, l2, as.ar);
    as.br = fma(mt_r, thn, as.br);
    as.dr = fma(-b2, dx, as.dr);                  // m conj(-dz) / |dz|^2
    as.di = fma(b2, dy, as.di);
    if (!REAL) {
        const double ai2 = ms_i * ir2, bi2 = mt_i * ir2;
        at.ai = fma(ms_i, l2, at.ai);
        at.bi = fma(ms_i, th, at.bi);
        at.dr = fma(ai2, dy, at.dr);
        at.di = fma(ai2, dx, at.di);
        as.ai = fma(mt_i, l2, as.ai);
        as.bi = fma(mt_i, thn, as.bi);
        as.dr = fma(-bi2, dy, as.dr);
        as.di = fma(-bi2, dx, as.di);
    }
}

struct SymArgs {
    const uint32_t* off;       // leaf offsets
    const int64_t* soff;       // strong CSR offsets (leaf level)
    const uint32_t* sidx;
    const uint32_t* mirror;    // per CSR entry: position of the row's leaf in the column leaf's row
    const uint32_t* selfpos;   // per leaf: position of the leaf in its own row
    const int64_t* lower;      // per leaf: first slot row
    const double4* src;
    const double* cx;
    const double* cy;
    const double2* loc;
    const fm::Tables* tab;
    double4* slot;
    double4* tsum;
    int p, G, tile, npass, rows, slot_w;
};

// dynamic shared memory: S[rows] | part[max(rows * tile, 2 * NEAR_T)] | Tables
template <bool REAL>
#ifndef FMM2D_SYM_MINB
#define FMM2D_SYM_MINB 5
#endif
__global__ void __launch_bounds__(NEAR_T, FMM2D_SYM_MINB) k_near_sym(SymArgs A)
{
    extern __shared__ __align__(16) unsigned char smem[];
    double4* S = reinterpret_cast<double4*>(smem);
    const int G = A.G, tile = A.tile, rows = A.rows;
    const int npart = max(rows * tile, 2 * NEAR_T);
    double4* part = S + rows;
    fm::Tables& T = *reinterpret_cast<fm::Tables*>(part + npart);
    __shared__ int cstart[33];
    __shared__ int cleaf[32];
    __shared__ int cinfo[1];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    load_tables(T, A.tab);
    const int64_t t = blockIdx.x;
    const uint32_t ts = A.off[t], te = A.off[t + 1];
    const int nt = (int)(te - ts);
    const int64_t q0 = A.soff[t], q1 = A.soff[t + 1];
    const int64_t qself = q0 + A.selfpos[t];
    const int per = (nt + A.npass - 1) / A.npass;            // targets per pass (<= 2 tile)
    const int tp = tid % tile, g = tid / tile;
    for (int pass = 0, i0 = 0; i0 < nt; ++pass, i0 += per) {
        const int ni = min(per, nt - i0);
        const int npair = (ni + 1) / 2;
        const bool active = (g < G) && (tp < npair);
        const int la = min(2 * tp, ni - 1), lb = min(2 * tp + 1, ni - 1);
        const double4 PA = A.src[ts + i0 + la];
        const double4 PB = A.src[ts + i0 + lb];
        const double mbr = (2 * tp + 1 < ni) ? PB.z : 0.0;   // odd count: B duplicates A on the s side
        const double mbi = (2 * tp + 1 < ni) ? PB.w : 0.0;
        PairAcc aa, ab;
        // ---- own leaf (one-sided, ordered pairs, j != i)
        __syncthreads();
        for (int e = tid; e < nt; e += NEAR_T) S[e] = A.src[ts + e];
        __syncthreads();
        if (active) {
            const int sa = i0 + la, sb = i0 + lb;
            for (int k = g; k < nt; k += G) {
                const double4 s = S[k];
                const bool xa = (k == sa), xb = (k == sb);
                pair_t<REAL>(aa, xa ? 1.0 : PA.x - s.x, xa ? 0.0 : PA.y - s.y, xa ? 0.0 : s.z, xa ? 0.0 : s.w, T);
                pair_t<REAL>(ab, xb ? 1.0 : PB.x - s.x, xb ? 0.0 : PB.y - s.y, xb ? 0.0 : s.z, xb ? 0.0 : s.w, T);
            }
        }
        // ---- upper leaves s > t: symmetric
        for (int64_t q = qself + 1; q < q1;) {
            __syncthreads();
            if (warp == 0) {
                const int64_t qq = q + lane;
                int sz = 0;
                if (qq < q1) {
                    const uint32_t lf = A.sidx[qq];
                    sz = (int)(A.off[lf + 1] - A.off[lf]);
                    cleaf[lane] = (int)lf;
                }
                int incl = sz;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    int v = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += v;
                }
                const unsigned fit = __ballot_sync(0xffffffffu, qq < q1 && incl <= rows);
                const int nl = __popc(fit);
                if (lane < nl) cstart[lane + 1] = incl;
                if (lane == 0) {
                    cstart[0] = 0;
                    cinfo[0] = nl;
                }
            }
            __syncthreads();
            const int nl = cinfo[0];
            for (int l = warp; l < nl; l += NEAR_T / 32) {
                const uint32_t s0 = A.off[cleaf[l]];
                const int c0 = cstart[l], sz = cstart[l + 1] - c0;
                for (int e = lane; e < sz; e += 32) S[c0 + e] = A.src[s0 + e];
            }
            __syncthreads();
            const int total = cstart[nl];
            if (active) {
                for (int k = g; k < total; k += G) {
                    const double4 s = S[k];
                    PairAcc ss;
                    pair_sym<REAL>(aa, ss, PA.x - s.x, PA.y - s.y, PA.z, PA.w, s.z, s.w, T);
                    pair_sym<REAL>(ab, ss, PB.x - s.x, PB.y - s.y, mbr, mbi, s.z, s.w, T);
                    part[k * tile + tp] = pack(ss);
                }
            }
            __syncthreads();
            // reduce the s-side partials of each row over the active target threads
            if (tid < total) {
                int l = 0;
                while (cstart[l + 1] <= tid) ++l;
                double4 v = part[tid * tile];
                for (int u = 1; u < npair; ++u) {
                    const double4 w = part[tid * tile + u];
                    v.x += w.x;
                    v.y += w.y;
                    v.z += w.z;
                    v.w += w.w;
                }
                const uint32_t sl = (uint32_t)cleaf[l];
                double4* dst = A.slot + (A.lower[sl] + A.mirror[q + l]) * A.slot_w + (tid - cstart[l]);
                if (pass > 0) {
                    const double4 o = *dst;
                    v.x += o.x;
                    v.y += o.y;
                    v.z += o.z;
                    v.w += o.w;
                }
                *dst = v;
            }
            q += nl;
        }
        // ---- t side: reduce over groups, add L2P, store in leaf order
        __syncthreads();
        double4(*red)[NEAR_T] = reinterpret_cast<double4(*)[NEAR_T]>(part);
        red[0][tid] = pack(aa);
        red[1][tid] = pack(ab);
        __syncthreads();
        for (int kk = tid; kk < ni; kk += NEAR_T) {
            const int ptp = kk >> 1, s = kk & 1;
            double4 acc = red[s][ptp];
            for (int gg = 1; gg < G; ++gg) {
                const double4 v = red[s][gg * tile + ptp];
                acc.x += v.x;
                acc.y += v.y;
                acc.z += v.z;
                acc.w += v.w;
            }
            const uint32_t i = ts + i0 + kk;
            const double4 me = A.src[i];
            double fr, fi, gr, gi;
            l2p(A.loc + t * (A.p + 1), A.p, me.x - A.cx[t], me.y - A.cy[t], fr, fi, gr, gi);
            A.tsum[i] = make_double4(acc.x + fr, acc.y + fi, acc.z + gr, acc.w + gi);
        }
    }
}

// per point: own-CTA sum + its slots (ascending), written at the input position
__global__ void __launch_bounds__(NEAR_T) k_near_gather(const uint32_t* __restrict__ off,
                                                        const uint32_t* __restrict__ selfpos,
                                                        const int64_t* __restrict__ lower, int slot_w,
                                                        const double4* __restrict__ tsum,
                                                        const double4* __restrict__ slot,
                                                        const uint32_t* __restrict__ perm, double2* __restrict__ phi,
                                                        double2* __restrict__ dphi)
{
    const int64_t s = blockIdx.x;
    const uint32_t s0 = off[s], s1 = off[s + 1];
    const int nlow = (int)selfpos[s];
    const int64_t base = lower[s];
    for (uint32_t i = s0 + threadIdx.x; i < s1; i += blockDim.x) {
        double4 v = tsum[i];
        for (int k = 0; k < nlow; ++k) {
            const double4 w = slot[(base + k) * slot_w + (i - s0)];
            v.x += w.x;
            v.y += w.y;
            v.z += w.z;
            v.w += w.w;
        }
        const uint32_t o = perm[i];
        if (phi) phi[o] = make_double2(v.x, v.y);
        if (dphi) dphi[o] = make_double2(v.z, v.w);
    }
}

// per leaf t: position of t in its own (sorted) row; per upper entry (t, s): position of t in row s
__global__ void k_sym_index(int64_t nl, const int64_t* __restrict__ soff, const uint32_t* __restrict__ sidx,
                            uint32_t* __restrict__ selfpos, uint32_t* __restrict__ mirror)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nl) return;
    const int64_t q0 = soff[t], q1 = soff[t + 1];
    for (int64_t q = q0; q < q1; ++q) {
        const uint32_t s = sidx[q];
        if (s == (uint32_t)t) selfpos[t] = (uint32_t)(q - q0);
        if (s > (uint32_t)t) {
            int64_t lo = soff[s], hi = soff[s + 1];             // lower_bound(t) in row s
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (sidx[mid] < (uint32_t)t) lo = mid + 1;
                else hi = mid;
            }
            mirror[q] = (uint32_t)(lo - soff[s]);
        }
    }
}

inline unsigned grid_for(int64_t n, int bs) { return (unsigned)((n + bs - 1) / bs); }

// per-device table copy (built once on the host, long double evaluation)
const fm::AllTables* device_tables(int dev, int* rc)
{
    static const fm::AllTables* cache[64] = {nullptr};
    static std::mutex mu;                            // plans may be built from several threads
    *rc = 0;
    if (dev < 0 || dev >= 64) {
        *rc = FMM2D_EINVAL;
        return nullptr;
    }
    std::lock_guard<std::mutex> lk(mu);
    if (cache[dev]) return cache[dev];
    static fm::AllTables h;
    fm::make_tables(&h.t);
    fm::make_tables_n(&h.n);
    fm::AllTables* d = nullptr;
    cudaError_t e = cudaMalloc((void**)&d, sizeof(fm::AllTables));
    if (e == cudaSuccess) e = cudaMemcpy(d, &h, sizeof(h), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        fmm2d_set_last_cuda_error(e, "device_tables", __FILE__, __LINE__);
        *rc = FMM2D_ECUDA;
        return nullptr;
    }
    cache[dev] = d;
    return d;
}

}  // namespace

int gather_strengths(fmm2d_plan* P, const double2* m)
{
    const int64_t k0 = P->pos0, k1 = P->pos1;
    k_gather_m<<<grid_for(k1 - k0, 256 * GM), 256, 0, P->stream>>>(m, P->perm, k0, k1, P->src);
    fmm2d::note_launch();
    FMM2D_CUDA_TRY(cudaGetLastError());
    return 0;
}

int prepare_near(fmm2d_plan* P)
{
    int rc = 0;
    P->tables = device_tables(P->device, &rc);
    return rc;
}

__global__ void k_to_i64(const uint32_t* __restrict__ a, int64_t n, int64_t* __restrict__ b)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = a[i];
    if (i == n) b[n] = 0;
}

constexpr int SYM_MAXLEAF = 64;

static size_t sym_smem(const fmm2d_plan* P)
{
    const int npart = std::max(P->sym_rows * P->sym_tile, 2 * NEAR_T);
    return sizeof(double4) * (P->sym_rows + npart) + sizeof(fm::Tables);
}

// Build-time set-up of the symmetric near field: leaves of at
// most SYM_MAXLEAF points; otherwise (or if the slot buffer does not fit) the one-sided
// kernel is used.
int prepare_near_sym(fmm2d_plan* P)
{
    P->sym = false;
    const int L = P->L, ml = P->stats.max_leaf;
    if (L < 1 || ml > SYM_MAXLEAF || ml < 1 || !(P->flags & FMM2D_SYMMETRIC_P2P) || P->nranks > 1 ||
        (P->flags & (FMM2D_RR_EXCHANGE | FMM2D_MIDPOINT)))
        return 0;
    cudaStream_t st = P->stream;
    const int64_t nl = nboxes(L);
    const Csr& S = P->strong[L];
    P->sym_npass = (ml + 31) / 32;
    const int per = (ml + P->sym_npass - 1) / P->sym_npass;
    P->sym_tile = (per + 1) / 2;
    P->sym_rows = std::max(ml, std::min(64, 2 * ml));
    P->slot_w = ml;
    FMM2D_TRY(dev_alloc(P, (void**)&P->sym_mirror, sizeof(uint32_t) * std::max<int64_t>(S.total, 1)));
    FMM2D_TRY(dev_alloc(P, (void**)&P->sym_selfpos, sizeof(uint32_t) * nl));
    FMM2D_TRY(dev_alloc(P, (void**)&P->sym_lower, sizeof(int64_t) * (nl + 1)));
    k_sym_index<<<grid_for(nl, 256), 256, 0, st>>>(nl, S.off, S.idx, P->sym_selfpos, P->sym_mirror);
    fmm2d::note_launch();
    int64_t* cnt = nullptr;
    void* scratch = nullptr;
    size_t sb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, sb, (int64_t*)nullptr, (int64_t*)nullptr, (int)(nl + 1), st);
    FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&cnt, sizeof(int64_t) * (nl + 1), st));
    FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&scratch, sb, st));
    k_to_i64<<<grid_for(nl + 1, 256), 256, 0, st>>>(P->sym_selfpos, nl, cnt);
    fmm2d::note_launch();
    FMM2D_CUDA_TRY(cub::DeviceScan::ExclusiveSum(scratch, sb, cnt, P->sym_lower, (int)(nl + 1), st));
    int64_t total = 0;
    FMM2D_CUDA_TRY(cudaMemcpyAsync(&total, P->sym_lower + nl, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    FMM2D_CUDA_TRY(cudaStreamSynchronize(st));
    cudaFreeAsync(cnt, st);
    cudaFreeAsync(scratch, st);
    if (dev_alloc(P, (void**)&P->sym_slot, sizeof(double4) * std::max<int64_t>(total, 1) * P->slot_w) ||
        dev_alloc(P, (void**)&P->sym_t, sizeof(double4) * P->n)) {
        cudaGetLastError();                       // out of memory: keep the one-sided kernel
        return 0;
    }
    const size_t smem = sym_smem(P);
    if (smem > 48 * 1024) {
        FMM2D_CUDA_TRY(cudaFuncSetAttribute(k_near_sym<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        FMM2D_CUDA_TRY(cudaFuncSetAttribute(k_near_sym<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    P->sym = true;
    return 0;
}

// mode 0: the whole near field (P2P + L2P + M2P, outputs); mode 1: P2P sums only into
// P->nacc (overlapped eval, before the expansions are done); mode 2: k_near_final.
int run_near(fmm2d_plan* P, double2* phi, double2* dphi, int mode)
{
    const int L = P->L;
    const int64_t t0 = P->box_lo(L), nl = P->box_hi(L) - t0;    // own target leaves
    const double* cx = P->cx + P->base[L];
    const double* cy = P->cy + P->base[L];
    const double2* loc = P->lcl[L];
    const uint32_t* off = P->boff + P->obase[L];
    const bool real = (P->flags & FMM2D_REAL_STRENGTHS) != 0;
    // P->tables: fm::AllTables {Tables t (rr.cu, symmetric kernel), TablesN n (k_near, k_near_wide)}
    const fm::Tables* tab = &((const fm::AllTables*)P->tables)->t;
    const fm::TablesN* tabn = &((const fm::AllTables*)P->tables)->n;
    const int64_t* m2p_off = (P->rr_nm2p > 0) ? P->rr_m2p.off : nullptr;     // r/R exchange
    double4* nacc = (mode == 1) ? P->nacc : nullptr;
    if (mode == 2) {
        k_near_final<<<grid_for(nl * 32, NEAR_T), NEAR_T, 0, P->stream>>>(t0, nl, P->p, off, P->nacc, P->src, cx, cy,
                                                                        loc, P->perm, phi, dphi, m2p_off, P->rr_acc);
        fmm2d::note_launch();
        FMM2D_CUDA_TRY(cudaGetLastError());
        return 0;
    }
    if (P->sym) {
        SymArgs A;
        A.off = off;
        A.soff = P->strong[L].off;
        A.sidx = P->strong[L].idx;
        A.mirror = P->sym_mirror;
        A.selfpos = P->sym_selfpos;
        A.lower = P->sym_lower;
        A.src = P->src;
        A.cx = cx;
        A.cy = cy;
        A.loc = loc;
        A.tab = tab;
        A.slot = P->sym_slot;
        A.tsum = P->sym_t;
        A.p = P->p;
        A.tile = P->sym_tile;
        A.G = NEAR_T / P->sym_tile;
        A.npass = P->sym_npass;
        A.rows = P->sym_rows;
        A.slot_w = P->slot_w;
        const size_t smem = sym_smem(P);
        if (real) k_near_sym<true><<<(unsigned)nl, NEAR_T, smem, P->stream>>>(A);
        else      k_near_sym<false><<<(unsigned)nl, NEAR_T, smem, P->stream>>>(A);
        fmm2d::note_launch();
        FMM2D_CUDA_TRY(cudaGetLastError());
        k_near_gather<<<(unsigned)nl, NEAR_T, 0, P->stream>>>(off, P->sym_selfpos, P->sym_lower, P->slot_w,
                                                               P->sym_t, P->sym_slot, P->perm, phi, dphi);
        fmm2d::note_launch();
        FMM2D_CUDA_TRY(cudaGetLastError());
        return 0;
    }
    if (P->stats.max_leaf <= NEAR_CHUNK) {
        // target tuples per leaf, groups so that tuples * G <= 128
        const int pairs = (std::max(1, P->stats.max_leaf) + NEAR_TPT - 1) / NEAR_TPT;
        // block size 64 / 96 / 128: the one whose G = T / tuples groups leave the fewest idle lanes
        // (C5: 12 tuples -> 96 threads, 8 groups, every lane busy; 128 threads would idle 8)
        int T = NEAR_T, G = 1;
        double best = -1.0;
        for (int cand = NEAR_T; cand >= 64; cand -= 32) {
            const int g = std::max(1, cand / std::min(pairs, cand));
            const double util = (double)std::min(pairs, cand) * g / cand;
            if (util > best + 1e-9) {
                best = util;
                T = cand;
                G = g;
            }
        }
        if (const char* e = getenv("FMM2D_NEAR_THREADS")) {      // tuning / tests: force the block size
            const int v = atoi(e);
            if (v == 64 || v == 96 || v == 128) {
                T = v;
                G = std::max(1, T / std::min(pairs, T));
            }
        }
        const unsigned grid = (unsigned)(nl + P->near_nseg);
        if (real)
            k_near<true><<<grid, T, 0, P->stream>>>(G, P->p, t0, nl, P->near_seg_off, P->near_segs,
                                                        P->near_part, P->stats.max_leaf, off, P->near.off,
                                                        P->near.idx, P->src, cx, cy, loc, P->perm, tabn, phi, dphi,
                                                        m2p_off, P->rr_acc, nacc, P->lmap, P->hsrc);
        else
            k_near<false><<<grid, T, 0, P->stream>>>(G, P->p, t0, nl, P->near_seg_off, P->near_segs,
                                                         P->near_part, P->stats.max_leaf, off, P->near.off,
                                                         P->near.idx, P->src, cx, cy, loc, P->perm, tabn, phi, dphi,
                                                         m2p_off, P->rr_acc, nacc, P->lmap, P->hsrc);
        if (P->near_nsplit > 0) {
            fmm2d::note_launch();
            FMM2D_CUDA_TRY(cudaGetLastError());
            k_near_combine<<<(unsigned)P->near_nsplit, NEAR_T, 0, P->stream>>>(
                P->near_split, P->near_seg_off, P->near_part, P->stats.max_leaf, P->p, off, P->src, cx, cy, loc,
                P->perm, phi, dphi, m2p_off, P->rr_acc, nacc);
        }
    } else {
        if (real)
            k_near_wide<true><<<(unsigned)nl, NEAR_T, 0, P->stream>>>(P->p, t0, off, P->near.off, P->near.idx,
                                                                     P->src, cx, cy, loc, P->perm, tabn, phi, dphi,
                                                                     m2p_off, P->rr_acc, P->lmap, P->hsrc);
        else
            k_near_wide<false><<<(unsigned)nl, NEAR_T, 0, P->stream>>>(P->p, t0, off, P->near.off, P->near.idx,
                                                                      P->src, cx, cy, loc, P->perm, tabn, phi, dphi,
                                                                      m2p_off, P->rr_acc, P->lmap, P->hsrc);
    }
    fmm2d::note_launch();
    FMM2D_CUDA_TRY(cudaGetLastError());
    return 0;
}

}  // namespace fmm2d
