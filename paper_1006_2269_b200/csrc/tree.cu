// tree.cu -- A0-A2: validation, the balanced median-split tree and the box discs.
//
// Paper: "The multipole mesh is constructed first and is obtained by recursively
// splitting the source points at or near their median in each coordinate
// direction"; the points live in "a 2^d-tree cut at a certain maximum
// level".  Readings R5-R8, R13.
//
// GPU formulation (bit-exact by construction):
//  1. Ranks.  The total orders (x, idx) and (y, idx) (R6) are computed once, by
//     stable radix sorts, as dense ranks rx[i], ry[i] in [0, n).  After that every
//     comparison of the method is an integer comparison of ranks, and a point is an
//     8-byte record {rx, ry}.  The sort key is a 32-bit monotone image of the
//     coordinate, key = floor((c - cmin) * (2^32 - 1) / (cmax - cmin)); a stable sort
//     by it yields (key, idx) order, and the runs of equal keys (distinct coordinates
//     that share a bucket) are re-sorted by (c, idx) in place.  Runs longer than
//     RUN_MAX (heavy ties or duplicates) switch that axis to a full 64-bit sort of the
//     orderable coordinate bits -- same result, more passes.
//  2. Two record lists are kept, one grouped by box and sorted by rx inside each box
//     (the x-list), one sorted by ry inside each box (the y-list).  An x-split takes
//     the first ceil(n/2) of the x-list segment (trivially partitioned; that list is
//     not rewritten) and stably partitions the y-list segment by rx < the first high
//     record's rx: one pass with a block scan and a decoupled look-back.  Stability
//     keeps both lists sorted, so the y-split is the same step with the axes swapped.
//     The segment of a record is found from its position (box sizes are a pure
//     function of n, so all offsets come from a tiny per-level kernel).
//  3. Bounding boxes are the coordinates of segment endpoints; after the last level
//     the y-list IS the leaf order (leaves ascending, (y, idx) inside: R13).  One pass
//     writes the permutation, the source rows and every level's exact radius.
// Every kernel works on a position range [k0, k1) of whole boxes, so a rank of a
// sharded build continues below the top levels with its own subtrees only.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <utility>
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "fmm2d_internal.cuh"

namespace fmm2d {

namespace {

constexpr int RUN_MAX = 32;            // longest equal-key run fixed in place

__device__ __forceinline__ uint64_t orderable(double v)
{
    uint64_t u = (uint64_t)__double_as_longlong(v);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// orderable bits of min / max (atomicMin / atomicMax on uint64 keep the order)
struct Bounds {
    unsigned long long xmin, xmax, ymin, ymax;
    int bad;
};

// A0 (pass 1): validate, map -0 -> +0 (x + 0.0), keep the canonical coordinates,
// reduce the coordinate ranges.
constexpr int CT = 256;
__global__ void __launch_bounds__(CT) k_canon(const double2* __restrict__ z, int64_t n, double2* __restrict__ zc,
                                              Bounds* __restrict__ B)
{
    int64_t i = (int64_t)blockIdx.x * CT + threadIdx.x;
    uint64_t xmn = ~0ull, xmx = 0, ymn = ~0ull, ymx = 0;
    int bad = 0;
    for (; i < n; i += (int64_t)gridDim.x * CT) {
        const double2 v = z[i];
        const double x = __dadd_rn(v.x, 0.0), y = __dadd_rn(v.y, 0.0);
        if (!isfinite(x) || !isfinite(y)) bad = 1;
        zc[i] = make_double2(x, y);
        const uint64_t kx = orderable(x), ky = orderable(y);
        xmn = min(xmn, kx);
        xmx = max(xmx, kx);
        ymn = min(ymn, ky);
        ymx = max(ymx, ky);
    }
    typedef cub::BlockReduce<unsigned long long, CT> R;
    __shared__ typename R::TempStorage t0, t1, t2, t3;
    const unsigned long long a = R(t0).Reduce((unsigned long long)xmn, cub::Min());
    const unsigned long long b = R(t1).Reduce((unsigned long long)xmx, cub::Max());
    const unsigned long long c = R(t2).Reduce((unsigned long long)ymn, cub::Min());
    const unsigned long long d = R(t3).Reduce((unsigned long long)ymx, cub::Max());
    bad = __syncthreads_or(bad);
    if (threadIdx.x == 0) {
        atomicMin(&B->xmin, a);
        atomicMax(&B->xmax, b);
        atomicMin(&B->ymin, c);
        atomicMax(&B->ymax, d);
        if (bad) atomicOr(&B->bad, 1);
    }
}

__device__ __forceinline__ double from_orderable(uint64_t k)
{
    uint64_t u = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
    return __longlong_as_double((long long)u);
}

// monotone (non-decreasing) 32-bit image of a coordinate: every step rounds
// monotonically, so c <= c' implies key(c) <= key(c')
__device__ __forceinline__ uint32_t key32(double c, double cmin, double scale)
{
    const double t = __dmul_rn(__dsub_rn(c, cmin), scale);
    return (uint32_t)fmin(fmax(t, 0.0), 4294967295.0);
}

__device__ __forceinline__ double key_scale(unsigned long long omin, unsigned long long omax, double* cmin)
{
    const double mn = from_orderable(omin), mx = from_orderable(omax);
    const double w = __dsub_rn(mx, mn);
    // width 0 or overflowing: scale 0, one run (the 64-bit path takes over)
    double sc = (w > 0.0 && isfinite(w)) ? 4294967295.0 / w : 0.0;
    if (!isfinite(sc)) sc = 0.0;
    *cmin = mn;
    return sc;
}

// A0 (pass 2): the x-sort's keys (32-bit image of x, or the full orderable 64 bits)
// and its payload {idx, 32-bit image of y} -- the y key rides along, so the y-sort's
// input comes out of the x-sort in x order without a gather.  The presort runs over
// m points: all of them (sub == nullptr), or the ascending input indices sub[0..m) of
// one level-k box of a partitioned build; its ranks are offset by roff (the box's first
// leaf-order position), so every rank of the plan is a position.
template <bool K64>
__global__ void k_keys_x(const double2* __restrict__ zc, const uint32_t* __restrict__ sub, int64_t m,
                         const Bounds* __restrict__ B, uint32_t* __restrict__ k32, uint64_t* __restrict__ k64,
                         uint64_t* __restrict__ val)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m) return;
    const uint32_t i = sub ? sub[t] : (uint32_t)t;
    double xmn, ymn;
    const double sx = key_scale(B->xmin, B->xmax, &xmn);
    const double sy = key_scale(B->ymin, B->ymax, &ymn);
    const double2 v = zc[i];
    if (K64) k64[t] = orderable(v.x);
    else k32[t] = key32(v.x, xmn, sx);
    val[t] = (uint64_t)i | ((uint64_t)key32(v.y, ymn, sy) << 32);
}

// y-sort input in x order: key = 32-bit image of y, payload {x rank, idx}
__global__ void k_prep_y(const uint64_t* __restrict__ vx, int64_t m, uint32_t roff, uint32_t* __restrict__ key,
                         uint64_t* __restrict__ val)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m) return;
    const uint64_t v = vx[k];
    key[k] = (uint32_t)(v >> 32);
    val[k] = (uint64_t)(roff + (uint32_t)k) | (v << 32);          // {rx, idx}
}

// 64-bit fallback of the y-sort: input in idx order (so ties leave in idx order),
// payload {x rank, idx}; the x ranks are scattered once (rare path)
__global__ void k_scatter_rx(const uint64_t* __restrict__ vx, int64_t m, uint32_t* __restrict__ rx)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < m) rx[(uint32_t)vx[k]] = (uint32_t)k;
}
__global__ void k_keys_y64(const double2* __restrict__ zc, const uint32_t* __restrict__ sub,
                           const uint32_t* __restrict__ rx, int64_t m, uint32_t roff, uint64_t* __restrict__ k64,
                           uint64_t* __restrict__ val)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m) return;
    const uint32_t i = sub ? sub[t] : (uint32_t)t;
    k64[t] = orderable(zc[i].y);
    val[t] = (uint64_t)(roff + rx[i]) | ((uint64_t)i << 32);
}

// Runs of equal 32-bit keys are re-sorted by (c, idx) (insertion sort, exact
// coordinates from zc; idx sits at bit `ishift` of the 64-bit payload).  A run
// longer than RUN_MAX raises *overflow and is left alone (the caller redoes the axis
// with 64-bit keys).
__device__ __forceinline__ void fix_run(const uint32_t* __restrict__ key, int64_t n, const double2* __restrict__ zc,
                                        int axis, int ishift, uint64_t* __restrict__ val, int* __restrict__ overflow,
                                        int64_t k, uint32_t v)
{
    int len = 2;
    while (k + len < n && key[k + len] == v && len <= RUN_MAX) ++len;
    if (len > RUN_MAX) {
        atomicOr(overflow, 1);
        return;
    }
    double cv[RUN_MAX];
    uint32_t iv[RUN_MAX];
    uint64_t pv[RUN_MAX];
    for (int a = 0; a < len; ++a) {
        const uint64_t pl = val[k + a];
        const uint32_t i = (uint32_t)(pl >> ishift);
        const double2 zz = zc[i];
        const double ci = axis ? zz.y : zz.x;
        int b = a;
        while (b > 0 && (cv[b - 1] > ci || (cv[b - 1] == ci && iv[b - 1] > i))) {
            cv[b] = cv[b - 1];
            iv[b] = iv[b - 1];
            pv[b] = pv[b - 1];
            --b;
        }
        cv[b] = ci;
        iv[b] = i;
        pv[b] = pl;
    }
    for (int a = 0; a < len; ++a) val[k + a] = pv[a];
}

// FR keys per thread (vector loads): the run starts among them -- key[k-1] != key[k] ==
// key[k+1] -- are fixed by fix_run (about 1 % of the points at C5; the scan itself is the
// cost: one pass over the keys at memory speed instead of three scalar loads per key)
constexpr int FR = 8;
__global__ void k_fix_runs(const uint32_t* __restrict__ key, int64_t n, const double2* __restrict__ zc, int axis,
                           int ishift, uint64_t* __restrict__ val, int* __restrict__ overflow)
{
    const int64_t k0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * FR;
    if (k0 >= n) return;
    uint32_t kk[FR + 2];                              // key[k0 - 1 .. k0 + FR]
    if (k0 + FR <= n && ((reinterpret_cast<uintptr_t>(key + k0) & 15) == 0)) {
        const uint4 a = *reinterpret_cast<const uint4*>(key + k0);
        const uint4 b = *reinterpret_cast<const uint4*>(key + k0 + 4);
        kk[1] = a.x; kk[2] = a.y; kk[3] = a.z; kk[4] = a.w;
        kk[5] = b.x; kk[6] = b.y; kk[7] = b.z; kk[8] = b.w;
    } else {
#pragma unroll
        for (int u = 0; u < FR; ++u) kk[u + 1] = (k0 + u < n) ? key[k0 + u] : 0u;
    }
    kk[0] = (k0 > 0) ? key[k0 - 1] : ~kk[1];
    kk[FR + 1] = (k0 + FR < n) ? key[k0 + FR] : 0u;
#pragma unroll
    for (int u = 0; u < FR; ++u) {
        const int64_t k = k0 + u;
        if (k + 1 >= n) break;                         // a run needs k + 1 < n
        const uint32_t v = kk[u + 1];
        if (kk[u] != v && kk[u + 2] == v) fix_run(key, n, zc, axis, ishift, val, overflow, k, v);
    }
}

// y-list and the (local) x-ranks in y order (the key of the sort that inverts them)
__global__ void k_make_ylist(const uint64_t* __restrict__ vy, int64_t m, uint32_t roff, uint2* __restrict__ yl,
                             uint32_t* __restrict__ keyd, uint32_t* __restrict__ iota)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m) return;
    const uint32_t rx = (uint32_t)vy[k];
    yl[k] = make_uint2(rx, roff + (uint32_t)k);
    keyd[k] = rx - roff;
    iota[k] = (uint32_t)k;
}

// 1: the x-list by a direct scatter xl[rx] = {rx, ry} inside k_make_ylist (one random
// 8-byte write per point); 0: by one more radix sort of the x ranks (k_make_xlist)
#ifndef FMM2D_PRESORT_SCATTER
#define FMM2D_PRESORT_SCATTER 2
#endif
// 2: the records first bucketed by the top 8 bits of their x rank (one stable radix pass),
// then scattered: each bucket's destinations form one window of the x-list small enough to
// stay in L2, so the 8-byte writes merge into whole sectors there instead of in DRAM
__global__ void k_scatter_xlist(const uint32_t* __restrict__ key, const uint32_t* __restrict__ val, int64_t m,
                                uint32_t roff, uint2* __restrict__ xl)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < m) xl[key[k]] = make_uint2(roff + key[k], roff + val[k]);
}
__global__ void k_make_lists(const uint64_t* __restrict__ vy, int64_t m, uint32_t roff, uint2* __restrict__ yl,
                             uint2* __restrict__ xl)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m) return;
    const uint32_t rx = (uint32_t)vy[k];
    const uint2 r = make_uint2(rx, roff + (uint32_t)k);
    yl[k] = r;
    xl[rx - roff] = r;
}

// x-list from the y ranks in x order
__global__ void k_make_xlist(const uint32_t* __restrict__ ryx, int64_t m, uint32_t roff, uint2* __restrict__ xl)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < m) xl[k] = make_uint2(roff + (uint32_t)k, roff + ryx[k]);
}

// ---------------------------------------------------------------- partitioned build (DESIGN 8)
// Levels 0..k-1 of a partitioned build without a full presort: the split record of every
// (half-)box -- the first high record in (coordinate, idx) order -- is found by radix
// selection over all points (replicated on every rank), then each rank presorts only the
// points of its own level-k boxes.  A split record is {orderable 64-bit coordinate, idx};
// "(c, i) >= record" is the high side.
struct TopRec {
    unsigned long long key;
    uint32_t idx, pad;
};

__device__ __forceinline__ bool rec_ge(unsigned long long key, uint32_t idx, const TopRec& r)
{
    return key > r.key || (key == r.key && idx >= r.idx);
}

// the (half-)box of point (x, y, i) after `steps` split steps (x-split, y-split, ...),
// given the records of those steps: xr[l][box], yr[l][half] packed level by level
__device__ __forceinline__ uint32_t top_segment(double x, double y, uint32_t i, int steps,
                                                const TopRec* __restrict__ recs, const int* __restrict__ roff)
{
    const unsigned long long kx = orderable(x), ky = orderable(y);
    uint32_t seg = 0;
    for (int st = 0; st < steps; ++st) {
        const bool ax = (st & 1) != 0;                  // even steps: x-split, odd: y-split
        const TopRec& r = recs[roff[st] + seg];
        seg = 2 * seg + (rec_ge(ax ? ky : kx, i, r) ? 1u : 0u);
    }
    return seg;
}

// Selection state of one segment: the record sought is the want-th (in (key, idx) order)
// of the segment's points inside the current range, which is split into SEL_BUCKETS buckets.
//   mode 1: keys in [lo, lo + SEL_BUCKETS << shift), bucket (key - lo) >> shift
//   mode 2: key == keyfix, idx in [lo, lo + SEL_BUCKETS << shift), bucket (idx - lo) >> shift
//   mode 3 / 4: as 1 / 2, collect the points of bucket 0 (candidates); mode 0: idle
struct SelSeg {
    unsigned long long lo, keyfix;
    int shift, mode;
};
constexpr int SEL_BITS = 12;
constexpr int SEL_BUCKETS = 1 << SEL_BITS;   // per segment and pass (a 16 KB shared histogram)
constexpr int SEL_SMEM_SEGS = 12;             // segments per pass that fit the shared histogram
constexpr int SEL_COLLECT = 4096;             // a bucket this small is sorted on the host

__device__ __forceinline__ int sel_bucket(const SelSeg& S, unsigned long long key, uint32_t i)
{
    unsigned long long v;
    if (S.mode == 1 || S.mode == 3) {
        if (key < S.lo) return -1;
        v = (key - S.lo) >> S.shift;
    } else if (S.mode == 2 || S.mode == 4) {
        if (key != S.keyfix || (unsigned long long)i < S.lo) return -1;
        v = ((unsigned long long)i - S.lo) >> S.shift;
    } else {
        return -1;
    }
    return v < (unsigned long long)SEL_BUCKETS ? (int)v : -1;
}

// histogram of the buckets of every segment in mode 1 / 2: persistent blocks, one shared
// histogram per block (flushed with one global atomic per non-zero bin), or global atomics
// when the segments' histograms do not fit (SMEM = false)
template <bool SMEM>
__global__ void __launch_bounds__(1024) k_top_hist(const double2* __restrict__ zc, int64_t i0, int64_t n, int step,
                                                   const TopRec* __restrict__ recs, const int* __restrict__ roff,
                                                   const SelSeg* __restrict__ sel, int nseg,
                                                   unsigned int* __restrict__ hist)
{
    extern __shared__ unsigned int shist[];
    if (SMEM) {
        for (int j = threadIdx.x; j < nseg * SEL_BUCKETS; j += blockDim.x) shist[j] = 0;
        __syncthreads();
    }
    for (int64_t i = i0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double2 v = zc[i];
        const uint32_t seg = top_segment(v.x, v.y, (uint32_t)i, step, recs, roff);
        const SelSeg S = sel[seg];
        if (S.mode != 1 && S.mode != 2) continue;
        const int b = sel_bucket(S, orderable((step & 1) ? v.y : v.x), (uint32_t)i);
        if (b < 0) continue;
        if (SMEM)
            atomicAdd(&shist[seg * SEL_BUCKETS + b], 1u);
        else
            atomicAdd(&hist[(int64_t)seg * SEL_BUCKETS + b], 1u);
    }
    if (SMEM) {
        __syncthreads();
        for (int j = threadIdx.x; j < nseg * SEL_BUCKETS; j += blockDim.x)
            if (shist[j]) atomicAdd(&hist[j], shist[j]);
    }
}

// the points of bucket 0 of every segment in mode 3 / 4: {key, idx} appended per segment
__global__ void k_top_cand(const double2* __restrict__ zc, int64_t i0, int64_t n, int step,
                           const TopRec* __restrict__ recs, const int* __restrict__ roff, const SelSeg* __restrict__ sel,
                           const int64_t* __restrict__ coff, unsigned int* __restrict__ ccnt, TopRec* __restrict__ cand)
{
    const int64_t i = i0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double2 v = zc[i];
    const uint32_t seg = top_segment(v.x, v.y, (uint32_t)i, step, recs, roff);
    const SelSeg S = sel[seg];
    if (S.mode != 3 && S.mode != 4) return;
    const unsigned long long k = orderable((step & 1) ? v.y : v.x);
    if (sel_bucket(S, k, (uint32_t)i) != 0) return;
    const unsigned int at = atomicAdd(&ccnt[seg], 1u);
    TopRec r;
    r.key = k;
    r.idx = (uint32_t)i;
    r.pad = 0;
    cand[coff[seg] + at] = r;
}

// level-k box of every point, and per level-k box the min / max orderable coordinates
// (shared-memory reduction per block, one global atomic per block and box)
__global__ void __launch_bounds__(256) k_top_box(const double2* __restrict__ zc, int64_t n, int steps,
                                                 const TopRec* __restrict__ recs, const int* __restrict__ roff,
                                                 int nbk, uint32_t* __restrict__ boxk,
                                                 unsigned long long* __restrict__ bb)   // [4][nbk]
{
    __shared__ unsigned long long sb[4][256];
    for (int j = threadIdx.x; j < 4 * nbk; j += 256) sb[j / nbk][j % nbk] = (j / nbk) & 1 ? 0ull : ~0ull;
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        const double2 v = zc[i];
        const uint32_t b = top_segment(v.x, v.y, (uint32_t)i, steps, recs, roff);
        boxk[i] = b;
        const unsigned long long kx = orderable(v.x), ky = orderable(v.y);
        atomicMin(&sb[0][b], kx);
        atomicMax(&sb[1][b], kx);
        atomicMin(&sb[2][b], ky);
        atomicMax(&sb[3][b], ky);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < nbk; j += 256) {
        if (sb[0][j] != ~0ull) {
            atomicMin(&bb[j], sb[0][j]);
            atomicMax(&bb[nbk + j], sb[1][j]);
            atomicMin(&bb[2 * nbk + j], sb[2][j]);
            atomicMax(&bb[3 * nbk + j], sb[3][j]);
        }
    }
}

// discs of levels 0..k from the level-k boxes' bounds (a box's bounds are the union of its
// descendants'); bounds of each level-k box also as the presort's key range (Bounds)
__global__ void k_top_discs(const unsigned long long* __restrict__ bb, int k, double* __restrict__ cx,
                            double* __restrict__ cy, double* __restrict__ r, Bounds* __restrict__ bnds)
{
    const int nbk = 1 << (2 * k);
    int g = 0;                                        // global box id over levels 0..k
    for (int l = 0; l <= k; ++l) {
        const int nb = 1 << (2 * l), span = 1 << (2 * (k - l));
        for (int b = threadIdx.x; b < nb; b += blockDim.x) {
            unsigned long long a = ~0ull, c = 0, d = ~0ull, e = 0;
            for (int q = b * span; q < (b + 1) * span; ++q) {
                a = min(a, bb[q]);
                c = max(c, bb[nbk + q]);
                d = min(d, bb[2 * nbk + q]);
                e = max(e, bb[3 * nbk + q]);
            }
            cx[g + b] = __dmul_rn(0.5, __dadd_rn(from_orderable(a), from_orderable(c)));
            cy[g + b] = __dmul_rn(0.5, __dadd_rn(from_orderable(d), from_orderable(e)));
            r[g + b] = 0.0;
            if (l == k) {
                bnds[b].xmin = a;
                bnds[b].xmax = c;
                bnds[b].ymin = d;
                bnds[b].ymax = e;
                bnds[b].bad = 0;
            }
        }
        g += nb;
    }
}

struct BoxIs {
    const uint32_t* boxk;
    uint32_t b;
    __device__ __forceinline__ bool operator()(const uint32_t& i) const { return boxk[i] == b; }
};

// offsets of level 0
__global__ void k_root_off(uint32_t* __restrict__ O, uint32_t n)
{
    O[0] = 0;
    O[1] = n;
}

// offsets of half-level l+1/2 (H) and level l+1 (C) from level l (O), DESIGN R5:
// a box of size s splits into x-halves (ceil(s/2), floor(s/2)), each into (ceil, floor).
__global__ void k_child_off(const uint32_t* __restrict__ O, int64_t nb, uint32_t* __restrict__ H,
                            uint32_t* __restrict__ C)
{
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    uint32_t s = O[b], sz = O[b + 1] - s;
    uint32_t h0 = sz - sz / 2, h1 = sz / 2;
    H[2 * b] = s;
    H[2 * b + 1] = s + h0;
    C[4 * b] = s;
    C[4 * b + 1] = s + (h0 - h0 / 2);
    C[4 * b + 2] = s + h0;
    C[4 * b + 3] = s + h0 + (h1 - h1 / 2);
    if (b == nb - 1) {
        H[2 * nb] = O[nb];
        C[4 * nb] = O[nb];
    }
}

// largest p in [lo, hi) with O[p] <= k  (O ascending, O[lo] <= k)
__device__ __forceinline__ uint32_t seg_search(const uint32_t* __restrict__ O, uint32_t lo, uint32_t hi, uint32_t k)
{
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (O[mid] <= k) lo = mid;
        else hi = mid;
    }
    return lo;
}

// Per parent segment p in [p0, p1) (threads q < np): the number of its high-side
// records (a function of the offsets) and the rank of its first high record on the
// split axis (the split value; ~0 if the high side is empty).  Per partition tile
// (threads q < ntiles): the segment of its first position (binary search).
__global__ void k_seg_prep(const uint32_t* __restrict__ par_off, const uint32_t* __restrict__ sub_off,
                           const uint2* __restrict__ split_list, int axis, int64_t p0, int64_t np, uint32_t k0,
                           int64_t ntiles, int tile_shift, uint32_t* __restrict__ hs, uint32_t* __restrict__ split,
                           uint32_t* __restrict__ tile_seg)
{
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q < np) {
        const int64_t p = p0 + q;
        const uint32_t pe = par_off[p + 1], sp = sub_off[2 * p + 1];
        hs[q] = pe - sp;
        uint32_t v = 0xFFFFFFFFu;
        if (sp < pe) {
            const uint2 r = split_list[sp];
            v = axis ? r.y : r.x;
        }
        split[q] = v;
    }
    if (q < ntiles) {
        const uint32_t k = k0 + ((uint32_t)q << tile_shift);
        int64_t lo = p0, hi = p0 + np;                 // largest p with par_off[p] <= k
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (par_off[mid] <= k) lo = mid;
            else hi = mid;
        }
        tile_seg[q] = (uint32_t)(lo - p0);
    }
}

// One split step over the positions of the parent segments [p0, p1), in one pass:
//   flag  = record is on the high side of its parent segment p, i.e. its rank on the
//           split axis >= split[p];
//   G(k)  = high records before position k in the range, from a block scan plus a
//           decoupled look-back across tiles (tiles in launch order);
//   dst   = stable position inside p: high -> sub_off[2p+1] + (G(k) - Gp[p]),
//           low -> k - (G(k) - Gp[p]), Gp[p] = highs before segment p (a scan of the
//           high sizes, a function of the offsets only).
// The tile's segments (from tile_seg, no search in global memory) and their table
// (start, first high position, Gp, split rank) are staged in shared memory; each record
// finds its segment by binary search there.
#ifndef FMM2D_PARTITION_TWO_PASS
#define FMM2D_PARTITION_TWO_PASS 0
#endif
#ifndef FMM2D_PART_PI
#define FMM2D_PART_PI 8
#endif
#ifndef FMM2D_PART_PT
#define FMM2D_PART_PT 256
#endif
// 1: the tile's records are regrouped in shared memory (lows, then highs, each in order)
// and written with consecutive threads on consecutive destinations; 0: each thread
// writes its own records (8-record stride across a warp)
#ifndef FMM2D_PART_MINB
#define FMM2D_PART_MINB 5             // 48 registers, 5 tiles per SM (measured best at C5)
#endif
#ifndef FMM2D_PART_STAGED_OUT
#define FMM2D_PART_STAGED_OUT 1
#endif
#ifndef FMM2D_PART_TMA
#define FMM2D_PART_TMA 1              // the tile staged by one cp.async.bulk (TMA) + mbarrier
#endif
constexpr int PT = FMM2D_PART_PT, PI = FMM2D_PART_PI, PTILE = PT * PI;
constexpr int PTILE_SHIFT = (PTILE == 1024) ? 10 : (PTILE == 2048) ? 11 : (PTILE == 4096) ? 12 : 13;
static_assert(PTILE == (1 << PTILE_SHIFT), "tile size");
constexpr int SEGMAX = 512;                          // larger tile spans: segment search in global memory
constexpr uint64_t ST_AGG = 1ull << 62, ST_PRE = 2ull << 62, ST_MASK = 3ull << 62;

struct SplitArgs {
    const uint2* list;          // partitioned list (read)
    const uint32_t* par_off;    // parent segment offsets
    const uint32_t* sub_off;    // child offsets: children of p are 2p, 2p+1
    const uint32_t* Gp;         // [p - p0] highs before segment p
    const uint32_t* split;      // [p - p0] split rank
    const uint32_t* tile_seg;   // [tile] segment (relative to p0) of the tile's first position
    uint2* out;
    unsigned long long* tstate;
    uint32_t* tile_cnt;         // two-pass mode: per tile high count (pass 1) / exclusive prefix (pass 2)
    uint32_t p0, p1;            // parent segments of the range
    uint32_t k0, k1;            // positions of the range (= par_off[p0], par_off[p1])
    uint32_t ntiles;
    int axis;                   // 0: compare rx, 1: compare ry
};

// MODE 0: one pass with the decoupled look-back; MODE 1: count pass (tile high counts);
// MODE 2: scatter pass with the tiles' exclusive prefix (a CUB scan of the counts).
template <int MODE>
__global__ void __launch_bounds__(PT, FMM2D_PART_MINB) k_partition(SplitArgs A)
{
    typedef cub::BlockScan<uint32_t, PT> Scan;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ uint32_t s_prefix;
#if FMM2D_PART_TMA
    // the tile by one bulk asynchronous copy (TMA) from the 16-byte-aligned record at or
    // before its start (stage0 = the tile's first record)
    __shared__ __align__(16) uint2 stage_buf[PTILE + 2];
    __shared__ __align__(8) unsigned long long sbar;
#else
    __shared__ __align__(16) uint2 stage[PTILE];
#endif
    __shared__ uint32_t s_off[SEGMAX + 1], s_hi[SEGMAX], s_gp[SEGMAX], s_split[SEGMAX];
#if FMM2D_PART_STAGED_OUT
    __shared__ uint32_t s_dst[PTILE];
#endif
    const int tid = threadIdx.x;
    const uint32_t tile = blockIdx.x;
    const uint32_t kt = A.k0 + tile * (uint32_t)PTILE;
    const int nrec = (int)min((uint32_t)PTILE, A.k1 - kt);
    const uint32_t qlo = A.tile_seg[tile];                                   // relative to p0
    const uint32_t qhi = (tile + 1 < A.ntiles) ? A.tile_seg[tile + 1] : (A.p1 - A.p0 - 1);
    const int nseg = (int)(qhi - qlo + 1);
    const bool small = nseg <= SEGMAX;
#if FMM2D_PART_TMA
    // (the list may be a virtual base: alignment from the address, not the index)
    const uint32_t ka = kt - (uint32_t)((reinterpret_cast<uintptr_t>(A.list + kt) >> 3) & 1u);   // 16-byte aligned
    const uint32_t nb = (kt + nrec - ka) & ~1u;                  // records copied (even, in range)
    uint2* stage = stage_buf + (kt - ka);
    if (tid == 32 && ((kt + nrec - ka) & 1u)) stage[nrec - 1] = A.list[kt + nrec - 1];   // odd tail
    const uint32_t sbar_s = (uint32_t)__cvta_generic_to_shared(&sbar);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar_s) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar_s), "r"(nb * 8u) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"((uint32_t)__cvta_generic_to_shared(stage_buf)), "l"(A.list + ka), "r"(nb * 8u),
                     "r"(sbar_s) : "memory");
    }
#else
    {   // stage the tile with coalesced 16-byte loads
        const uint4* g = reinterpret_cast<const uint4*>(A.list + kt);
        uint4* sv = reinterpret_cast<uint4*>(stage);
        const int nvec = nrec / 2;
        if ((kt & 1u) == 0) {
            for (int v = tid; v < nvec; v += PT) sv[v] = g[v];
            if (tid == 0 && (nrec & 1)) stage[nrec - 1] = A.list[kt + nrec - 1];
        } else {
            for (int v = tid; v < nrec; v += PT) stage[v] = A.list[kt + v];
        }
    }
#endif
    if (small) {
        for (int j = tid; j < nseg; j += PT) {
            const uint32_t q = qlo + j, p = A.p0 + q;
            s_off[j] = A.par_off[p];
            s_hi[j] = A.sub_off[2 * p + 1];
            s_gp[j] = A.Gp[q];
            s_split[j] = A.split[q];
            if (j == nseg - 1) s_off[nseg] = A.par_off[p + 1];
        }
    }
    __syncthreads();
#if FMM2D_PART_TMA
    {
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(sbar_s) : "memory");
    }
#endif
    uint2 r[PI];
    uint32_t seg[PI], f[PI];
    uint32_t cnt = 0;
    const int i0 = tid * PI;
    uint32_t sj = 0;
    if (i0 < nrec) {
        // first item: binary search in the tile's segment table, then walk forward
        const uint32_t k = kt + i0;
        if (small) {
            uint32_t lo = 0, hi = (uint32_t)nseg;
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (s_off[mid] <= k) lo = mid;
                else hi = mid;
            }
            sj = lo;
        } else {
            uint32_t lo = A.p0 + qlo, hi = A.p0 + qhi + 1;
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (A.par_off[mid] <= k) lo = mid;
                else hi = mid;
            }
            sj = lo - A.p0;                                                  // relative to p0
        }
    }
#pragma unroll
    for (int u = 0; u < PI; ++u) {
        f[u] = 0;
        seg[u] = 0;
        if (i0 + u < nrec) {
            const uint32_t k = kt + i0 + u;
            uint32_t sv;
            if (small) {
                while (k >= s_off[sj + 1]) ++sj;
                sv = s_split[sj];
            } else {
                while (k >= A.par_off[A.p0 + sj + 1]) ++sj;
                sv = A.split[sj];
            }
            r[u] = stage[i0 + u];
            seg[u] = sj;
            const uint32_t rank = A.axis ? r[u].y : r[u].x;
            f[u] = (rank >= sv) ? 1u : 0u;
        }
        cnt += f[u];
    }
    uint32_t excl, agg;
    Scan(scan_tmp).ExclusiveSum(cnt, excl, agg);
    if (MODE == 1) {
        if (tid == 0) A.tile_cnt[tile] = agg;
        return;
    }
    if (MODE == 2) {
        if (tid == 0) s_prefix = A.tile_cnt[tile];
    } else if (tid < 32) {       // decoupled look-back (warp 0)
        uint32_t prefix = 0;
        if (tile == 0) {
            if (tid == 0) atomicExch(&A.tstate[0], ST_PRE | agg);
        } else {
            if (tid == 0) atomicExch(&A.tstate[tile], ST_AGG | agg);
            int64_t j = (int64_t)tile - 1 - tid;
            for (;;) {
                unsigned long long s = 0;
                if (j >= 0) {
                    do {
                        s = *((volatile unsigned long long*)&A.tstate[j]);
                    } while ((s & ST_MASK) == 0);
                } else {
                    s = ST_PRE;                     // before tile 0: inclusive prefix 0
                }
                const unsigned pre = __ballot_sync(0xffffffffu, (s & ST_MASK) == ST_PRE);
                const int first = pre ? __ffs(pre) - 1 : 32;    // nearest tile with a prefix
                uint32_t v = (tid <= first) ? (uint32_t)(s & ~ST_MASK) : 0u;
                for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                prefix += v;
                if (pre) break;
                j -= 32;
            }
            if (tid == 0) atomicExch(&A.tstate[tile], ST_PRE | (prefix + agg));
        }
        if (tid == 0) s_prefix = prefix;
    }
    __syncthreads();
    uint32_t g = s_prefix + excl;             // G(k) for the first item of this thread
#if FMM2D_PART_STAGED_OUT
    // every thread holds its records in registers (stage is free): lows at their rank
    // among the tile's lows, highs after them at their rank among the tile's highs
    uint32_t hl = excl;                       // highs before the item inside the tile
    const uint32_t nlow = (uint32_t)nrec - agg;
#endif
#pragma unroll
    for (int u = 0; u < PI; ++u) {
        if (i0 + u < nrec) {
            const uint32_t k = kt + i0 + u;
            const uint32_t j = seg[u];
            uint32_t gp, hstart;
            if (small) {
                gp = s_gp[j];
                hstart = s_hi[j];
            } else {
                gp = A.Gp[j];
                hstart = A.sub_off[2 * (A.p0 + j) + 1];
            }
            const uint32_t hb = g - gp;       // highs before k inside its segment
            const uint32_t dst = f[u] ? hstart + hb : k - hb;
#if FMM2D_PART_STAGED_OUT
            const uint32_t loc = f[u] ? nlow + hl : (uint32_t)(i0 + u) - hl;
            stage[loc] = r[u];
            s_dst[loc] = dst;
            hl += f[u];
#else
            A.out[dst] = r[u];
#endif
        }
        g += f[u];
    }
#if FMM2D_PART_STAGED_OUT
    __syncthreads();
    for (int v = tid; v < nrec; v += PT) A.out[s_dst[v]] = stage[v];
#endif
}

// The deepest levels in shared memory: once a box holds at most LMAX points, one CTA
// takes it (both of its sorted lists) and performs every remaining split step and the
// bounding boxes of every level below it on chip, then writes its final y-list (the
// leaf order) back in place.  The step is the same stable segmented partition as
// k_partition: one block-wide scan of the high flags, "highs before k inside its
// segment" = scan - Gp[segment] (Gp from the offsets), segments found by binary search
// in the box's local offsets.
constexpr int LT = 512, LI = 4, LMAX = LT * LI;      // 2048 points per box
constexpr int LLEV = 4;                              // at most 4 levels on chip
constexpr int LSEG = 1 << (2 * LLEV - 1);            // half-level segments of the last step (128)

struct LocalArgs {
    uint2* yl;                                       // y-list (in: level l0 grouping, out: leaf order)
    const uint2* xl;                                 // x-list (level l0 grouping)
    const uint32_t* boff;
    int64_t obase[FMM2D_MAXL + 1];
    int64_t hbase[FMM2D_MAXL + 1];
    int l0, L;
    int64_t b0;                                      // first box (level l0) of the launch
    const uint64_t* vx;
    const uint64_t* vy;
    const double2* zc;
    double* cx[FMM2D_MAXL + 1];
    double* cy[FMM2D_MAXL + 1];
    double* r[FMM2D_MAXL + 1];
};

struct LocalSmem {
    uint2 buf[3][LMAX + 2];                          // (+2: a TMA load may start one record early)
    uint32_t segs[2 * LSEG + 1];                     // segment starts (local positions)
    uint32_t subs[4 * LSEG + 1];                     // sub-segment starts
    uint32_t split[2 * LSEG], gp[2 * LSEG];
};

__device__ __forceinline__ uint32_t local_seg(const uint32_t* __restrict__ O, int nseg, uint32_t k)
{
    int lo = 0, hi = nseg;                           // largest j < nseg with O[j] <= k
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (O[mid] <= k) lo = mid;
        else hi = mid;
    }
    return (uint32_t)lo;
}

#ifndef FMM2D_LOCAL_TMA
#define FMM2D_LOCAL_TMA 1                 // k_tree_local: both lists by cp.async.bulk (TMA)
#endif
#ifndef FMM2D_LOCAL_MINB
#define FMM2D_LOCAL_MINB 3
#endif
__global__ void __launch_bounds__(LT, FMM2D_LOCAL_MINB) k_tree_local(LocalArgs A)
{
    extern __shared__ __align__(16) unsigned char lsm[];
    LocalSmem& S = *reinterpret_cast<LocalSmem*>(lsm);
    typedef cub::BlockScan<uint32_t, LT> Scan;
    __shared__ typename Scan::TempStorage scan_tmp;
    const int tid = threadIdx.x;
    const int64_t b = A.b0 + blockIdx.x;
    const uint32_t* O0 = A.boff + A.obase[A.l0];
    const uint32_t s0 = O0[b];
    const int n = (int)(O0[b + 1] - s0);
    uint2* X = S.buf[0];
    uint2* Y = S.buf[1];
    uint2* T = S.buf[2];
#if FMM2D_LOCAL_TMA
    {   // both lists by two bulk asynchronous copies (TMA) from 16-byte-aligned starts
        __shared__ __align__(8) unsigned long long lbar;
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&lbar);
        const uint32_t mx = (uint32_t)((reinterpret_cast<uintptr_t>(A.xl + s0) >> 3) & 1u);
        const uint32_t my = (uint32_t)((reinterpret_cast<uintptr_t>(A.yl + s0) >> 3) & 1u);
        const uint32_t nbx = ((uint32_t)n + mx) & ~1u, nby = ((uint32_t)n + my) & ~1u;
        X = S.buf[0] + mx;
        Y = S.buf[1] + my;
        if (tid == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((nbx + nby) * 8u)
                         : "memory");
            if (nbx)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"((uint32_t)__cvta_generic_to_shared(S.buf[0])), "l"(A.xl + s0 - mx), "r"(nbx * 8u),
                             "r"(bar) : "memory");
            if (nby)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"((uint32_t)__cvta_generic_to_shared(S.buf[1])), "l"(A.yl + s0 - my), "r"(nby * 8u),
                             "r"(bar) : "memory");
        }
        if (tid == 32 && (((uint32_t)n + mx) & 1u)) X[n - 1] = A.xl[s0 + n - 1];    // odd tails
        if (tid == 64 && (((uint32_t)n + my) & 1u)) Y[n - 1] = A.yl[s0 + n - 1];
        __syncthreads();                              // (mbarrier init before the waits; tails)
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(bar) : "memory");
    }
#else
    for (int k = tid; k < n; k += LT) {
        X[k] = A.xl[s0 + k];
        Y[k] = A.yl[s0 + k];
    }
#endif
    for (int l = A.l0; l < A.L; ++l) {
        const int64_t nb = (int64_t)1 << (2 * (l - A.l0));         // level-l boxes of this CTA
        const int64_t gb = b * nb;                                  // first one, level-local id
        const uint32_t* O = A.boff + A.obase[l] + gb;
        const uint32_t* H = A.boff + A.hbase[l] + 2 * gb;
        const uint32_t* C = A.boff + A.obase[l + 1] + 4 * gb;
        // two steps: x-split of Y (segments: boxes, subs: halves, split on rx from X),
        // then y-split of X (segments: halves, subs: children, split on ry from Y)
        for (int step = 0; step < 2; ++step) {
            const int nseg = (int)(step == 0 ? nb : 2 * nb);
            const uint32_t* SO = step == 0 ? O : H;
            const uint32_t* SU = step == 0 ? H : C;
            uint2* L_ = step == 0 ? Y : X;                         // list partitioned
            const uint2* SL = step == 0 ? X : Y;                   // list giving the split ranks
            __syncthreads();
            for (int j = tid; j <= nseg; j += LT) S.segs[j] = SO[j] - s0;
            for (int j = tid; j <= 2 * nseg; j += LT) S.subs[j] = SU[j] - s0;
            __syncthreads();
            if (tid < 32) {                                        // split ranks and Gp (warp 0)
                uint32_t run = 0;
                for (int j0 = 0; j0 < nseg; j0 += 32) {
                    const int j = j0 + tid;
                    uint32_t hsz = 0;
                    if (j < nseg) {
                        const uint32_t sp = S.subs[2 * j + 1], pe = S.segs[j + 1];
                        hsz = pe - sp;
                        const uint2 rr = (sp < pe) ? SL[sp] : make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
                        S.split[j] = step == 0 ? rr.x : rr.y;
                    }
                    uint32_t incl = hsz;
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                        if (tid >= o) incl += v;
                    }
                    if (j < nseg) S.gp[j] = run + incl - hsz;
                    run += __shfl_sync(0xffffffffu, incl, 31);
                }
            }
            __syncthreads();
            uint2 rec[LI];
            uint32_t f[LI], sg[LI], cnt = 0;
#pragma unroll
            for (int u = 0; u < LI; ++u) {
                const int k = tid * LI + u;
                f[u] = 0;
                sg[u] = 0;
                if (k < n) {
                    rec[u] = L_[k];
                    sg[u] = local_seg(S.segs, nseg, (uint32_t)k);
                    const uint32_t rank = step == 0 ? rec[u].x : rec[u].y;
                    f[u] = rank >= S.split[sg[u]] ? 1u : 0u;
                }
                cnt += f[u];
            }
            uint32_t excl;
            Scan(scan_tmp).ExclusiveSum(cnt, excl);
#pragma unroll
            for (int u = 0; u < LI; ++u) {
                const int k = tid * LI + u;
                if (k < n) {
                    const uint32_t hb = excl - S.gp[sg[u]];
                    const uint32_t dst = f[u] ? S.subs[2 * sg[u] + 1] + hb : (uint32_t)k - hb;
                    T[dst] = rec[u];
                }
                excl += f[u];
            }
            __syncthreads();
            if (step == 0) { uint2* t = Y; Y = T; T = t; }
            else           { uint2* t = X; X = T; T = t; }
        }
        // bounding boxes of the level-(l+1) boxes (S.subs holds their local starts)
        for (int c = tid; c < 4 * nb; c += LT) {
            const uint32_t s = S.subs[c], e = S.subs[c + 1];
            const double xmin = A.zc[(uint32_t)A.vx[X[s].x]].x, xmax = A.zc[(uint32_t)A.vx[X[e - 1].x]].x;
            const double ymin = A.zc[(uint32_t)(A.vy[Y[s].y] >> 32)].y;
            const double ymax = A.zc[(uint32_t)(A.vy[Y[e - 1].y] >> 32)].y;
            const int64_t gbx = 4 * gb + c;
            A.cx[l + 1][gbx] = __dmul_rn(0.5, __dadd_rn(xmin, xmax));
            A.cy[l + 1][gbx] = __dmul_rn(0.5, __dadd_rn(ymin, ymax));
            A.r[l + 1][gbx] = 0.0;
        }
    }
    __syncthreads();
    for (int k = tid; k < n; k += LT) A.yl[s0 + k] = Y[k];
}

// A2 (part 1): tight bounding box from the segment endpoints of both sorted lists;
// centre = 0.5 (min + max) (DESIGN R8).  Radius reset for part 2.
// (x rank -> idx: low half of vx; y rank -> idx: high half of vy)
__global__ void k_bbox(const uint2* __restrict__ xl, const uint2* __restrict__ yl, const uint64_t* __restrict__ vx,
                       const uint64_t* __restrict__ vy, const double2* __restrict__ zc,
                       const uint32_t* __restrict__ off, int64_t b0, int64_t b1, double* __restrict__ cx,
                       double* __restrict__ cy, double* __restrict__ r)
{
    const int64_t b = b0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= b1) return;
    const uint32_t s = off[b], e = off[b + 1];
    const double xmin = zc[(uint32_t)vx[xl[s].x]].x, xmax = zc[(uint32_t)vx[xl[e - 1].x]].x;
    const double ymin = zc[(uint32_t)(vy[yl[s].y] >> 32)].y, ymax = zc[(uint32_t)(vy[yl[e - 1].y] >> 32)].y;
    cx[b] = __dmul_rn(0.5, __dadd_rn(xmin, xmax));
    cy[b] = __dmul_rn(0.5, __dadd_rn(ymin, ymax));
    r[b] = 0.0;
}

// Final order + A2 (part 2) for every level in one pass.  The final y-list is the
// leaf order (leaves ascending, (y, idx) inside, R13): write perm and the source
// rows, then r(box) = exact max distance (correctly rounded sqrt, no FMA) for the
// box of every level containing the point.  A block takes FIN_C chunks of FIN_T
// consecutive positions (the gathers of all chunks in flight together).  Levels at which
// the block's whole range lies in one box: per-thread then per-warp max, the warps'
// maxima of all such levels combined after ONE barrier, one atomicMax per level and
// block; other levels: a segmented warp max per chunk, one atomicMax per run (on the
// bit pattern: non-negative doubles order like their uint64 bits).
#ifndef FMM2D_FIN_C
#define FMM2D_FIN_C 4
#endif
constexpr int FIN_T = 256, FIN_C = FMM2D_FIN_C, FIN_B = FIN_T * FIN_C;
struct RadArgs {
    const double* cx[FMM2D_MAXL + 1];
    const double* cy[FMM2D_MAXL + 1];
    double* r[FMM2D_MAXL + 1];
};
__global__ void __launch_bounds__(FIN_T) k_finish(const uint2* __restrict__ yl, const uint64_t* __restrict__ vy,
                                                  const double2* __restrict__ zc,
                                                  uint32_t k0, uint32_t k1, int L, const uint32_t* __restrict__ offL,
                                                  uint32_t lf0, uint32_t lf1, uint32_t* __restrict__ perm,
                                                  double4* __restrict__ src, RadArgs A)
{
    __shared__ uint32_t s_lo, s_hi;
    __shared__ double wmax[FMM2D_MAXL + 1][FIN_T / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t kb = k0 + blockIdx.x * FIN_B;
    const int nvalid = (int)min((uint32_t)FIN_B, k1 - kb);
    if (tid == 0) {
        const uint32_t lo = seg_search(offL, lf0, lf1, kb);
        s_lo = lo;
        s_hi = seg_search(offL, lo, lf1, kb + nvalid - 1) + 1;
    }
    uint32_t ry[FIN_C], idx[FIN_C], leaf[FIN_C];
    double x[FIN_C], y[FIN_C];
#pragma unroll
    for (int c = 0; c < FIN_C; ++c) {
        const int i = c * FIN_T + tid;
        ry[c] = i < nvalid ? yl[kb + i].y : 0u;
    }
#pragma unroll
    for (int c = 0; c < FIN_C; ++c) idx[c] = (c * FIN_T + tid < nvalid) ? (uint32_t)(vy[ry[c]] >> 32) : 0u;
#pragma unroll
    for (int c = 0; c < FIN_C; ++c) {
        x[c] = y[c] = 0.0;
        if (c * FIN_T + tid < nvalid) {
            const double2 zz = zc[idx[c]];
            x[c] = zz.x;
            y[c] = zz.y;
        }
    }
    __syncthreads();
    const uint32_t l0 = s_lo, l1 = s_hi - 1;
#pragma unroll
    for (int c = 0; c < FIN_C; ++c) {
        const int i = c * FIN_T + tid;
        leaf[c] = 0;
        if (i < nvalid) {
            const uint32_t k = kb + i;
            leaf[c] = seg_search(offL, l0, l1 + 1, k);
            perm[k] = idx[c];
            src[k] = make_double4(x[c], y[c], 0.0, 0.0);
        }
    }
    for (int l = L; l >= 0; --l) {
        const int sh = 2 * (L - l);
        if ((l0 >> sh) == (l1 >> sh)) {                   // block-uniform
            const uint32_t box = l0 >> sh;
            const double ccx = A.cx[l][box], ccy = A.cy[l][box];
            double d = 0.0;
#pragma unroll
            for (int c = 0; c < FIN_C; ++c)
                if (c * FIN_T + tid < nvalid) d = fmax(d, rn_dist2(x[c], y[c], ccx, ccy));   // squared
            for (int o = 16; o; o >>= 1) d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
            if (lane == 0) wmax[l][warp] = d;
        } else {
#pragma unroll
            for (int c = 0; c < FIN_C; ++c) {
                const bool valid = c * FIN_T + tid < nvalid;
                const uint32_t box = leaf[c] >> sh;
                double d = 0.0;
                if (valid) d = rn_dist2(x[c], y[c], A.cx[l][box], A.cy[l][box]);
                // segmented max over lanes [lane, end of my box's run) (runs are contiguous)
                for (int o = 1; o < 32; o <<= 1) {
                    const double dv = __shfl_down_sync(0xffffffffu, d, o);
                    const uint32_t bv = __shfl_down_sync(0xffffffffu, box, o);
                    const bool vv = __shfl_down_sync(0xffffffffu, valid ? 1 : 0, o) != 0;
                    if (lane + o < 32 && vv && bv == box) d = fmax(d, dv);
                }
                const uint32_t bprev = __shfl_up_sync(0xffffffffu, box, 1);
                if (valid && (lane == 0 || bprev != box))
                    atomicMax((unsigned long long*)(A.r[l] + box), (unsigned long long)__double_as_longlong(d));
            }
        }
    }
    __syncthreads();
    if (tid <= L) {
        const int l = tid, sh = 2 * (L - l);
        if ((l0 >> sh) == (l1 >> sh)) {
            double m = wmax[l][0];
            for (int w = 1; w < FIN_T / 32; ++w) m = fmax(m, wmax[l][w]);
            atomicMax((unsigned long long*)(A.r[l] + (l0 >> sh)), (unsigned long long)__double_as_longlong(m));
        }
    }
}

// r = sqrt_rn(max squared distance); an empty box (midpoint tree) keeps r = -1
__global__ void k_sqrt(double* __restrict__ r, int64_t nb)
{
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b < nb && r[b] >= 0.0) r[b] = __dsqrt_rn(r[b]);
}

// ---------------------------------------------------------------- midpoint tree (DESIGN R26)
// The uniform baseline of Fig. 4: the bounding square split at geometric midpoints to
// depth L (x then y, children 4b + 2 xside + yside), empty boxes allowed.  A point's leaf
// is (floor((x - x0) S), floor((y - y0) S)) clamped, S = 2^L / side (host division),
// interleaved x-high-first; leaves ascending, input order inside (stable sort).
__device__ __forceinline__ uint32_t spread15(uint32_t v)
{
    v &= 0x7FFFu;
    v = (v | (v << 8)) & 0x00FF00FFu;
    v = (v | (v << 4)) & 0x0F0F0F0Fu;
    v = (v | (v << 2)) & 0x33333333u;
    v = (v | (v << 1)) & 0x55555555u;
    return v;
}

__global__ void k_mid_keys(const double2* __restrict__ zc, int64_t n, double x0, double y0, double S, int L,
                           uint32_t* __restrict__ key, uint32_t* __restrict__ iota)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double2 v = zc[i];
    const int64_t cmax = ((int64_t)1 << L) - 1;
    int64_t ix = (int64_t)floor(__dmul_rn(__dsub_rn(v.x, x0), S));
    int64_t iy = (int64_t)floor(__dmul_rn(__dsub_rn(v.y, y0), S));
    ix = min(max(ix, (int64_t)0), cmax);
    iy = min(max(iy, (int64_t)0), cmax);
    key[i] = (spread15((uint32_t)ix) << 1) | spread15((uint32_t)iy);
    iota[i] = (uint32_t)i;
}

// leaf offsets: off[b] = first sorted position with key >= b
__global__ void k_mid_leaf_off(const uint32_t* __restrict__ skey, int64_t n, int64_t nl, uint32_t* __restrict__ off)
{
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b > nl) return;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)skey[mid] < b) lo = mid + 1;
        else hi = mid;
    }
    off[b] = (uint32_t)lo;
}

__global__ void k_mid_level_off(const uint32_t* __restrict__ offL, int shift, int64_t nb, uint32_t* __restrict__ off)
{
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b <= nb) off[b] = offL[b << shift];
}

__global__ void k_mid_rows(const uint32_t* __restrict__ sidx, const double2* __restrict__ zc, int64_t n,
                           uint32_t* __restrict__ perm, double4* __restrict__ src)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint32_t i = sidx[k];
    const double2 v = zc[i];
    perm[k] = i;
    src[k] = make_double4(v.x, v.y, 0.0, 0.0);
}

// per box of every level: min / max of the orderable coordinate bits (segmented warp
// reductions over the leaf-ordered points, one atomic per run)
__global__ void __launch_bounds__(256) k_mid_bounds(const uint32_t* __restrict__ skey, const double4* __restrict__ src,
                                                    int64_t n, int L, const int64_t* __restrict__ gbase,
                                                    unsigned long long* __restrict__ bb)   // [4][nbox_total]
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool valid = k < n;
    uint32_t leaf = valid ? skey[k] : 0u;
    double4 v = valid ? src[k] : make_double4(0, 0, 0, 0);
    const unsigned long long ox = orderable(v.x), oy = orderable(v.y);
    const int64_t nbt = gbase[L + 1];
    for (int l = L; l >= 0; --l) {
        const uint32_t box = leaf >> (2 * (L - l));
        unsigned long long a = ox, b = ox, c = oy, d = oy;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long a2 = __shfl_down_sync(0xffffffffu, a, o), b2 = __shfl_down_sync(0xffffffffu, b, o);
            const unsigned long long c2 = __shfl_down_sync(0xffffffffu, c, o), d2 = __shfl_down_sync(0xffffffffu, d, o);
            const uint32_t bv = __shfl_down_sync(0xffffffffu, box, o);
            const bool vv = __shfl_down_sync(0xffffffffu, valid ? 1 : 0, o) != 0;
            if (lane + o < 32 && vv && bv == box) {
                a = min(a, a2);
                b = max(b, b2);
                c = min(c, c2);
                d = max(d, d2);
            }
        }
        const uint32_t bprev = __shfl_up_sync(0xffffffffu, box, 1);
        if (valid && (lane == 0 || bprev != box)) {
            const int64_t g = gbase[l] + box;
            atomicMin(&bb[g], a);
            atomicMax(&bb[nbt + g], b);
            atomicMin(&bb[2 * nbt + g], c);
            atomicMax(&bb[3 * nbt + g], d);
        }
    }
}

__global__ void k_mid_centres(const unsigned long long* __restrict__ bb, int64_t nbt, double* __restrict__ cx,
                              double* __restrict__ cy, double* __restrict__ r)
{
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= nbt) return;
    if (bb[g] == ~0ull) {                                     // no point: empty box
        cx[g] = 0.0;
        cy[g] = 0.0;
        r[g] = -1.0;
        return;
    }
    cx[g] = __dmul_rn(0.5, __dadd_rn(from_orderable(bb[g]), from_orderable(bb[nbt + g])));
    cy[g] = __dmul_rn(0.5, __dadd_rn(from_orderable(bb[2 * nbt + g]), from_orderable(bb[3 * nbt + g])));
    r[g] = 0.0;
}

// squared radii of every level (the sqrt follows in finish_radii)
__global__ void __launch_bounds__(256) k_mid_radius(const uint32_t* __restrict__ skey, const double4* __restrict__ src,
                                                    int64_t n, int L, const int64_t* __restrict__ gbase,
                                                    const double* __restrict__ cx, const double* __restrict__ cy,
                                                    double* __restrict__ r)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool valid = k < n;
    const uint32_t leaf = valid ? skey[k] : 0u;
    const double4 v = valid ? src[k] : make_double4(0, 0, 0, 0);
    for (int l = L; l >= 0; --l) {
        const uint32_t box = leaf >> (2 * (L - l));
        const int64_t g = gbase[l] + box;
        double d = valid ? rn_dist2(v.x, v.y, cx[g], cy[g]) : 0.0;
        for (int o = 1; o < 32; o <<= 1) {
            const double dv = __shfl_down_sync(0xffffffffu, d, o);
            const uint32_t bv = __shfl_down_sync(0xffffffffu, box, o);
            const bool vv = __shfl_down_sync(0xffffffffu, valid ? 1 : 0, o) != 0;
            if (lane + o < 32 && vv && bv == box) d = fmax(d, dv);
        }
        const uint32_t bprev = __shfl_up_sync(0xffffffffu, box, 1);
        if (valid && (lane == 0 || bprev != box))
            atomicMax((unsigned long long*)(r + g), (unsigned long long)__double_as_longlong(d));
    }
}

__global__ void k_mid_leaf_stats(const uint32_t* __restrict__ offL, int64_t nl, unsigned int* __restrict__ mm)
{
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nl) return;
    const unsigned int sz = offL[b + 1] - offL[b];
    atomicMax(&mm[0], sz);
    atomicMin(&mm[1], sz);
}

inline unsigned grid_for(int64_t n, int bs) { return (unsigned)((n + bs - 1) / bs); }

}  // namespace

// r = sqrt_rn(max squared distance) for every box of the plan (after the cross-rank
// max of the replicated top levels in a sharded build)
int finish_radii(fmm2d_plan* P)
{
    k_sqrt<<<grid_for(P->nbox_total, 256), 256, 0, P->stream>>>(P->r, P->nbox_total);
    fmm2d::note_launch();
    FMM2D_CUDA_TRY(cudaGetLastError());
    return 0;
}

static int build_tree_midpoint(fmm2d_plan* P, const double2* z);

// Partitioned build, levels 0..k (DESIGN 8): split records by selection, level-k boxes and
// their discs (replicated, identical on every rank), then the presort of each own level-k
// box's points (ascending input index, ranks offset by the box's first position).
template <class Presort>
static int top_levels_sharded(fmm2d_plan* P, const double2* zc, const Bounds& hb_all, const std::vector<int64_t>& hbase,
                              Presort& presort)
{
    cudaStream_t st = P->stream;
    const int64_t n = P->n;
    const int k = P->kpart;
    const int nsteps = 2 * k;
    const int BS = 256;
    // segments of each step and their sizes (pure functions of n: host offsets)
    std::vector<int> roff(nsteps + 1, 0);
    std::vector<int64_t> seg_n, seg_hi;             // per step, per segment: size, first high index
    auto bstart = [&](int l, int64_t b) -> int64_t {     // start of box b of level l (b = 4^l: n)
        return (b >= ((int64_t)1 << (2 * l))) ? n : box_start_host(n, l, b);
    };
    for (int s = 0; s < nsteps; ++s) {
        const int l = s / 2;
        const int nseg = (s & 1) ? 2 << (2 * l) : 1 << (2 * l);
        roff[s + 1] = roff[s] + nseg;
        for (int g = 0; g < nseg; ++g) {
            int64_t a, b;
            if (s & 1) {                                // half g of level-l box g/2
                const int64_t bs = bstart(l, g / 2), be = bstart(l, g / 2 + 1);
                const int64_t sz = be - bs, h0 = sz - sz / 2;
                a = (g & 1) ? bs + h0 : bs;
                b = (g & 1) ? be : bs + h0;
            } else {
                a = bstart(l, g);
                b = bstart(l, g + 1);
            }
            seg_n.push_back(b - a);
            seg_hi.push_back((b - a) - (b - a) / 2);     // index of the first high record
        }
    }
    TopRec* d_recs = nullptr;
    int* d_roff = nullptr;
    unsigned int *hist = nullptr, *ccnt = nullptr;
    SelSeg* sel = nullptr;
    int64_t* coff = nullptr;
    TopRec* cand = nullptr;
    uint32_t *boxk = nullptr, *sub = nullptr;
    int64_t* d_nsel = nullptr;
    unsigned long long* bb = nullptr;
    Bounds* bnds = nullptr;
    void* scratch = nullptr;
    std::vector<void*> tmp;
    auto talloc = [&](void** p, size_t b) -> int {
        if (fmm2d::pool_malloc((void**)p, b ? b : 16, st) != cudaSuccess) return FMM2D_ENOMEM;
        tmp.push_back(*p);
        return 0;
    };
    const int maxseg = 2 << (2 * (k - 1));
    const int nbk = 1 << (2 * k);
    // Sliced selection: with NCCL every rank counts (histogram passes) and collects
    // (candidate pass) over its own slice [n r / R, n (r+1) / R) of the input only; the
    // histograms are summed by an all-reduce and the candidate blocks all-gathered, so every
    // rank sees the global counts and candidates.  Loopback with FMM2D_SEL_SLICED=1 runs the
    // same slices one after the other into the same buffers (the emulation the tests use);
    // otherwise one pass over all points.
    const int R = P->nranks, myrank = P->rank;
    const bool nccl = shard_has_comm(P);
    const bool emul = !nccl && std::getenv("FMM2D_SEL_SLICED") != nullptr;
    const int nblk = (nccl || emul) ? R : 1;              // candidate blocks (one per slice)
    auto slice_lo = [&](int r) { return n * r / R; };
    PhaseTrace tr(st);
    tr.mark("start");
    auto body = [&]() -> int {
        FMM2D_TRY(talloc((void**)&d_recs, sizeof(TopRec) * std::max(1, roff[nsteps])));
        FMM2D_TRY(talloc((void**)&d_roff, sizeof(int) * (nsteps + 1)));
        FMM2D_TRY(talloc((void**)&hist, sizeof(unsigned int) * SEL_BUCKETS * maxseg));
        FMM2D_TRY(talloc((void**)&sel, sizeof(SelSeg) * maxseg));
        FMM2D_TRY(talloc((void**)&cand, sizeof(TopRec) * SEL_COLLECT * maxseg * nblk));
        FMM2D_TRY(talloc((void**)&ccnt, sizeof(unsigned int) * maxseg * nblk));
        FMM2D_TRY(talloc((void**)&coff, sizeof(int64_t) * maxseg));
        FMM2D_TRY(talloc((void**)&boxk, sizeof(uint32_t) * n));
        FMM2D_TRY(talloc((void**)&sub, sizeof(uint32_t) * n));
        FMM2D_TRY(talloc((void**)&d_nsel, sizeof(int64_t)));
        FMM2D_TRY(talloc((void**)&bb, sizeof(unsigned long long) * 4 * nbk));
        FMM2D_TRY(talloc((void**)&bnds, sizeof(Bounds) * nbk));
        FMM2D_CUDA_TRY(cudaMemcpyAsync(d_roff, roff.data(), sizeof(int) * (nsteps + 1), cudaMemcpyHostToDevice, st));
        std::vector<TopRec> h_recs(std::max(1, roff[nsteps]));
        std::vector<unsigned int> h_hist((size_t)SEL_BUCKETS * maxseg);
        std::vector<SelSeg> hs(maxseg);
        std::vector<int64_t> want(maxseg), hcoff(maxseg), ccap(maxseg);
        auto shift_for = [](unsigned long long range) {
            int s = 0;
            while (s < 63 && (range >> s) >= (unsigned long long)SEL_BUCKETS) ++s;
            return s;
        };
        int64_t si = 0;                                  // index into seg_n / seg_hi
        for (int s = 0; s < nsteps; ++s) {
            const int nseg = roff[s + 1] - roff[s];
            const unsigned long long gmin = (s & 1) ? hb_all.ymin : hb_all.xmin;
            const unsigned long long gmax = (s & 1) ? hb_all.ymax : hb_all.xmax;
            int nhist = 0;
            for (int g = 0; g < nseg; ++g) {
                want[g] = seg_hi[si + g];
                hs[g].lo = gmin;
                hs[g].keyfix = 0;
                hs[g].shift = shift_for(gmax - gmin);
                if (want[g] >= seg_n[si + g]) {          // no high record: every point is low
                    hs[g].mode = 0;
                    h_recs[roff[s] + g] = TopRec{~0ull, ~0u, 0u};
                } else {
                    hs[g].mode = 1;
                    ++nhist;
                }
            }
            // narrow each segment's range until its bucket holds at most SEL_COLLECT points
            int npass = 0;
            while (nhist > 0) {
                ++npass;
                FMM2D_CUDA_TRY(cudaMemcpyAsync(sel, hs.data(), sizeof(SelSeg) * nseg, cudaMemcpyHostToDevice, st));
                FMM2D_CUDA_TRY(cudaMemsetAsync(hist, 0, sizeof(unsigned int) * SEL_BUCKETS * nseg, st));
                auto hist_pass = [&](int64_t a, int64_t b) -> int {
                    if (b <= a) return 0;
                    if (nseg <= SEL_SMEM_SEGS) {
                        const int sm = nseg * SEL_BUCKETS * 4;
                        FMM2D_CUDA_TRY(cudaFuncSetAttribute(k_top_hist<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
                        const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>(148, (b - a + 1023) / 1024));
                        k_top_hist<true><<<g, 1024, sm, st>>>(zc, a, b, s, d_recs, d_roff, sel, nseg, hist);
                    } else {
                        k_top_hist<false><<<grid_for(b - a, BS), BS, 0, st>>>(zc, a, b, s, d_recs, d_roff, sel, nseg, hist);
                    }
                    note_launch();
                    return 0;
                };
                if (nccl) {
                    FMM2D_TRY(hist_pass(slice_lo(myrank), slice_lo(myrank + 1)));
                    FMM2D_TRY(shard_allreduce_sum_u32(P, hist, (size_t)SEL_BUCKETS * nseg));
                } else if (emul) {
                    for (int r = 0; r < R; ++r) FMM2D_TRY(hist_pass(slice_lo(r), slice_lo(r + 1)));
                } else {
                    FMM2D_TRY(hist_pass(0, n));
                }
                FMM2D_CUDA_TRY(cudaMemcpyAsync(h_hist.data(), hist, sizeof(unsigned int) * SEL_BUCKETS * nseg,
                                               cudaMemcpyDeviceToHost, st));
                FMM2D_CUDA_TRY(cudaStreamSynchronize(st));
                nhist = 0;
                for (int g = 0; g < nseg; ++g) {
                    SelSeg& S = hs[g];
                    if (S.mode != 1 && S.mode != 2) continue;
                    const unsigned int* H = h_hist.data() + (size_t)g * SEL_BUCKETS;
                    int64_t acc = 0;
                    int b = 0;
                    for (; b < SEL_BUCKETS; ++b) {
                        if (acc + H[b] > want[g]) break;
                        acc += H[b];
                    }
                    if (b == SEL_BUCKETS) return FMM2D_ECUDA;     // inconsistent counts (cannot happen)
                    want[g] -= acc;
                    S.lo += (unsigned long long)b << S.shift;
                    if (H[b] <= (unsigned)SEL_COLLECT) {
                        S.mode += 2;                              // collect bucket 0 of [lo, ...)
                        ccap[g] = H[b];
                    } else if (S.shift > SEL_BITS) {
                        S.shift -= SEL_BITS;
                        ++nhist;
                    } else if (S.shift > 0) {
                        S.shift = 0;
                        ++nhist;
                    } else if (S.mode == 1) {                     // one key, many points: select by idx
                        S.mode = 2;
                        S.keyfix = S.lo;
                        S.lo = 0;
                        S.shift = shift_for((unsigned long long)n);
                        ++nhist;
                    } else {
                        return FMM2D_ECUDA;                       // one (key, idx) counted twice
                    }
                }
            }
            int64_t ctot = 0;
            int ncol = 0;
            for (int g = 0; g < nseg; ++g) {
                hcoff[g] = ctot;
                if (hs[g].mode >= 3) {
                    ctot += ccap[g];
                    ++ncol;
                }
            }
            if (ncol > 0) {
                // candidate block r (slice r, or everything when not sliced): entries of
                // segment g at [blk r + coff_g, + count[r][g])
                const int64_t bstride = (int64_t)SEL_COLLECT * maxseg;
                FMM2D_CUDA_TRY(cudaMemcpyAsync(sel, hs.data(), sizeof(SelSeg) * nseg, cudaMemcpyHostToDevice, st));
                FMM2D_CUDA_TRY(cudaMemcpyAsync(coff, hcoff.data(), sizeof(int64_t) * nseg, cudaMemcpyHostToDevice, st));
                FMM2D_CUDA_TRY(cudaMemsetAsync(ccnt, 0, sizeof(unsigned int) * maxseg * nblk, st));
                auto cand_pass = [&](int blk, int64_t a, int64_t b) {
                    if (b > a)
                        k_top_cand<<<grid_for(b - a, BS), BS, 0, st>>>(zc, a, b, s, d_recs, d_roff, sel, coff,
                                                                       ccnt + (int64_t)blk * maxseg,
                                                                       cand + (int64_t)blk * bstride);
                    note_launch();
                };
                if (nccl) {
                    cand_pass(myrank, slice_lo(myrank), slice_lo(myrank + 1));
                    FMM2D_TRY(shard_allgather_inplace(P, cand, sizeof(TopRec) * bstride));
                    FMM2D_TRY(shard_allgather_inplace(P, ccnt, sizeof(unsigned int) * maxseg));
                } else if (emul) {
                    for (int r = 0; r < R; ++r) cand_pass(r, slice_lo(r), slice_lo(r + 1));
                } else {
                    cand_pass(0, 0, n);
                }
                FMM2D_CUDA_TRY(cudaGetLastError());
                std::vector<TopRec> hc((size_t)std::max<int64_t>(ctot, 1) * nblk);
                std::vector<unsigned int> hcnt((size_t)maxseg * nblk);
                for (int r = 0; r < nblk; ++r)
                    FMM2D_CUDA_TRY(cudaMemcpyAsync(hc.data() + (size_t)r * std::max<int64_t>(ctot, 1),
                                                   cand + (int64_t)r * bstride, sizeof(TopRec) * ctot,
                                                   cudaMemcpyDeviceToHost, st));
                FMM2D_CUDA_TRY(cudaMemcpyAsync(hcnt.data(), ccnt, sizeof(unsigned int) * maxseg * nblk,
                                               cudaMemcpyDeviceToHost, st));
                FMM2D_CUDA_TRY(cudaStreamSynchronize(st));
                std::vector<TopRec> seg;
                for (int g = 0; g < nseg; ++g) {
                    if (hs[g].mode < 3) continue;
                    seg.clear();
                    for (int r = 0; r < nblk; ++r) {
                        const TopRec* b0 = hc.data() + (size_t)r * std::max<int64_t>(ctot, 1) + hcoff[g];
                        seg.insert(seg.end(), b0, b0 + hcnt[(size_t)r * maxseg + g]);
                    }
                    if ((int64_t)seg.size() != ccap[g]) return FMM2D_ECUDA;   // counts and candidates disagree
                    std::sort(seg.begin(), seg.end(), [](const TopRec& a, const TopRec& b) {
                        return a.key < b.key || (a.key == b.key && a.idx < b.idx);
                    });
                    h_recs[roff[s] + g] = seg[want[g]];
                }
            }
            FMM2D_CUDA_TRY(cudaMemcpyAsync(d_recs + roff[s], h_recs.data() + roff[s], sizeof(TopRec) * nseg,
                                           cudaMemcpyHostToDevice, st));
            si += nseg;
            tr.mark("select step " + std::to_string(s) + " (" + std::to_string(npass) + " passes)");
        }
        // level-k boxes of all points, their bounds; discs of levels 0..k
        std::vector<unsigned long long> hbb(4 * (size_t)nbk);
        for (int j = 0; j < nbk; ++j) {
            hbb[j] = ~0ull;
            hbb[nbk + j] = 0;
            hbb[2 * nbk + j] = ~0ull;
            hbb[3 * nbk + j] = 0;
        }
        FMM2D_CUDA_TRY(cudaMemcpyAsync(bb, hbb.data(), 8 * hbb.size(), cudaMemcpyHostToDevice, st));
        k_top_box<<<grid_for(n, 256), 256, 0, st>>>(zc, n, nsteps, d_recs, d_roff, nbk, boxk, bb);
        note_launch();
        k_top_discs<<<1, 256, 0, st>>>(bb, k, P->cx, P->cy, P->r, bnds);
        note_launch();
        FMM2D_CUDA_TRY(cudaGetLastError());
        tr.mark("level-k boxes");
        // presort of each own level-k box (its points in ascending input index)
        size_t sb = 0;
        thrust::counting_iterator<uint32_t> it(0);
        cub::DeviceSelect::If(nullptr, sb, it, sub, d_nsel, (int64_t)n, BoxIs{boxk, 0u}, st);
        FMM2D_TRY(talloc(&scratch, sb));
        for (int64_t R = P->own_lo(k); R < P->own_hi(k); ++R) {
            size_t s2 = sb;
            FMM2D_CUDA_TRY(cub::DeviceSelect::If(scratch, s2, it, sub, d_nsel, (int64_t)n, BoxIs{boxk, (uint32_t)R}, st));
            const int64_t r0 = bstart(k, R), r1 = bstart(k, R + 1);
            FMM2D_TRY(presort(sub, r1 - r0, (uint32_t)r0, bnds + R));
            tr.mark("presort box " + std::to_string(R));
        }
        return 0;
    };
    const int rc = body();
    for (void* p : tmp) cudaFreeAsync(p, st);
    return rc;
}

int build_tree(fmm2d_plan* P, const double2* z)
{
    if (P->flags & FMM2D_MIDPOINT) return build_tree_midpoint(P, z);
    const int64_t n = P->n;
    const int L = P->L;
    cudaStream_t st = P->stream;
    const int BS = 256;

    // ---- offsets: level l at obase[l] (4^l + 1), half-level l+1/2 at hbase[l] (2 4^l + 1)
    P->obase.assign(L + 1, 0);
    std::vector<int64_t> hbase(L, 0);
    int64_t tot = 0;
    for (int l = 0; l <= L; ++l) { P->obase[l] = tot; tot += nboxes(l) + 1; }
    for (int l = 0; l < L; ++l) { hbase[l] = tot; tot += 2 * nboxes(l) + 1; }
    FMM2D_TRY(dev_alloc(P, (void**)&P->boff, sizeof(uint32_t) * tot));
    k_root_off<<<1, 1, 0, st>>>(P->boff + P->obase[0], (uint32_t)n);
    fmm2d::note_launch();
    for (int l = 0; l < L; ++l) {
        k_child_off<<<grid_for(nboxes(l), BS), BS, 0, st>>>(P->boff + P->obase[l], nboxes(l), P->boff + hbase[l],
                                                           P->boff + P->obase[l + 1]);
        fmm2d::note_launch();
    }
    // leaf sizes are floor(n / 4^L) or ceil(n / 4^L) (DESIGN R5)
    P->stats.min_leaf = (int)(n / nboxes(L));
    P->stats.max_leaf = (int)((n + nboxes(L) - 1) / nboxes(L));

    // ---- scratch
    double2* zc;
    uint32_t *k32a, *k32b, *u32a, *u32b, *hs, *Gp, *spl, *tseg, *tcnt, *tpre;
    uint64_t *vx, *vy, *v64a, *k64a, *k64b;
    uint2 *xl, *yl, *tmp;
    Bounds* bnd;
    int* ovf;
    unsigned long long* tstate;
    void* scratch = nullptr;
    size_t s32 = 0, s64 = 0, sd = 0, scan_bytes = 0;
    const int64_t npmax = (L > 0) ? 2 * nboxes(L - 1) : 1;        // parents of the widest step
    // a partitioned build keeps only its own positions [pos0, pos1) in the position-indexed
    // arrays (virtual bases), and presorts one own level-k box at a time (at most mmax points)
    const int64_t nown = (int64_t)P->pos1 - (int64_t)P->pos0;
    const int64_t mmax = (P->nranks == 1) ? n : (n + nboxes(P->kpart) - 1) / nboxes(P->kpart);
    const int64_t ntiles = (nown + PTILE - 1) / PTILE;
    int nbits = 1;
    while (((int64_t)1 << nbits) < mmax) ++nbits;
    cub::DeviceRadixSort::SortPairs(nullptr, s32, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint64_t*)nullptr,
                                    (uint64_t*)nullptr, (int)mmax, 0, 32, st);
    cub::DeviceRadixSort::SortPairs(nullptr, s64, (uint64_t*)nullptr, (uint64_t*)nullptr, (uint64_t*)nullptr,
                                    (uint64_t*)nullptr, (int)mmax, 0, 64, st);
    cub::DeviceRadixSort::SortPairs(nullptr, sd, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (uint32_t*)nullptr, (int)mmax, 0, nbits, st);
    cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (int)std::max<int64_t>(npmax, ntiles), st);
    const size_t cub_bytes = std::max(std::max(s32, s64), std::max(sd, scan_bytes));
    std::vector<void*> tmp_ptrs;
    auto talloc = [&](void** p, size_t b) -> int {
        cudaError_t e = fmm2d::pool_malloc((void**)p, b ? b : 16, st);
        if (e != cudaSuccess) return FMM2D_ENOMEM;
        tmp_ptrs.push_back(*p);
        return 0;
    };
    auto tfree = [&]() {
        for (void* p : tmp_ptrs) cudaFreeAsync(p, st);
        tmp_ptrs.clear();
    };
    int rc = 0;
    do {
        if ((rc = talloc((void**)&zc, 16 * n))) break;
        if ((rc = talloc((void**)&k32a, 4 * mmax))) break;
        if ((rc = talloc((void**)&k32b, 4 * mmax))) break;
        if ((rc = talloc((void**)&u32a, 4 * n))) break;       // also x ranks by input index (64-bit y path)
        if ((rc = talloc((void**)&u32b, 4 * mmax))) break;
        if ((rc = talloc((void**)&v64a, 8 * mmax))) break;
        if ((rc = talloc((void**)&vx, 8 * nown))) break;
        if ((rc = talloc((void**)&vy, 8 * nown))) break;
        if ((rc = talloc((void**)&hs, 4 * npmax))) break;
        if ((rc = talloc((void**)&Gp, 4 * npmax))) break;
        if ((rc = talloc((void**)&spl, 4 * npmax))) break;
        if ((rc = talloc((void**)&tseg, 4 * (ntiles + 1)))) break;
        if ((rc = talloc((void**)&tcnt, 4 * (ntiles + 1)))) break;
        if ((rc = talloc((void**)&tpre, 4 * (ntiles + 1)))) break;
        if ((rc = talloc((void**)&tstate, 8 * ntiles))) break;
        if ((rc = talloc((void**)&xl, sizeof(uint2) * nown))) break;
        if ((rc = talloc((void**)&yl, sizeof(uint2) * nown))) break;
        if ((rc = talloc((void**)&tmp, sizeof(uint2) * nown))) break;
        if ((rc = talloc((void**)&bnd, sizeof(Bounds)))) break;
        if ((rc = talloc((void**)&ovf, 2 * sizeof(int)))) break;
        if ((rc = talloc(&scratch, cub_bytes))) break;
    } while (0);
    if (rc) { tfree(); return rc; }
    vx -= P->pos0;                          // position-indexed: virtual bases
    vy -= P->pos0;
    xl -= P->pos0;
    yl -= P->pos0;
    tmp -= P->pos0;
    k64a = k64b = nullptr;                  // 64-bit keys of the fallback: allocated when needed

    Bounds hall;                            // host copy of the global ranges (partitioned top levels)
    PhaseTrace trb(st);
    trb.mark("tree start");
    auto body = [&]() -> int {
        // ---- A0: validate, canonical coordinates, ranges
        {
            Bounds h;
            h.xmin = h.ymin = ~0ull;
            h.xmax = h.ymax = 0;
            h.bad = 0;
            FMM2D_CUDA_TRY(cudaMemcpyAsync(bnd, &h, sizeof(h), cudaMemcpyHostToDevice, st));
            const unsigned g = (unsigned)std::min<int64_t>(grid_for(n, CT), 148 * 8);
            k_canon<<<g, CT, 0, st>>>(z, n, zc, bnd);
            fmm2d::note_launch();
            FMM2D_CUDA_TRY(cudaGetLastError());
            FMM2D_CUDA_TRY(cudaMemcpyAsync(&h, bnd, sizeof(h), cudaMemcpyDeviceToHost, st));
            FMM2D_CUDA_TRY(cudaStreamSynchronize(st));
            if (h.bad) return FMM2D_ENONFINITE;
            hall = h;
            trb.mark("canon");
        }
        // ---- presort: the (x, idx) order, then the (y, idx) order, as ranks (DESIGN 6.1),
        // of m points (all, or one level-k box of a partitioned build: sub, roff, its bounds)
        const bool force64 = (P->flags & FMM2D_TREE_KEY64) != 0;
        auto presort = [&](const uint32_t* sub, int64_t m, uint32_t roff, const Bounds* bm) -> int {
            if (m == 0) return 0;
            int mbits = 1;
            while (((int64_t)1 << mbits) < m) ++mbits;
            uint64_t* vxm = vx + roff;
            uint64_t* vym = vy + roff;
            int h_ovf[2] = {0, 0};
            FMM2D_CUDA_TRY(cudaMemsetAsync(ovf, 0, 2 * sizeof(int), st));
            size_t sb = cub_bytes;
            if (!force64) {
                // x: stable sort of 32-bit keys, payload {idx, y key}; equal-key runs fixed
                k_keys_x<false><<<grid_for(m, BS), BS, 0, st>>>(zc, sub, m, bm, k32a, nullptr, v64a);
                fmm2d::note_launch();
                FMM2D_CUDA_TRY(cub::DeviceRadixSort::SortPairs(scratch, sb, k32a, k32b, v64a, vxm, (int)m, 0, 32, st));
                k_fix_runs<<<grid_for((m + FR - 1) / FR, BS), BS, 0, st>>>(k32b, m, zc, 0, 0, vxm, ovf);
                fmm2d::note_launch();
                FMM2D_CUDA_TRY(cudaMemcpyAsync(&h_ovf[0], ovf, sizeof(int), cudaMemcpyDeviceToHost, st));
                FMM2D_CUDA_TRY(cudaStreamSynchronize(st));
            }
            uint64_t* k64buf = nullptr;
            if (force64 || h_ovf[0]) {
                // heavy ties in x: full 64-bit orderable keys (ties leave in idx order)
                if (!k64buf) {
                    FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&k64buf, 16 * m, st));
                    k64a = k64buf;
                    k64b = k64buf + m;
                }
                k_keys_x<true><<<grid_for(m, BS), BS, 0, st>>>(zc, sub, m, bm, nullptr, k64a, v64a);
                fmm2d::note_launch();
                sb = cub_bytes;
                FMM2D_CUDA_TRY(cub::DeviceRadixSort::SortPairs(scratch, sb, k64a, k64b, v64a, vxm, (int)m, 0, 64, st));
            }
            if (!force64) {
                // y: input in x order, key = y key, payload {x rank, idx}; runs fixed by (y, idx)
                k_prep_y<<<grid_for(m, BS), BS, 0, st>>>(vxm, m, roff, k32a, v64a);
                fmm2d::note_launch();
                sb = cub_bytes;
                FMM2D_CUDA_TRY(cub::DeviceRadixSort::SortPairs(scratch, sb, k32a, k32b, v64a, vym, (int)m, 0, 32, st));
                k_fix_runs<<<grid_for((m + FR - 1) / FR, BS), BS, 0, st>>>(k32b, m, zc, 1, 32, vym, ovf + 1);
                fmm2d::note_launch();
                FMM2D_CUDA_TRY(cudaMemcpyAsync(&h_ovf[1], ovf + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
                FMM2D_CUDA_TRY(cudaStreamSynchronize(st));
            }
            if (force64 || h_ovf[1]) {
                // heavy ties in y: 64-bit keys over the input in idx order
                if (!k64buf) {
                    FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&k64buf, 16 * m, st));
                    k64a = k64buf;
                    k64b = k64buf + m;
                }
                k_scatter_rx<<<grid_for(m, BS), BS, 0, st>>>(vxm, m, u32a);
                fmm2d::note_launch();
                k_keys_y64<<<grid_for(m, BS), BS, 0, st>>>(zc, sub, u32a, m, roff, k64a, v64a);
                fmm2d::note_launch();
                sb = cub_bytes;
                FMM2D_CUDA_TRY(cub::DeviceRadixSort::SortPairs(scratch, sb, k64a, k64b, v64a, vym, (int)m, 0, 64, st));
            }
            if (k64buf) cudaFreeAsync(k64buf, st);
            FMM2D_CUDA_TRY(cudaGetLastError());
            P->stats.tree_key64 |= (force64 || h_ovf[0] ? 1 : 0) + (force64 || h_ovf[1] ? 2 : 0);
            if (FMM2D_PRESORT_SCATTER == 2) {
                // y-list {rx, ry}; local x ranks bucketed by their top 8 bits, then scattered
                k_make_ylist<<<grid_for(m, BS), BS, 0, st>>>(vym, m, roff, yl + roff, k32a, u32a);
                fmm2d::note_launch();
                sb = cub_bytes;
                FMM2D_CUDA_TRY(cub::DeviceRadixSort::SortPairs(scratch, sb, k32a, k32b, u32a, u32b, (int)m,
                                                               std::max(0, mbits - 8), mbits, st));
                k_scatter_xlist<<<grid_for(m, BS), BS, 0, st>>>(k32b, u32b, m, roff, xl + roff);
                fmm2d::note_launch();
            } else if (FMM2D_PRESORT_SCATTER == 1) {
                // y-list {rx, ry} in y order, and the same records scattered to x order
                k_make_lists<<<grid_for(m, BS), BS, 0, st>>>(vym, m, roff, yl + roff, xl + roff);
                fmm2d::note_launch();
            } else {
                // y-list {rx, k}; the y ranks in x order by one more sort (keys = local x ranks)
                k_make_ylist<<<grid_for(m, BS), BS, 0, st>>>(vym, m, roff, yl + roff, k32a, u32a);
                fmm2d::note_launch();
                sb = cub_bytes;
                FMM2D_CUDA_TRY(cub::DeviceRadixSort::SortPairs(scratch, sb, k32a, k32b, u32a, u32b, (int)m, 0, mbits, st));
                k_make_xlist<<<grid_for(m, BS), BS, 0, st>>>(u32b, m, roff, xl + roff);
                fmm2d::note_launch();
            }
            FMM2D_CUDA_TRY(cudaGetLastError());
            return 0;
        };
        if (P->nranks == 1) {
            FMM2D_TRY(presort(nullptr, n, 0, bnd));
        } else {
            FMM2D_TRY(top_levels_sharded(P, zc, hall, hbase, presort));
        }
        trb.mark("presort / top levels");
        if (P->nranks == 1) {
            k_bbox<<<1, 32, 0, st>>>(xl, yl, vx, vy, zc, P->boff + P->obase[0], 0, 1, P->cx + P->base[0],
                                     P->cy + P->base[0], P->r + P->base[0]);
            fmm2d::note_launch();
        }
        // one split step: partition `list` inside the parent segments (par_off) [p0, p1),
        // positions [k0, k1), into the sub-segments sub_off, comparing ranks on `axis`
        // against `split`
        auto split_step = [&](const uint2* list, const uint2* split, const uint32_t* par_off, const uint32_t* sub_off,
                              int64_t p0, int64_t p1, uint32_t k0, uint32_t k1, int axis, uint2* out) -> int {
            const int64_t np = p1 - p0;
            const int64_t nt = ((int64_t)k1 - k0 + PTILE - 1) / PTILE;
            k_seg_prep<<<grid_for(std::max(np, nt), BS), BS, 0, st>>>(par_off, sub_off, split, axis, p0, np, k0, nt,
                                                                      PTILE_SHIFT, hs, spl, tseg);
            fmm2d::note_launch();
            size_t b2 = cub_bytes;
            FMM2D_CUDA_TRY(cub::DeviceScan::ExclusiveSum(scratch, b2, hs, Gp, (int)np, st));
            SplitArgs A;
            A.list = list;
            A.par_off = par_off;
            A.sub_off = sub_off;
            A.Gp = Gp;
            A.split = spl;
            A.tile_seg = tseg;
            A.out = out;
            A.tstate = tstate;
            A.p0 = (uint32_t)p0;
            A.p1 = (uint32_t)p1;
            A.k0 = k0;
            A.k1 = k1;
            A.axis = axis;
            A.ntiles = (uint32_t)nt;
#if FMM2D_PARTITION_TWO_PASS
            // count pass, scan of the tile counts, scatter pass (no look-back chain)
            A.tile_cnt = tcnt;
            k_partition<1><<<(unsigned)nt, PT, 0, st>>>(A);
            fmm2d::note_launch();
            size_t b3 = cub_bytes;
            FMM2D_CUDA_TRY(cub::DeviceScan::ExclusiveSum(scratch, b3, tcnt, tpre, (int)nt, st));
            A.tile_cnt = tpre;
            k_partition<2><<<(unsigned)nt, PT, 0, st>>>(A);
            fmm2d::note_launch();
#else
            FMM2D_CUDA_TRY(cudaMemsetAsync(tstate, 0, 8 * nt, st));
            k_partition<0><<<(unsigned)nt, PT, 0, st>>>(A);
            fmm2d::note_launch();
#endif
            FMM2D_CUDA_TRY(cudaGetLastError());
            return 0;
        };
        // levels 0..kpart-1: every box (replicated on every rank); levels >= kpart: the
        // rank's own subtrees only (the whole tree on one GPU, kpart = 0)
        // levels l0 .. L-1 on chip (k_tree_local): boxes of at most LMAX points, at most
        // LLEV levels below them; never above the partition level
        int l0 = L;
        for (int l = std::max(P->kpart, L - LLEV); l < L; ++l)
            if ((n + nboxes(l) - 1) / nboxes(l) <= LMAX) { l0 = l; break; }
        if (P->flags & FMM2D_TREE_GLOBAL_ONLY) l0 = L;
        for (int l = (P->nranks > 1 ? P->kpart : 0); l < l0; ++l) {   // partitioned: top levels done by selection
            const uint32_t* O = P->boff + P->obase[l];
            const uint32_t* H = P->boff + hbase[l];
            const uint32_t* C = P->boff + P->obase[l + 1];
            const int64_t b0 = (l < P->kpart) ? 0 : P->own_lo(l), b1 = (l < P->kpart) ? nboxes(l) : P->own_hi(l);
            const uint32_t k0 = (l < P->kpart) ? 0u : P->pos0, k1 = (l < P->kpart) ? (uint32_t)n : P->pos1;
            // x-split: the y-list (grouped by level-l boxes) is partitioned by rx against
            // the x-list's first high record of each box
            FMM2D_TRY(split_step(yl, xl, O, H, b0, b1, k0, k1, 0, tmp));
            std::swap(yl, tmp);
            // y-split of each half: the x-list (grouped by half-level boxes) is partitioned
            // by ry against the y-list's first high record of each half
            FMM2D_TRY(split_step(xl, yl, H, C, 2 * b0, 2 * b1, k0, k1, 1, tmp));
            std::swap(xl, tmp);
            const int64_t c0 = P->box_lo(l + 1), c1 = P->box_hi(l + 1);
            k_bbox<<<grid_for(c1 - c0, BS), BS, 0, st>>>(xl, yl, vx, vy, zc, C, c0, c1, P->cx + P->base[l + 1],
                                                         P->cy + P->base[l + 1], P->r + P->base[l + 1]);
            fmm2d::note_launch();
            FMM2D_CUDA_TRY(cudaGetLastError());
        }
        trb.mark("global split levels");
        if (l0 < L) {
            LocalArgs A;
            A.yl = yl;
            A.xl = xl;
            A.boff = P->boff;
            for (int l = 0; l <= L; ++l) A.obase[l] = P->obase[l];
            for (int l = 0; l < L; ++l) A.hbase[l] = hbase[l];
            A.l0 = l0;
            A.L = L;
            const int64_t b0 = (l0 < P->kpart) ? 0 : P->own_lo(l0), b1 = (l0 < P->kpart) ? nboxes(l0) : P->own_hi(l0);
            A.b0 = b0;
            A.vx = vx;
            A.vy = vy;
            A.zc = zc;
            for (int l = 0; l <= L; ++l) {
                A.cx[l] = P->cx + P->base[l];
                A.cy[l] = P->cy + P->base[l];
                A.r[l] = P->r + P->base[l];
            }
            const int smem = (int)sizeof(LocalSmem);
            FMM2D_CUDA_TRY(cudaFuncSetAttribute(k_tree_local, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            k_tree_local<<<(unsigned)(b1 - b0), LT, smem, st>>>(A);
            fmm2d::note_launch();
            FMM2D_CUDA_TRY(cudaGetLastError());
        }
        // radii of every level from the own positions (squared; a sharded build
        // max-reduces the replicated top levels across ranks before the square root)
        FMM2D_CUDA_TRY(cudaMemsetAsync(P->r, 0, sizeof(double) * P->base[P->kpart + 1], st));
        RadArgs A;
        for (int l = 0; l <= L; ++l) {
            A.cx[l] = P->cx + P->base[l];
            A.cy[l] = P->cy + P->base[l];
            A.r[l] = P->r + P->base[l];
        }
        const uint32_t nown = P->pos1 - P->pos0;
        k_finish<<<grid_for(nown, FIN_B), FIN_T, 0, st>>>(yl, vy, zc, P->pos0, P->pos1, L,
                                                          P->boff + P->obase[L], (uint32_t)P->box_lo(L),
                                                          (uint32_t)P->box_hi(L), P->perm, P->src, A);
        fmm2d::note_launch();
        FMM2D_CUDA_TRY(cudaGetLastError());
        if (P->nranks == 1) FMM2D_TRY(finish_radii(P));
        trb.mark("local levels + finish");
        return 0;
    };
    rc = body();
    tfree();
    return rc;
}

// the midpoint tree (DESIGN R26): keys, one stable sort, offsets by search, discs by
// segmented reductions over the leaf order
static int build_tree_midpoint(fmm2d_plan* P, const double2* z)
{
    const int64_t n = P->n;
    const int L = P->L;
    cudaStream_t st = P->stream;
    const int BS = 256;
    const int64_t nl = nboxes(L), nbt = P->nbox_total;
    P->obase.assign(L + 1, 0);
    int64_t tot = 0;
    for (int l = 0; l <= L; ++l) { P->obase[l] = tot; tot += nboxes(l) + 1; }
    FMM2D_TRY(dev_alloc(P, (void**)&P->boff, sizeof(uint32_t) * tot));
    double2* zc = nullptr;
    uint32_t *key, *skey, *iota, *sidx;
    unsigned long long* bb = nullptr;
    int64_t* gbase = nullptr;
    Bounds* bnd = nullptr;
    unsigned int* mm = nullptr;
    void* scratch = nullptr;
    size_t sb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sb, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (uint32_t*)nullptr, (int)n, 0, std::max(1, 2 * L), st);
    std::vector<void*> tmp;
    auto talloc = [&](void** p, size_t b) -> int {
        if (fmm2d::pool_malloc((void**)p, b ? b : 16, st) != cudaSuccess) return FMM2D_ENOMEM;
        tmp.push_back(*p);
        return 0;
    };
    int rc = 0;
    do {
        if ((rc = talloc((void**)&zc, 16 * n))) break;
        if ((rc = talloc((void**)&key, 4 * n))) break;
        if ((rc = talloc((void**)&skey, 4 * n))) break;
        if ((rc = talloc((void**)&iota, 4 * n))) break;
        if ((rc = talloc((void**)&sidx, 4 * n))) break;
        if ((rc = talloc((void**)&bb, 8 * 4 * nbt))) break;
        if ((rc = talloc((void**)&gbase, 8 * (L + 2)))) break;
        if ((rc = talloc((void**)&bnd, sizeof(Bounds)))) break;
        if ((rc = talloc((void**)&mm, 8))) break;
        if ((rc = talloc(&scratch, sb))) break;
    } while (0);
    auto body = [&]() -> int {
        if (rc) return rc;
        Bounds h;
        h.xmin = h.ymin = ~0ull;
        h.xmax = h.ymax = 0;
        h.bad = 0;
        FMM2D_CUDA_TRY(cudaMemcpyAsync(bnd, &h, sizeof(h), cudaMemcpyHostToDevice, st));
        const unsigned g = (unsigned)std::min<int64_t>(grid_for(n, CT), 148 * 8);
        k_canon<<<g, CT, 0, st>>>(z, n, zc, bnd);
        fmm2d::note_launch();
        FMM2D_CUDA_TRY(cudaMemcpyAsync(&h, bnd, sizeof(h), cudaMemcpyDeviceToHost, st));
        FMM2D_CUDA_TRY(cudaStreamSynchronize(st));
        if (h.bad) return FMM2D_ENONFINITE;
        auto host_from_orderable = [](unsigned long long k) {
            uint64_t u = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
            double d;
            memcpy(&d, &u, 8);
            return d;
        };
        const double x0 = host_from_orderable(h.xmin), x1 = host_from_orderable(h.xmax);
        const double y0 = host_from_orderable(h.ymin), y1 = host_from_orderable(h.ymax);
        double side = std::max(x1 - x0, y1 - y0);
        if (!(side > 0.0)) side = 1.0;
        const double S = std::ldexp(1.0, L) / side;
        k_mid_keys<<<grid_for(n, BS), BS, 0, st>>>(zc, n, x0, y0, S, L, key, iota);
        fmm2d::note_launch();
        size_t s2 = sb;
        FMM2D_CUDA_TRY(cub::DeviceRadixSort::SortPairs(scratch, s2, key, skey, iota, sidx, (int)n, 0,
                                                       std::max(1, 2 * L), st));
        uint32_t* offL = P->boff + P->obase[L];
        k_mid_leaf_off<<<grid_for(nl + 1, BS), BS, 0, st>>>(skey, n, nl, offL);
        fmm2d::note_launch();
        for (int l = 0; l < L; ++l) {
            k_mid_level_off<<<grid_for(nboxes(l) + 1, BS), BS, 0, st>>>(offL, 2 * (L - l), nboxes(l),
                                                                        P->boff + P->obase[l]);
            fmm2d::note_launch();
        }
        k_mid_rows<<<grid_for(n, BS), BS, 0, st>>>(sidx, zc, n, P->perm, P->src);
        fmm2d::note_launch();
        std::vector<int64_t> hb(L + 2);
        for (int l = 0; l <= L + 1; ++l) hb[l] = P->base[l];
        FMM2D_CUDA_TRY(cudaMemcpyAsync(gbase, hb.data(), 8 * (L + 2), cudaMemcpyHostToDevice, st));
        FMM2D_CUDA_TRY(cudaMemsetAsync(bb, 0xFF, 8 * nbt, st));                    // min: ~0
        FMM2D_CUDA_TRY(cudaMemsetAsync(bb + nbt, 0, 8 * nbt, st));                 // max: 0
        FMM2D_CUDA_TRY(cudaMemsetAsync(bb + 2 * nbt, 0xFF, 8 * nbt, st));
        FMM2D_CUDA_TRY(cudaMemsetAsync(bb + 3 * nbt, 0, 8 * nbt, st));
        k_mid_bounds<<<grid_for(n, 256), 256, 0, st>>>(skey, P->src, n, L, gbase, bb);
        fmm2d::note_launch();
        k_mid_centres<<<grid_for(nbt, BS), BS, 0, st>>>(bb, nbt, P->cx, P->cy, P->r);
        fmm2d::note_launch();
        k_mid_radius<<<grid_for(n, 256), 256, 0, st>>>(skey, P->src, n, L, gbase, P->cx, P->cy, P->r);
        fmm2d::note_launch();
        unsigned int hmm[2] = {0u, 0xFFFFFFFFu};
        FMM2D_CUDA_TRY(cudaMemcpyAsync(mm, hmm, 8, cudaMemcpyHostToDevice, st));
        k_mid_leaf_stats<<<grid_for(nl, BS), BS, 0, st>>>(offL, nl, mm);
        fmm2d::note_launch();
        FMM2D_CUDA_TRY(cudaMemcpyAsync(hmm, mm, 8, cudaMemcpyDeviceToHost, st));
        FMM2D_CUDA_TRY(cudaStreamSynchronize(st));
        P->stats.max_leaf = (int)hmm[0];
        P->stats.min_leaf = (int)hmm[1];
        FMM2D_CUDA_TRY(cudaGetLastError());
        if (P->nranks == 1) FMM2D_TRY(finish_radii(P));
        return 0;
    };
    rc = body();
    for (void* p : tmp) cudaFreeAsync(p, st);
    return rc;
}

}  // namespace fmm2d
