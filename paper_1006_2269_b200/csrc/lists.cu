// lists.cu -- A3: connectivity from the theta-criterion.
//
// Paper: "For each box b, the strong connections S(p) of its parent box
// p are examined; all children of a box in S(p) that satisfy the theta-criterion
// with respect to b become weakly coupled to b -- the rest remain strongly coupled.
// This simple rule together with the fact that a box is always strongly connected
// to itself recursively defines the connectivity for the whole tree.  The resulting
// topology is conveniently stored in sparse matrices with sparsity patterns known
// before each level is to be examined."
// Criterion 1: well separated iff R + theta r <= theta d (readings
// R9-R11: d > 0 required, non-strict, no FMA, exact operation order).
//
// GPU formulation: one warp per parent box (its four children share the candidate list:
// the children of the parent's strong list, in ascending order), walked 32 candidates at a
// time; each lane evaluates the predicate against the four children, and ballot/popc
// compaction writes weak and strong entries in candidate order (so lists come out
// ascending, R13) into per-box slots; a scan of the counts and a compaction pass follow.
#include <cub/cub.cuh>

#include "fmm2d_internal.cuh"

namespace fmm2d {

namespace {

__device__ __forceinline__ bool well_separated(double cbx, double cby, double rb, double ccx, double ccy,
                                               double rc, double theta)
{
    double dx = __dsub_rn(cbx, ccx);
    double dy = __dsub_rn(cby, ccy);
    double d = __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
    double R = fmax(rb, rc);
    double r = fmin(rb, rc);
    return (d > 0.0) && (__dadd_rn(R, __dmul_rn(theta, r)) <= __dmul_rn(theta, d));
}

// Parent merge (DESIGN R25; `merge`): a candidate group of four children of q
// (four consecutive lanes) that are ALL weak to b, with Criterion 1 also true for (b, q)
// itself (q's disc at level l-1: pcx, pcy, pr), becomes one cross-level entry q.
// One pass per level: the entries go to per-box slots of a scratch array (capacity
// 4 |S(parent)| per box -- the candidates -- at a closed-form slot start), with the
// counts; k_compact_lists then packs them into the CSR lists after a scan of the counts.
__device__ __forceinline__ int64_t cand_slot(const int64_t* __restrict__ poff, int64_t b)
{
    const int64_t par = b >> 2;
    return 16 * poff[par] + 4 * (b & 3) * (poff[par + 1] - poff[par]);
}

// One warp per box (used where the parents' strong lists are long: one warp per parent would
// serialise four long candidate walks)
__global__ void k_lists_box(int64_t b0, int64_t b1, const double* __restrict__ cx, const double* __restrict__ cy,
                        const double* __restrict__ r, double theta, const int64_t* __restrict__ poff,
                        const uint32_t* __restrict__ pidx, int64_t* __restrict__ wcnt, int64_t* __restrict__ scnt,
                        uint32_t* __restrict__ wtmp, uint32_t* __restrict__ stmp, bool merge,
                        const double* __restrict__ pcx, const double* __restrict__ pcy, const double* __restrict__ pr,
                        int64_t* __restrict__ xcnt, uint32_t* __restrict__ xtmp)
{
    int64_t b = b0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    int lane = threadIdx.x & 31;
    if (b >= b1) return;
    int64_t par = b >> 2;
    int64_t o0 = poff[par];
    int64_t ncand = 4 * (poff[par + 1] - o0);
    double bx = cx[b], by = cy[b], br = r[b];
    int64_t nw = 0, ns = 0, nx = 0;
    if (br < 0.0) ncand = 0;                 // empty box (midpoint tree): no connections
    const int64_t slot = cand_slot(poff, b), xslot = slot / 4;
    unsigned lt = (1u << lane) - 1u;
    for (int64_t t0 = 0; t0 < ncand; t0 += 32) {
        int64_t t = t0 + lane;
        bool valid = t < ncand;
        uint32_t c = 0, q = 0;
        bool ws = false;
        if (valid) {
            q = pidx[o0 + (t >> 2)];
            c = 4u * q + (uint32_t)(t & 3);
            valid = r[c] >= 0.0;                 // empty candidates (midpoint tree) take no part
            ws = valid && (c != (uint32_t)b) && well_separated(bx, by, br, cx[c], cy[c], r[c], theta);
        }
        unsigned wm = __ballot_sync(0xffffffffu, valid && ws);
        bool merged = false;                        // my group of four merges into its parent q
        if (merge) {
            const bool all4 = ((wm >> (lane & ~3)) & 0xFu) == 0xFu;
            bool mq = false;
            if (all4 && (lane & 3) == 0) mq = well_separated(bx, by, br, pcx[q], pcy[q], pr[q], theta);
            merged = __shfl_sync(0xffffffffu, mq ? 1 : 0, lane & ~3) != 0;
            wm = __ballot_sync(0xffffffffu, valid && ws && !merged);
        }
        unsigned sm = __ballot_sync(0xffffffffu, valid && !ws);
        unsigned xm = __ballot_sync(0xffffffffu, merged && (lane & 3) == 0);
        if (valid) {
            if (merged) {
                if ((lane & 3) == 0) xtmp[xslot + nx + __popc(xm & lt)] = q;
            } else if (ws) {
                wtmp[slot + nw + __popc(wm & lt)] = c;
            } else {
                stmp[slot + ns + __popc(sm & lt)] = c;
            }
        }
        nw += __popc(wm);
        ns += __popc(sm);
        nx += __popc(xm);
    }
    if (lane == 0) {
        wcnt[b] = nw;
        scnt[b] = ns;
        if (merge) xcnt[b] = nx;
    }
}

// One THREAD per box (FMM2D_LISTS_THREAD; short parent lists): the box walks its candidates
// (the children of its parent's strong list, in order) itself -- siblings sit in adjacent
// threads, so the candidates' discs are shared through L1 -- and writes its slots in the
// same order as the ballot compactions of the warp forms (bit-identical lists).
#ifndef FMM2D_LISTS_THREAD
#define FMM2D_LISTS_THREAD 1
#endif
__global__ void __launch_bounds__(256) k_lists_t(int64_t b0, int64_t b1, const double* __restrict__ cx,
                                                 const double* __restrict__ cy, const double* __restrict__ r,
                                                 double theta, const int64_t* __restrict__ poff,
                                                 const uint32_t* __restrict__ pidx, int64_t* __restrict__ wcnt,
                                                 int64_t* __restrict__ scnt, uint32_t* __restrict__ wtmp,
                                                 uint32_t* __restrict__ stmp, bool merge,
                                                 const double* __restrict__ pcx, const double* __restrict__ pcy,
                                                 const double* __restrict__ pr, int64_t* __restrict__ xcnt,
                                                 uint32_t* __restrict__ xtmp)
{
    const int64_t b = b0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= b1) return;
    const int64_t par = b >> 2;
    const int64_t o0 = poff[par], nq = poff[par + 1] - o0;
    const double bx = cx[b], by = cy[b], br = r[b];
    const int64_t slot = cand_slot(poff, b), xslot = slot / 4;
    int64_t nw = 0, ns = 0, nx = 0;
    if (br >= 0.0) {                                // empty box (midpoint tree): no connections
        for (int64_t k = 0; k < nq; ++k) {
            const uint32_t q = pidx[o0 + k];
            bool valid[4], ws[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t c = 4u * q + (uint32_t)j;
                valid[j] = r[c] >= 0.0;             // empty candidates (midpoint tree) take no part
                ws[j] = valid[j] && (c != (uint32_t)b) && well_separated(bx, by, br, cx[c], cy[c], r[c], theta);
            }
            if (merge && ws[0] && ws[1] && ws[2] && ws[3] && well_separated(bx, by, br, pcx[q], pcy[q], pr[q], theta)) {
                xtmp[xslot + nx++] = q;
                continue;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (!valid[j]) continue;
                const uint32_t c = 4u * q + (uint32_t)j;
                if (ws[j]) wtmp[slot + nw++] = c;
                else stmp[slot + ns++] = c;
            }
        }
    }
    wcnt[b] = nw;
    scnt[b] = ns;
    if (merge) xcnt[b] = nx;
}

#ifndef FMM2D_LISTS_MINB
#define FMM2D_LISTS_MINB 3            // 80 registers: 3 blocks of 256 per SM (measured best at C5)
#endif
// One warp per PARENT: its four children share the candidate list (the children of the
// parent's strong list), so each candidate's disc is loaded once and tested against the four
// children; per child the ballots and slots are those of the box-per-warp formulation.
__global__ void __launch_bounds__(256, FMM2D_LISTS_MINB) k_lists(int64_t b0, int64_t b1, const double* __restrict__ cx, const double* __restrict__ cy,
                        const double* __restrict__ r, double theta, const int64_t* __restrict__ poff,
                        const uint32_t* __restrict__ pidx, int64_t* __restrict__ wcnt, int64_t* __restrict__ scnt,
                        uint32_t* __restrict__ wtmp, uint32_t* __restrict__ stmp, bool merge,
                        const double* __restrict__ pcx, const double* __restrict__ pcy, const double* __restrict__ pr,
                        int64_t* __restrict__ xcnt, uint32_t* __restrict__ xtmp)
{
    const int64_t par = (b0 >> 2) + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (4 * par >= b1) return;
    const int64_t o0 = poff[par];
    const int64_t ncand = 4 * (poff[par + 1] - o0);
    double bx[4], by[4], br[4];
    bool live[4], conn[4];
    int64_t slot[4], nw[4], ns[4], nx[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int64_t b = 4 * par + j;
        live[j] = b >= b0 && b < b1;
        bx[j] = by[j] = br[j] = 0.0;
        if (live[j]) {
            bx[j] = cx[b];
            by[j] = cy[b];
            br[j] = r[b];
        }
        conn[j] = live[j] && br[j] >= 0.0;          // empty box (midpoint tree): no connections
        slot[j] = cand_slot(poff, b);
        nw[j] = ns[j] = nx[j] = 0;
    }
    const unsigned lt = (1u << lane) - 1u;
    for (int64_t t0 = 0; t0 < ncand; t0 += 32) {
        const int64_t t = t0 + lane;
        bool valid = t < ncand;
        uint32_t c = 0, q = 0;
        double ccx = 0.0, ccy = 0.0, crr = 0.0, qx = 0.0, qy = 0.0, qr = 0.0;
        if (valid) {
            q = pidx[o0 + (t >> 2)];
            c = 4u * q + (uint32_t)(t & 3);
            ccx = cx[c];
            ccy = cy[c];
            crr = r[c];
            valid = crr >= 0.0;                      // empty candidates (midpoint tree) take no part
            if (merge && (lane & 3) == 0) {
                qx = pcx[q];
                qy = pcy[q];
                qr = pr[q];
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (!conn[j]) continue;                  // warp-uniform
            const uint32_t b = (uint32_t)(4 * par + j);
            const bool ws = valid && (c != b) && well_separated(bx[j], by[j], br[j], ccx, ccy, crr, theta);
            unsigned wm = __ballot_sync(0xffffffffu, valid && ws);
            bool merged = false;                    // my group of four merges into its parent q
            if (merge) {
                const bool all4 = ((wm >> (lane & ~3)) & 0xFu) == 0xFu;
                bool mq = false;
                if (all4 && (lane & 3) == 0) mq = well_separated(bx[j], by[j], br[j], qx, qy, qr, theta);
                merged = __shfl_sync(0xffffffffu, mq ? 1 : 0, lane & ~3) != 0;
                wm = __ballot_sync(0xffffffffu, valid && ws && !merged);
            }
            const unsigned sm = __ballot_sync(0xffffffffu, valid && !ws);
            const unsigned xm = __ballot_sync(0xffffffffu, merged && (lane & 3) == 0);
            if (valid) {
                if (merged) {
                    if ((lane & 3) == 0) xtmp[slot[j] / 4 + nx[j] + __popc(xm & lt)] = q;
                } else if (ws) {
                    wtmp[slot[j] + nw[j] + __popc(wm & lt)] = c;
                } else {
                    stmp[slot[j] + ns[j] + __popc(sm & lt)] = c;
                }
            }
            nw[j] += __popc(wm);
            ns[j] += __popc(sm);
            nx[j] += __popc(xm);
        }
    }
    if (lane < 4 && live[lane]) {
        const int64_t b = 4 * par + lane;
        // (register arrays indexed by lane: select instead of local memory)
        int64_t w = nw[0], sct = ns[0], x = nx[0];
#pragma unroll
        for (int j = 1; j < 4; ++j)
            if (lane == j) {
                w = nw[j];
                sct = ns[j];
                x = nx[j];
            }
        wcnt[b] = w;
        scnt[b] = sct;
        if (merge) xcnt[b] = x;
    }
}

// pack the slots into the CSR lists (warp per box)
__global__ void k_compact_lists(int64_t b0, int64_t b1, const int64_t* __restrict__ poff,
                                const uint32_t* __restrict__ wtmp, const uint32_t* __restrict__ stmp,
                                const uint32_t* __restrict__ xtmp, const int64_t* __restrict__ woff,
                                const int64_t* __restrict__ soff, const int64_t* __restrict__ xoff,
                                uint32_t* __restrict__ widx, uint32_t* __restrict__ sidx, uint32_t* __restrict__ xidx)
{
    const int64_t b = b0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (b >= b1) return;
    const int64_t slot = cand_slot(poff, b);
    for (int64_t k = lane; k < woff[b + 1] - woff[b]; k += 32) widx[woff[b] + k] = wtmp[slot + k];
    for (int64_t k = lane; k < soff[b + 1] - soff[b]; k += 32) sidx[soff[b] + k] = stmp[slot + k];
    if (xoff)
        for (int64_t k = lane; k < xoff[b + 1] - xoff[b]; k += 32) xidx[xoff[b] + k] = xtmp[slot / 4 + k];
}

// pack the slots into the CSR lists: one warp per parent, its four children's slot regions
// (contiguous, 4|S(parent)| entries each) into their (contiguous) CSR ranges; each list is
// copied as one flat range over the four children
__global__ void k_compact_lists4(int64_t b0, int64_t b1, const int64_t* __restrict__ poff,
                                const uint32_t* __restrict__ wtmp, const uint32_t* __restrict__ stmp,
                                const uint32_t* __restrict__ xtmp, const int64_t* __restrict__ woff,
                                const int64_t* __restrict__ soff, const int64_t* __restrict__ xoff,
                                uint32_t* __restrict__ widx, uint32_t* __restrict__ sidx, uint32_t* __restrict__ xidx)
{
    const int64_t par = (b0 >> 2) + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (4 * par >= b1) return;
    const int64_t c0 = max(4 * par, b0), c1 = min(4 * par + 4, b1);    // own children
    const int64_t reg = 4 * (poff[par + 1] - poff[par]);                 // slot region per child
    const int64_t base = cand_slot(poff, c0);
    auto copy = [&](const int64_t* __restrict__ off, const uint32_t* __restrict__ tmp, uint32_t* __restrict__ idx,
                    int64_t rg, int64_t bs) {
        const int64_t o0 = off[c0], tot = off[c1] - o0;
        int64_t j = c0, jstart = 0, jend = off[c0 + 1] - o0;         // child of output entry k
        for (int64_t k = lane; k < tot; k += 32) {
            while (k >= jend) {
                ++j;
                jstart = jend;
                jend = off[j + 1] - o0;
            }
            idx[o0 + k] = tmp[bs + (j - c0) * rg + (k - jstart)];
        }
    };
    copy(woff, wtmp, widx, reg, base);
    copy(soff, stmp, sidx, reg, base);
    if (xoff) copy(xoff, xtmp, xidx, reg / 4, base / 4);
}

// M2L work order of one level: inside each window of M2L_WIN consecutive boxes (tree
// order: neighbouring targets share source multipoles in cache), targets by descending
// weak-list length (clamped to 255), so the 32 targets of a warp walk lists of nearly
// equal length.  key = window << 8 | (255 - len), value = box.
#ifndef FMM2D_M2L_WIN
#define FMM2D_M2L_WIN 16384
#endif
__global__ void k_m2l_keys(int64_t b0, int64_t b1, const int64_t* __restrict__ woff, const int64_t* __restrict__ xoff,
                           uint32_t* __restrict__ key, uint32_t* __restrict__ box)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t b = b0 + i;
    if (b >= b1) return;
    const int64_t len = woff[b + 1] - woff[b] + (xoff ? xoff[b + 1] - xoff[b] : 0);
    key[i] = ((uint32_t)(i / FMM2D_M2L_WIN) << 8) | (uint32_t)(255 - (len < 255 ? len : 255));
    box[i] = (uint32_t)b;
}

// r/R exchange (DESIGN R23): Criterion 1 with the roles of r and R exchanged,
// r + theta R <= theta d for r < R strictly, evaluated in the same operation order.
__device__ __forceinline__ bool rr_exchange(double cbx, double cby, double rb, double ccx, double ccy, double rc,
                                            double theta)
{
    double dx = __dsub_rn(cbx, ccx);
    double dy = __dsub_rn(cby, ccy);
    double d = __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
    double R = fmax(rb, rc);
    double r = fmin(rb, rc);
    return (r < R) && (d > 0.0) && (__dadd_rn(r, __dmul_rn(theta, R)) <= __dmul_rn(theta, d));
}

// Split of the leaf strong lists: class 0 near (direct), 1 P2L into this smaller leaf, 2 M2P
// of a smaller leaf here; the order of each list is the strong list's.  Lists of at most
// RRL_THREAD entries (every leaf on near-uniform inputs): a thread per leaf (k_rr_lists_t);
// longer ones (non-uniform inputs) are collected by its count pass and split by a warp per
// leaf (k_rr_lists, ballot compaction).
constexpr int64_t RRL_THREAD = 64;
template <bool FILL>
__global__ void k_rr_lists_t(int64_t t0, int64_t t1, const double* __restrict__ cx, const double* __restrict__ cy,
                             const double* __restrict__ r, double theta, const int64_t* __restrict__ soff,
                             const uint32_t* __restrict__ sidx, int64_t* __restrict__ cnt,   // [3][nl + 1]
                             const int64_t* __restrict__ o0, const int64_t* __restrict__ o1,
                             const int64_t* __restrict__ o2, uint32_t* __restrict__ i0, uint32_t* __restrict__ i1,
                             uint32_t* __restrict__ i2, int64_t nl, uint32_t* __restrict__ longs,
                             unsigned int* __restrict__ nlong)
{
    const int64_t t = t0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= t1) return;
    const int64_t qa = soff[t], qb = soff[t + 1];
    if (qb - qa > RRL_THREAD) {                     // a warp's job (k_rr_lists)
        if (!FILL) longs[atomicAdd(nlong, 1u)] = (uint32_t)t;
        return;
    }
    const double tx = cx[t], ty = cy[t], tr = r[t];
    int64_t n0 = 0, n1 = 0, n2 = 0;
    for (int64_t q = qa; q < qb; ++q) {
        const uint32_t s = sidx[q];
        int cls = 0;
        if (s != (uint32_t)t && rr_exchange(tx, ty, tr, cx[s], cy[s], r[s], theta)) cls = (tr < r[s]) ? 1 : 2;
        if (FILL) {
            if (cls == 0) i0[o0[t] + n0] = s;
            else if (cls == 1) i1[o1[t] + n1] = s;
            else i2[o2[t] + n2] = s;
        }
        n0 += cls == 0;
        n1 += cls == 1;
        n2 += cls == 2;
    }
    if (!FILL) {
        cnt[t] = n0;
        cnt[(nl + 1) + t] = n1;
        cnt[2 * (nl + 1) + t] = n2;
    }
}

// warp per leaf: leaves t0 + w (leaves == nullptr) or leaves[w] (w < nleaves)
template <bool FILL>
__global__ void k_rr_lists(int64_t t0, int64_t t1, const double* __restrict__ cx, const double* __restrict__ cy,
                           const double* __restrict__ r, double theta, const int64_t* __restrict__ soff,
                           const uint32_t* __restrict__ sidx, int64_t* __restrict__ cnt,   // [3][nl + 1]
                           const int64_t* __restrict__ o0, const int64_t* __restrict__ o1,
                           const int64_t* __restrict__ o2, uint32_t* __restrict__ i0, uint32_t* __restrict__ i1,
                           uint32_t* __restrict__ i2, int64_t nl, const uint32_t* __restrict__ leaves = nullptr,
                           int64_t nleaves = 0)
{
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    int64_t t;
    if (leaves) {
        if (w >= nleaves) return;
        t = leaves[w];
    } else {
        t = t0 + w;
        if (t >= t1) return;
    }
    const double tx = cx[t], ty = cy[t], tr = r[t];
    const unsigned lt = (1u << lane) - 1u;
    int64_t n0 = 0, n1 = 0, n2 = 0;
    for (int64_t q0 = soff[t]; q0 < soff[t + 1]; q0 += 32) {
        const int64_t q = q0 + lane;
        const bool valid = q < soff[t + 1];
        uint32_t s = 0;
        int cls = 0;
        if (valid) {
            s = sidx[q];
            if (s != (uint32_t)t && rr_exchange(tx, ty, tr, cx[s], cy[s], r[s], theta)) cls = (tr < r[s]) ? 1 : 2;
        }
        const unsigned m0 = __ballot_sync(0xffffffffu, valid && cls == 0);
        const unsigned m1 = __ballot_sync(0xffffffffu, valid && cls == 1);
        const unsigned m2 = __ballot_sync(0xffffffffu, valid && cls == 2);
        if (FILL && valid) {
            if (cls == 0) i0[o0[t] + n0 + __popc(m0 & lt)] = s;
            else if (cls == 1) i1[o1[t] + n1 + __popc(m1 & lt)] = s;
            else i2[o2[t] + n2 + __popc(m2 & lt)] = s;
        }
        n0 += __popc(m0);
        n1 += __popc(m1);
        n2 += __popc(m2);
    }
    if (!FILL && lane == 0) {
        cnt[t] = n0;
        cnt[(nl + 1) + t] = n1;
        cnt[2 * (nl + 1) + t] = n2;
    }
}

// targets of one level with a long weak list (global ids; order irrelevant)
__global__ void k_long_lists(int64_t b0, int64_t b1, int64_t gbase, const int64_t* __restrict__ woff,
                             const int64_t* __restrict__ xoff, uint32_t* __restrict__ out, unsigned int* __restrict__ n)
{
    const int64_t b = b0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b < b1 && woff[b + 1] - woff[b] + (xoff ? xoff[b + 1] - xoff[b] : 0) > FMM2D_M2L_LONG)
        out[atomicAdd(n, 1u)] = (uint32_t)(gbase + b);
}

// leaves with a non-empty list (compacted ids)
// leaves with a non-empty list: those with at most short_max entries from the front of out
// (count n[0]), the longer ones from the back (count n[1]; out has t1 - t0 slots)
__global__ void k_nonempty(int64_t t0, int64_t t1, const int64_t* __restrict__ off, int64_t short_max,
                           uint32_t* __restrict__ out, unsigned int* __restrict__ n)
{
    const int64_t t = t0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= t1) return;
    const int64_t len = off[t + 1] - off[t];
    if (len <= 0) return;
    if (len <= short_max) out[atomicAdd(&n[0], 1u)] = (uint32_t)t;
    else out[(t1 - t0) - 1 - atomicAdd(&n[1], 1u)] = (uint32_t)t;
}

// Long near lists (non-uniform inputs: a leaf can be strongly coupled to thousands of
// leaves): cut at leaf boundaries into segments of about FMM2D_NEAR_SPLIT source rows,
// each evaluated by its own k_near CTA.  Entry q lies in bucket floor(rows before q /
// FMM2D_NEAR_SPLIT); a segment starts at every entry whose bucket differs from the
// previous entry's.  One warp per leaf (scans + ballots); lists of at most
// FMM2D_NEAR_SPLIT rows are not split (count 0).  Pass 1 counts, pass 2 writes.
template <bool FILL>
__global__ void k_near_segs(int64_t t0, int64_t t1, const int64_t* __restrict__ noff, const uint32_t* __restrict__ nidx,
                            const uint32_t* __restrict__ boff, int64_t* __restrict__ cnt,
                            const int64_t* __restrict__ seg_off, NearSeg* __restrict__ segs)
{
    const int64_t t = t0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (t >= t1) return;
    if (FILL && seg_off[t + 1] == seg_off[t]) return;
    const int64_t q0 = noff[t], q1 = noff[t + 1];
    const int64_t base = FILL ? seg_off[t] : 0;
    int64_t run = 0, prev_bucket = -1, nstart = 0;
    const unsigned lt = (1u << lane) - 1u;
    for (int64_t qc = q0; qc < q1; qc += 32) {
        const int64_t q = qc + lane;
        const bool valid = q < q1;
        const int64_t sz = valid ? (int64_t)(boff[nidx[q] + 1] - boff[nidx[q]]) : 0;
        int64_t incl = sz;
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const int64_t bucket = (run + incl - sz) / FMM2D_NEAR_SPLIT;
        int64_t pb = __shfl_up_sync(0xffffffffu, bucket, 1);
        if (lane == 0) pb = prev_bucket;
        const bool start = valid && bucket != pb;
        const unsigned sm = __ballot_sync(0xffffffffu, start);
        if (FILL && start) {
            const int64_t k = nstart + __popc(sm & lt);     // segment number
            segs[base + k].qa = q;
            segs[base + k].t = (uint32_t)t;
            if (k > 0) segs[base + k - 1].qb = q;
        }
        nstart += __popc(sm);
        const int last = (int)min((int64_t)31, q1 - 1 - qc);
        prev_bucket = __shfl_sync(0xffffffffu, bucket, last);
        run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) {
        if (FILL) segs[base + nstart - 1].qb = q1;
        else cnt[t] = (run > FMM2D_NEAR_SPLIT) ? nstart : 0;
    }
}

// ordered P2P pairs (j != i) of one evaluation: sum_t n_t * sum_{s in S(t)} n_s - N
__global__ void k_pair_count(int64_t t0, int64_t t1, const uint32_t* __restrict__ off,
                             const int64_t* __restrict__ soff, const uint32_t* __restrict__ sidx,
                             unsigned long long* __restrict__ total, unsigned long long* __restrict__ max_rows)
{
    int64_t t = t0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long v = 0, mx = 0;
    if (t < t1) {
        unsigned long long ns = 0;
        for (int64_t q = soff[t]; q < soff[t + 1]; ++q) {
            uint32_t s = sidx[q];
            ns += off[s + 1] - off[s];
        }
        unsigned long long nt = off[t + 1] - off[t];
        v = nt * ns - nt;
        mx = ns;
    }
    for (int o = 16; o; o >>= 1) {
        v += __shfl_xor_sync(0xffffffffu, v, o);
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(total, v);
    if ((threadIdx.x & 31) == 0 && mx) atomicMax(max_rows, mx);     // longest near list (source rows)
}

inline unsigned grid_for(int64_t n, int bs) { return (unsigned)((n + bs - 1) / bs); }

}  // namespace

// r/R exchange (DESIGN R23): split the leaf strong lists into near / P2L / M2P CSR
// lists and collect the leaves that have P2L or M2P work.
static int build_rr_lists(fmm2d_plan* P)
{
    cudaStream_t st = P->stream;
    const int L = P->L;
    const int64_t nl = nboxes(L), t0 = P->box_lo(L), t1 = P->box_hi(L);
    const double* cx = P->cx + P->base[L];
    const double* cy = P->cy + P->base[L];
    const double* r = P->r + P->base[L];
    const Csr& S = P->strong[L];
    int64_t* cnt = nullptr;
    void* scratch = nullptr;
    size_t sb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, sb, (int64_t*)nullptr, (int64_t*)nullptr, (int)(nl + 1), st);
    uint32_t* longs = nullptr;
    unsigned int* nlong_d = nullptr;
    FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&cnt, sizeof(int64_t) * 3 * (nl + 1), st));
    FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&scratch, sb, st));
    FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&longs, sizeof(uint32_t) * std::max<int64_t>(nl, 1) + 16, st));
    nlong_d = reinterpret_cast<unsigned int*>(longs + std::max<int64_t>(nl, 1));
    auto body = [&]() -> int {
        FMM2D_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * 3 * (nl + 1), st));
        // short lists: a thread per leaf (the long ones collected for a warp each)
        FMM2D_CUDA_TRY(cudaMemsetAsync(nlong_d, 0, sizeof(unsigned int), st));
        k_rr_lists_t<false><<<grid_for(t1 - t0, 256), 256, 0, st>>>(t0, t1, cx, cy, r, P->theta, S.off, S.idx, cnt,
                                                                    nullptr, nullptr, nullptr, nullptr, nullptr,
                                                                    nullptr, nl, longs, nlong_d);
        note_launch();
        unsigned int nlong = 0;
        FMM2D_CUDA_TRY(cudaMemcpyAsync(&nlong, nlong_d, sizeof(nlong), cudaMemcpyDeviceToHost, st));
        FMM2D_CUDA_TRY(cudaStreamSynchronize(st));
        const unsigned grid = grid_for((int64_t)nlong * 32, 256);
        if (nlong) {
            k_rr_lists<false><<<grid, 256, 0, st>>>(t0, t1, cx, cy, r, P->theta, S.off, S.idx, cnt, nullptr, nullptr,
                                                    nullptr, nullptr, nullptr, nullptr, nl, longs, nlong);
            note_launch();
        }
        Csr* C[3] = {&P->near, &P->rr_p2l, &P->rr_m2p};
        int64_t tot[3];
        for (int c = 0; c < 3; ++c) {
            *C[c] = Csr();
            FMM2D_TRY(dev_alloc(P, (void**)&C[c]->off, sizeof(int64_t) * (nl + 1)));
            size_t s2 = sb;
            FMM2D_CUDA_TRY(cub::DeviceScan::ExclusiveSum(scratch, s2, cnt + c * (nl + 1), C[c]->off, (int)(nl + 1), st));
            FMM2D_CUDA_TRY(cudaMemcpyAsync(&tot[c], C[c]->off + nl, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        }
        FMM2D_CUDA_TRY(cudaStreamSynchronize(st));
        for (int c = 0; c < 3; ++c) {
            C[c]->total = tot[c];
            FMM2D_TRY(dev_alloc(P, (void**)&C[c]->idx, sizeof(uint32_t) * std::max<int64_t>(tot[c], 1)));
        }
        k_rr_lists_t<true><<<grid_for(t1 - t0, 256), 256, 0, st>>>(t0, t1, cx, cy, r, P->theta, S.off, S.idx,
                                                                   nullptr, P->near.off, P->rr_p2l.off,
                                                                   P->rr_m2p.off, P->near.idx, P->rr_p2l.idx,
                                                                   P->rr_m2p.idx, nl, nullptr, nullptr);
        note_launch();
        if (nlong) {
            k_rr_lists<true><<<grid, 256, 0, st>>>(t0, t1, cx, cy, r, P->theta, S.off, S.idx, nullptr, P->near.off,
                                                   P->rr_p2l.off, P->rr_m2p.off, P->near.idx, P->rr_p2l.idx,
                                                   P->rr_m2p.idx, nl, longs, nlong);
            note_launch();
        }
        // leaves with P2L / M2P work (the order is irrelevant: each leaf is independent)
        // (short lists from the front, long ones from the back: a warp or a block each, rr.cu)
        unsigned int* d_n = (unsigned int*)cnt;
        FMM2D_CUDA_TRY(cudaMemsetAsync(d_n, 0, 4 * sizeof(unsigned int), st));
        const int64_t cap = std::max<int64_t>(t1 - t0, 1);
        FMM2D_TRY(dev_alloc(P, (void**)&P->rr_p2l_leaves, sizeof(uint32_t) * cap));
        FMM2D_TRY(dev_alloc(P, (void**)&P->rr_m2p_leaves, sizeof(uint32_t) * cap));
        k_nonempty<<<grid_for(t1 - t0, 256), 256, 0, st>>>(t0, t1, P->rr_p2l.off, FMM2D_RR_SHORT, P->rr_p2l_leaves, d_n);
        note_launch();
        k_nonempty<<<grid_for(t1 - t0, 256), 256, 0, st>>>(t0, t1, P->rr_m2p.off, FMM2D_RR_SHORT, P->rr_m2p_leaves, d_n + 2);
        note_launch();
        unsigned int h_n[4];
        FMM2D_CUDA_TRY(cudaMemcpyAsync(h_n, d_n, sizeof(h_n), cudaMemcpyDeviceToHost, st));
        FMM2D_CUDA_TRY(cudaStreamSynchronize(st));
        P->rr_np2l = (int64_t)h_n[0] + h_n[1];
        P->rr_nm2p = (int64_t)h_n[2] + h_n[3];
        P->rr_np2l_short = h_n[0];
        P->rr_nm2p_short = h_n[2];
        P->rr_leaf_cap = cap;
        FMM2D_TRY(dev_alloc(P, (void**)&P->rr_acc, sizeof(double4) * P->n));
        return 0;
    };
    const int rc = body();
    cudaFreeAsync(cnt, st);
    cudaFreeAsync(scratch, st);
    cudaFreeAsync(longs, st);
    return rc;
}

static int build_near_segments(fmm2d_plan* P)
{
    cudaStream_t st = P->stream;
    const int L = P->L;
    const int64_t nl = nboxes(L), t0 = P->box_lo(L), t1 = P->box_hi(L);
    const uint32_t* boff = P->boff + P->obase[L];
    int64_t* cnt = nullptr;
    void* scratch = nullptr;
    size_t sb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, sb, (int64_t*)nullptr, (int64_t*)nullptr, (int)(nl + 1), st);
    FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&cnt, sizeof(int64_t) * (nl + 1), st));
    FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&scratch, sb, st));
    auto body = [&]() -> int {
        FMM2D_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (nl + 1), st));
        k_near_segs<false><<<grid_for((t1 - t0) * 32, 256), 256, 0, st>>>(t0, t1, P->near.off, P->near.idx, boff,
                                                                           cnt, nullptr, nullptr);
        note_launch();
        int64_t* soff = nullptr;
        FMM2D_TRY(dev_alloc(P, (void**)&soff, sizeof(int64_t) * (nl + 1)));
        size_t s2 = sb;
        FMM2D_CUDA_TRY(cub::DeviceScan::ExclusiveSum(scratch, s2, cnt, soff, (int)(nl + 1), st));
        int64_t tot = 0;
        FMM2D_CUDA_TRY(cudaMemcpyAsync(&tot, soff + nl, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        FMM2D_CUDA_TRY(cudaStreamSynchronize(st));
        P->near_nseg = tot;
        if (tot == 0) return 0;                         // nothing split: k_near skips the lookups
        P->near_seg_off = soff;
        FMM2D_TRY(dev_alloc(P, (void**)&P->near_segs, sizeof(NearSeg) * tot));
        FMM2D_TRY(dev_alloc(P, (void**)&P->near_part, sizeof(double4) * tot * std::max(1, P->stats.max_leaf)));
        k_near_segs<true><<<grid_for((t1 - t0) * 32, 256), 256, 0, st>>>(t0, t1, P->near.off, P->near.idx, boff,
                                                                          nullptr, soff, P->near_segs);
        note_launch();
        FMM2D_TRY(dev_alloc(P, (void**)&P->near_split, sizeof(uint32_t) * std::max<int64_t>(t1 - t0, 1)));
        unsigned int* d_n = (unsigned int*)cnt;
        FMM2D_CUDA_TRY(cudaMemsetAsync(d_n, 0, 2 * sizeof(unsigned int), st));
        k_nonempty<<<grid_for(t1 - t0, 256), 256, 0, st>>>(t0, t1, soff, INT64_MAX, P->near_split, d_n);
        note_launch();
        unsigned int h_n = 0;
        FMM2D_CUDA_TRY(cudaMemcpyAsync(&h_n, d_n, sizeof(h_n), cudaMemcpyDeviceToHost, st));
        FMM2D_CUDA_TRY(cudaStreamSynchronize(st));
        P->near_nsplit = h_n;
        return 0;
    };
    const int rc = body();
    cudaFreeAsync(cnt, st);
    cudaFreeAsync(scratch, st);
    return rc;
}

int build_lists(fmm2d_plan* P)
{
    const int L = P->L;
    cudaStream_t st = P->stream;
    P->strong.assign(L + 1, Csr());
    P->weak.assign(L + 1, Csr());
    P->xweak.assign(L + 1, Csr());
    // level 0: S(root) = {root}, no weak pairs
    {
        int64_t h_off[2] = {0, 1}, h_woff[2] = {0, 0};
        uint32_t zero = 0;
        FMM2D_TRY(dev_alloc(P, (void**)&P->strong[0].off, sizeof(h_off)));
        FMM2D_TRY(dev_alloc(P, (void**)&P->strong[0].idx, sizeof(uint32_t)));
        FMM2D_TRY(dev_alloc(P, (void**)&P->weak[0].off, sizeof(h_woff)));
        FMM2D_CUDA_TRY(cudaMemcpyAsync(P->strong[0].off, h_off, sizeof(h_off), cudaMemcpyHostToDevice, st));
        FMM2D_CUDA_TRY(cudaMemcpyAsync(P->strong[0].idx, &zero, sizeof(zero), cudaMemcpyHostToDevice, st));
        FMM2D_CUDA_TRY(cudaMemcpyAsync(P->weak[0].off, h_woff, sizeof(h_woff), cudaMemcpyHostToDevice, st));
        FMM2D_CUDA_TRY(cudaStreamSynchronize(st));   // host sources go out of scope
        P->strong[0].total = 1;
        P->weak[0].total = 0;
    }
    if (L == 0) {
        P->stats.strong_leaf_pairs = 1;
        P->stats.p2p_pairs = P->n * (P->n - 1);
        P->near = P->strong[0];
        return 0;
    }
    int64_t nbmax = nboxes(L);
    int64_t *cnt_w = nullptr, *cnt_s = nullptr, *cnt_x = nullptr;
    void* scratch = nullptr;
    size_t scan_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (int64_t*)nullptr, (int64_t*)nullptr, (int)(nbmax + 1), st);
    FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&cnt_w, sizeof(int64_t) * (nbmax + 1), st));
    FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&cnt_s, sizeof(int64_t) * (nbmax + 1), st));
    FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&cnt_x, sizeof(int64_t) * (nbmax + 1), st));
    FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&scratch, scan_bytes, st));
    PhaseTrace tr(st);
    tr.mark("lists start");
    uint32_t *wtmp = nullptr, *stmp = nullptr, *xtmp = nullptr;
    int64_t tmp_cap = 0;
    auto body = [&]() -> int {
        const bool merge_on = (P->flags & FMM2D_PARENT_MERGE) != 0;
        for (int l = 1; l <= L; ++l) {
            int64_t nb = nboxes(l);
            Csr& W = P->weak[l];
            Csr& S = P->strong[l];
            Csr& X = P->xweak[l];
            const Csr& PS = P->strong[l - 1];
            const double* cx = P->cx + P->base[l];
            const double* cy = P->cy + P->base[l];
            const double* r = P->r + P->base[l];
            const bool merge = merge_on && l >= 2;
            FMM2D_TRY(dev_alloc(P, (void**)&W.off, sizeof(int64_t) * (nb + 1)));
            FMM2D_TRY(dev_alloc(P, (void**)&S.off, sizeof(int64_t) * (nb + 1)));
            if (merge) FMM2D_TRY(dev_alloc(P, (void**)&X.off, sizeof(int64_t) * (nb + 1)));
            // boxes of this rank: all of a replicated level, the own subtrees below it
            const int64_t b0 = P->box_lo(l), b1 = P->box_hi(l);
            if (b1 - b0 < nb || merge) {
                FMM2D_CUDA_TRY(cudaMemsetAsync(cnt_w, 0, sizeof(int64_t) * (nb + 1), st));
                FMM2D_CUDA_TRY(cudaMemsetAsync(cnt_s, 0, sizeof(int64_t) * (nb + 1), st));
                if (merge) FMM2D_CUDA_TRY(cudaMemsetAsync(cnt_x, 0, sizeof(int64_t) * (nb + 1), st));
            } else {
                FMM2D_CUDA_TRY(cudaMemsetAsync(cnt_w + nb, 0, sizeof(int64_t), st));
                FMM2D_CUDA_TRY(cudaMemsetAsync(cnt_s + nb, 0, sizeof(int64_t), st));
            }
            const double* pcx = P->cx + P->base[l - 1];
            const double* pcy = P->cy + P->base[l - 1];
            const double* pr = P->r + P->base[l - 1];
            unsigned grid = grid_for((b1 - b0) * 32, 256);
            const unsigned grid4 = grid_for((((b1 + 3) >> 2) - (b0 >> 2)) * 32, 256);   // warp per parent
            const int64_t cap = 16 * PS.total;          // sum of the candidate counts of all boxes
            // slot buffers kept across levels and grown geometrically (few, large pool
            // allocations instead of three fresh ones per level)
            if (cap > tmp_cap) {
                if (wtmp) cudaFreeAsync(wtmp, st);
                if (stmp) cudaFreeAsync(stmp, st);
                if (xtmp) cudaFreeAsync(xtmp, st);
                wtmp = stmp = xtmp = nullptr;
                tmp_cap = std::max<int64_t>(cap, 2 * tmp_cap);
                FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&wtmp, sizeof(uint32_t) * tmp_cap, st));
                FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&stmp, sizeof(uint32_t) * tmp_cap, st));
                FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&xtmp, sizeof(uint32_t) * (tmp_cap / 4 + 1), st));
            }
            // per parent while the parents' strong lists are short (C5: ~11), per box when long
            const int64_t npar = ((b1 + 3) >> 2) - (b0 >> 2);
            if (FMM2D_LISTS_THREAD && PS.total <= 32 * std::max<int64_t>(npar, 1))
                k_lists_t<<<grid_for(b1 - b0, 256), 256, 0, st>>>(b0, b1, cx, cy, r, P->theta, PS.off, PS.idx, cnt_w,
                                                                  cnt_s, wtmp, stmp, merge, pcx, pcy, pr, cnt_x, xtmp);
            else if (PS.total <= 32 * std::max<int64_t>(npar, 1))
                k_lists<<<grid4, 256, 0, st>>>(b0, b1, cx, cy, r, P->theta, PS.off, PS.idx, cnt_w, cnt_s, wtmp, stmp,
                                              merge, pcx, pcy, pr, cnt_x, xtmp);
            else
                k_lists_box<<<grid, 256, 0, st>>>(b0, b1, cx, cy, r, P->theta, PS.off, PS.idx, cnt_w, cnt_s, wtmp, stmp,
                                                  merge, pcx, pcy, pr, cnt_x, xtmp);
            fmm2d::note_launch();
            FMM2D_CUDA_TRY(cudaGetLastError());
            size_t sb = scan_bytes;
            FMM2D_CUDA_TRY(cub::DeviceScan::ExclusiveSum(scratch, sb, cnt_w, W.off, (int)(nb + 1), st));
            sb = scan_bytes;
            FMM2D_CUDA_TRY(cub::DeviceScan::ExclusiveSum(scratch, sb, cnt_s, S.off, (int)(nb + 1), st));
            if (merge) {
                sb = scan_bytes;
                FMM2D_CUDA_TRY(cub::DeviceScan::ExclusiveSum(scratch, sb, cnt_x, X.off, (int)(nb + 1), st));
            }
            int64_t tot[3] = {0, 0, 0};
            FMM2D_CUDA_TRY(cudaMemcpyAsync(&tot[0], W.off + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
            FMM2D_CUDA_TRY(cudaMemcpyAsync(&tot[1], S.off + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
            if (merge)
                FMM2D_CUDA_TRY(cudaMemcpyAsync(&tot[2], X.off + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
            FMM2D_CUDA_TRY(cudaStreamSynchronize(st));
            W.total = tot[0];
            S.total = tot[1];
            X.total = tot[2];
            FMM2D_TRY(dev_alloc(P, (void**)&W.idx, sizeof(uint32_t) * std::max<int64_t>(W.total, 1)));
            FMM2D_TRY(dev_alloc(P, (void**)&S.idx, sizeof(uint32_t) * std::max<int64_t>(S.total, 1)));
            if (merge) FMM2D_TRY(dev_alloc(P, (void**)&X.idx, sizeof(uint32_t) * std::max<int64_t>(X.total, 1)));
            if (PS.total <= 16 * std::max<int64_t>(npar, 1))      // short lists: a warp per parent
                k_compact_lists4<<<grid4, 256, 0, st>>>(b0, b1, PS.off, wtmp, stmp, xtmp, W.off, S.off,
                                                        merge ? X.off : nullptr, W.idx, S.idx, X.idx);
            else
                k_compact_lists<<<grid, 256, 0, st>>>(b0, b1, PS.off, wtmp, stmp, xtmp, W.off, S.off,
                                                      merge ? X.off : nullptr, W.idx, S.idx, X.idx);
            fmm2d::note_launch();
            FMM2D_CUDA_TRY(cudaGetLastError());

            P->stats.weak_pairs += W.total + X.total;
            tr.mark("lists level " + std::to_string(l));
        }
        // M2L work order (k_m2l_keys)
        {
            int64_t tot = 0;
            for (int l = 1; l <= L; ++l) tot += P->box_hi(l) - P->box_lo(l);
            FMM2D_TRY(dev_alloc(P, (void**)&P->m2l_order, sizeof(uint32_t) * std::max<int64_t>(tot, 1)));
            uint32_t *k0 = nullptr, *k1 = nullptr;
            uint32_t* v0 = nullptr;
            void* sc = nullptr;
            size_t sb = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, sb, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                            (uint32_t*)nullptr, (int)nbmax, 0, 32, st);
            FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&k0, sizeof(uint32_t) * nbmax, st));
            FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&k1, sizeof(uint32_t) * nbmax, st));
            FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&v0, sizeof(uint32_t) * std::max<int64_t>(tot, nbmax), st));
            FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&sc, std::max<size_t>(sb, 16), st));
            int64_t o = 0;
            for (int l = 1; l <= L; ++l) {
                const int64_t b0 = P->box_lo(l), b1 = P->box_hi(l), nb = b1 - b0;
                k_m2l_keys<<<grid_for(nb, 256), 256, 0, st>>>(b0, b1, P->weak[l].off, P->xweak[l].off, k0, v0);
                fmm2d::note_launch();
                int bits = 8;
                while (((int64_t)1 << (bits - 8)) * FMM2D_M2L_WIN < nb) ++bits;
                size_t s2 = sb;
                FMM2D_CUDA_TRY(cub::DeviceRadixSort::SortPairs(sc, s2, k0, k1, v0, P->m2l_order + o, (int)nb, 0, bits,
                                                               st));
                o += nb;
            }
            // targets with long weak lists (k_m2l_long)
            unsigned int* d_n = (unsigned int*)k1;
            FMM2D_CUDA_TRY(cudaMemsetAsync(d_n, 0, sizeof(unsigned int), st));
            for (int l = 1; l <= L; ++l) {
                const int64_t b0 = P->box_lo(l), b1 = P->box_hi(l);
                k_long_lists<<<grid_for(b1 - b0, 256), 256, 0, st>>>(b0, b1, P->base[l], P->weak[l].off,
                                                                     P->xweak[l].off, v0, d_n);
                fmm2d::note_launch();
            }
            unsigned int h_n = 0;
            FMM2D_CUDA_TRY(cudaMemcpyAsync(&h_n, d_n, sizeof(h_n), cudaMemcpyDeviceToHost, st));
            FMM2D_CUDA_TRY(cudaStreamSynchronize(st));
            P->m2l_nlong = h_n;
            FMM2D_TRY(dev_alloc(P, (void**)&P->m2l_long, sizeof(uint32_t) * std::max<int64_t>(h_n, 1)));
            if (h_n)
                FMM2D_CUDA_TRY(cudaMemcpyAsync(P->m2l_long, v0, sizeof(uint32_t) * h_n, cudaMemcpyDeviceToDevice, st));
            cudaFreeAsync(k0, st);
            cudaFreeAsync(k1, st);
            cudaFreeAsync(v0, st);
            cudaFreeAsync(sc, st);
        }
        P->stats.strong_leaf_pairs = P->strong[L].total;
        const int64_t t0 = P->box_lo(L), t1 = P->box_hi(L);
        P->near = P->strong[L];                     // the direct pairs (all strong pairs unless r/R exchange)
        tr.mark("m2l order + long lists");
        if (P->flags & FMM2D_RR_EXCHANGE) FMM2D_TRY(build_rr_lists(P));
        unsigned long long* d_tot = (unsigned long long*)cnt_w;   // reuse scratch
        FMM2D_CUDA_TRY(cudaMemsetAsync(d_tot, 0, 2 * sizeof(unsigned long long), st));
        k_pair_count<<<grid_for(t1 - t0, 256), 256, 0, st>>>(t0, t1, P->boff + P->obase[L], P->near.off,
                                                             P->near.idx, d_tot, d_tot + 1); fmm2d::note_launch();
        FMM2D_CUDA_TRY(cudaGetLastError());
        unsigned long long h_tot[2] = {0, 0};
        FMM2D_CUDA_TRY(cudaMemcpyAsync(h_tot, d_tot, sizeof(h_tot), cudaMemcpyDeviceToHost, st));
        FMM2D_CUDA_TRY(cudaStreamSynchronize(st));
        P->stats.p2p_pairs = (int64_t)h_tot[0];
        // long near lists: segments for k_near (only if some list exceeds the split size)
        tr.mark("rr lists + pair count");
        if (P->stats.max_leaf <= FMM2D_NEAR_CHUNK && h_tot[1] > FMM2D_NEAR_SPLIT) FMM2D_TRY(build_near_segments(P));
        tr.mark("near segments");
        return 0;
    };
    int rc = body();
    if (wtmp) cudaFreeAsync(wtmp, st);
    if (stmp) cudaFreeAsync(stmp, st);
    if (xtmp) cudaFreeAsync(xtmp, st);
    cudaFreeAsync(cnt_w, st);
    cudaFreeAsync(cnt_s, st);
    cudaFreeAsync(cnt_x, st);
    cudaFreeAsync(scratch, st);
    return rc;
}

}  // namespace fmm2d
