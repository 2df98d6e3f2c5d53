// tree.cu -- A0-A2: validation, the balanced median-split tree and the box discs.
//
// Paper: "The multipole mesh is constructed first and is obtained by recursively
// splitting the source points at or near their median in each coordinate
// direction"; the points live in "a 2^d-tree cut at a certain maximum
// level".  Readings R5-R8, R13.
//
// GPU formulation (bit-exact by construction): two record
// lists are kept, one sorted by (x, idx) and one by (y, idx) inside every box.
// A split along x takes the first ceil(n/2) of the x-list (trivially partitioned)
// and stably partitions the y-list by "(x, idx) < the first x-high record": one
// flag pass, one device-wide scan, one scatter.  Stability keeps both lists sorted,
// so the y-split is the same step with the axes swapped.  The list that is only
// trivially split is never rewritten: its records keep the id of the previous
// (half-)level and every reader refines it from the record's position and the
// offsets ("stale id + refine").  Box sizes are a pure function of N, so all
// offsets come from a tiny per-level kernel.  The presort is two stable radix sorts
// of orderable 64-bit keys (ties leave in index order); the sorted key itself gives
// the sort coordinate back, only the other coordinate is gathered.
#include <cub/cub.cuh>

#include "fmm2d_internal.cuh"

namespace fmm2d {

namespace {

__device__ __forceinline__ uint64_t orderable(double v)
{
    uint64_t u = (uint64_t)__double_as_longlong(v);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double from_orderable(uint64_t k)
{
    uint64_t u = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
    return __longlong_as_double((long long)u);
}

// A0: validate, map -0 -> +0 (x + 0.0), order keys, identity indices.
__global__ void k_canon(const double2* __restrict__ z, int64_t n, double* __restrict__ xs,
                        double* __restrict__ ys, uint64_t* __restrict__ kx, uint64_t* __restrict__ ky,
                        uint32_t* __restrict__ iota, int* __restrict__ bad)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double2 v = z[i];
    double x = __dadd_rn(v.x, 0.0), y = __dadd_rn(v.y, 0.0);
    if (!isfinite(x) || !isfinite(y)) atomicOr(bad, 1);
    xs[i] = x;
    ys[i] = y;
    kx[i] = orderable(x);
    ky[i] = orderable(y);
    iota[i] = (uint32_t)i;
}

// records of one presorted list: the sort coordinate from the key, the other gathered
__global__ void k_make_recs(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ order,
                            const double* __restrict__ other, int axis, int64_t n, Rec* __restrict__ out)
{
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    uint32_t i = order[k];
    double c = from_orderable(keys[k]), o = other[i];
    Rec r;
    r.x = axis ? o : c;
    r.y = axis ? c : o;
    r.idx = i;
    r.box = 0;
    out[k] = r;
}

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

// (coord, idx) < (coord', idx') on axis 0 = x, 1 = y  (DESIGN R6)
__device__ __forceinline__ bool rec_less(const Rec& a, const Rec& b, int axis)
{
    double ca = axis ? a.y : a.x, cb = axis ? b.y : b.x;
    return (ca < cb) || (ca == cb && a.idx < b.idx);
}

// parent segment of position k: the record's (stale) id, refined by one split if needed
__device__ __forceinline__ uint32_t parent_of(uint32_t box, int64_t k, const uint32_t* __restrict__ refine)
{
    return refine ? 2 * box + ((uint32_t)k >= refine[2 * box + 1] ? 1u : 0u) : box;
}

// Per parent segment p: number of high-side records (the split rule fixes it).
__global__ void k_high_sizes(const uint32_t* __restrict__ par_off, const uint32_t* __restrict__ sub_off,
                             int64_t np, uint32_t* __restrict__ hs)
{
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < np) hs[p] = par_off[p + 1] - sub_off[2 * p + 1];
}

// One split step in a single pass (replaces flag -> device scan -> scatter):
//   flag  = record is on the high side of its parent segment p, i.e.
//           (coord, idx) >= the first high record split_list[sub_off[2p+1]];
//   G(k)  = number of high records before position k over the whole list, from a
//           block scan + decoupled look-back across tiles (tile ids taken in launch
//           order from a counter, so predecessors always make progress);
//   dst   = stable position inside p: high -> sub_off[2p+1] + (G(k) - Gp[p]),
//           low -> k - (G(k) - Gp[p]), where Gp[p] = high records before segment p
//           (exclusive scan of k_high_sizes, a function of the offsets only).
constexpr int PT = 256, PI = 4, PTILE = PT * PI;
constexpr uint64_t ST_AGG = 1ull << 62, ST_PRE = 2ull << 62, ST_MASK = 3ull << 62;

__global__ void __launch_bounds__(PT) k_partition(const Rec* __restrict__ list, const Rec* __restrict__ split_list,
                                                  const uint32_t* __restrict__ refine,
                                                  const uint32_t* __restrict__ par_off,
                                                  const uint32_t* __restrict__ sub_off,
                                                  const uint32_t* __restrict__ Gp, int axis, int64_t n,
                                                  Rec* __restrict__ out, unsigned long long* __restrict__ tstate,
                                                  unsigned int* __restrict__ ticket)
{
    typedef cub::BlockScan<uint32_t, PT> Scan;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ uint32_t s_tile, s_prefix;
    __shared__ __align__(16) Rec stage[PTILE];
    const int tid = threadIdx.x;
    if (tid == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const int64_t k0 = (int64_t)tile * PTILE + (int64_t)tid * PI;
    // stage the tile through shared memory with coalesced 16-byte loads (all independent)
    const int64_t kt = (int64_t)tile * PTILE;
    const int nrec = (int)((n - kt) < PTILE ? (n - kt) : PTILE);
    {
        const uint4* g = reinterpret_cast<const uint4*>(list + kt);
        uint4* s = reinterpret_cast<uint4*>(stage);
        const int nvec = (nrec * (int)sizeof(Rec)) / 16;            // whole vectors
        for (int v = tid; v < nvec; v += PT) s[v] = g[v];
        if (tid == 0 && (nrec * (int)sizeof(Rec)) % 16) stage[nrec - 1] = list[kt + nrec - 1];
    }
    __syncthreads();
    Rec r[PI];
    uint32_t par[PI], f[PI];
    uint32_t cnt = 0;
#pragma unroll
    for (int u = 0; u < PI; ++u) {
        const int64_t k = k0 + u;
        f[u] = 0;
        par[u] = 0;
        if (k < n) {
            r[u] = stage[tid * PI + u];
            const uint32_t p = parent_of(r[u].box, k, refine);
            par[u] = p;
            const uint32_t sp = sub_off[2 * p + 1];
            if (sp < par_off[p + 1]) f[u] = rec_less(r[u], split_list[sp], axis) ? 0u : 1u;
        }
        cnt += f[u];
    }
    uint32_t excl, agg;
    Scan(scan_tmp).ExclusiveSum(cnt, excl, agg);
    // decoupled look-back (warp 0)
    if (tid < 32) {
        uint32_t prefix = 0;
        if (tile == 0) {
            if (tid == 0) atomicExch(&tstate[0], ST_PRE | agg);
        } else {
            if (tid == 0) atomicExch(&tstate[tile], ST_AGG | agg);
            int64_t j = (int64_t)tile - 1 - tid;
            for (;;) {
                unsigned long long s = 0;
                if (j >= 0) {
                    do {
                        s = *((volatile unsigned long long*)&tstate[j]);
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
            if (tid == 0) atomicExch(&tstate[tile], ST_PRE | (prefix + agg));
        }
        if (tid == 0) s_prefix = prefix;
    }
    __syncthreads();
    uint32_t g = s_prefix + excl;             // G(k) for the first item of this thread
#pragma unroll
    for (int u = 0; u < PI; ++u) {
        const int64_t k = k0 + u;
        if (k < n) {
            const uint32_t p = par[u];
            const uint32_t hb = g - Gp[p];    // highs before k inside p
            const uint32_t dst = f[u] ? sub_off[2 * p + 1] + hb : (uint32_t)k - hb;
            Rec o = r[u];
            o.box = 2 * p + f[u];
            out[dst] = o;
        }
        g += f[u];
    }
}

// A2 (part 1): tight bounding box from the segment endpoints of both sorted lists;
// centre = 0.5 (min + max) (DESIGN R8).  Radius reset for part 2.
__global__ void k_bbox(const Rec* __restrict__ xl, const Rec* __restrict__ yl,
                       const uint32_t* __restrict__ off, int64_t nb, double* __restrict__ cx,
                       double* __restrict__ cy, double* __restrict__ r)
{
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    uint32_t s = off[b], e = off[b + 1];
    double xmin = xl[s].x, xmax = xl[e - 1].x, ymin = yl[s].y, ymax = yl[e - 1].y;
    cx[b] = __dmul_rn(0.5, __dadd_rn(xmin, xmax));
    cy[b] = __dmul_rn(0.5, __dadd_rn(ymin, ymax));
    r[b] = 0.0;
}

// Final order + A2 (part 2) for every level in one pass.  The final y-list is the
// leaf order (leaves ascending, (y, idx) inside, R13): write perm and the source
// rows, then r(box) = exact max distance (correctly rounded sqrt, no FMA) for the
// box of every level containing the point: a block-wide max when the whole block
// lies in one box (upper levels), else a segmented warp max; one atomicMax on the
// bit pattern per segment (non-negative doubles order like their uint64 bits).
constexpr int FIN_T = 256;
struct RadArgs {
    const double* cx[FMM2D_MAXL + 1];
    const double* cy[FMM2D_MAXL + 1];
    double* r[FMM2D_MAXL + 1];
};
__global__ void __launch_bounds__(FIN_T) k_finish(const Rec* __restrict__ yl, int64_t n, int L,
                                                  const uint32_t* __restrict__ offL, uint32_t* __restrict__ perm,
                                                  double4* __restrict__ src, RadArgs A)
{
    __shared__ uint32_t sleaf[FIN_T];
    __shared__ double wmax[FIN_T / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t k0 = (int64_t)blockIdx.x * FIN_T;
    const int64_t k = k0 + tid;
    const int nvalid = (int)((n - k0) < FIN_T ? (n - k0) : FIN_T);
    const bool valid = k < n;
    double x = 0.0, y = 0.0;
    uint32_t leaf = 0;
    if (valid) {
        Rec r = yl[k];
        leaf = (L > 0) ? parent_of(r.box, k, offL) : 0u;
        x = r.x;
        y = r.y;
        perm[k] = r.idx;
        src[k] = make_double4(x, y, 0.0, 0.0);
    }
    sleaf[tid] = leaf;
    __syncthreads();
    const uint32_t lf0 = sleaf[0], lf1 = sleaf[nvalid - 1];
    for (int l = L; l >= 0; --l) {
        const int sh = 2 * (L - l);
        const uint32_t box = leaf >> sh;
        double d = 0.0;
        if (valid) d = rn_dist2(x, y, A.cx[l][box], A.cy[l][box]);     // squared; sqrt below
        if ((lf0 >> sh) == (lf1 >> sh)) {                 // block-uniform (warp-uniform too)
            for (int o = 16; o; o >>= 1) d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
            if (lane == 0) wmax[warp] = d;
            __syncthreads();
            if (tid == 0) {
                double m = wmax[0];
                for (int w = 1; w < FIN_T / 32; ++w) m = fmax(m, wmax[w]);
                atomicMax((unsigned long long*)(A.r[l] + (lf0 >> sh)), (unsigned long long)__double_as_longlong(m));
            }
            __syncthreads();
        } else {
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

// r = sqrt_rn(max squared distance), every box of every level
__global__ void k_sqrt(double* __restrict__ r, int64_t nb)
{
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b < nb) r[b] = __dsqrt_rn(r[b]);
}

inline unsigned grid_for(int64_t n, int bs) { return (unsigned)((n + bs - 1) / bs); }

}  // namespace

int build_tree(fmm2d_plan* P, const double2* z)
{
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
    double *xs, *ys;
    uint64_t *kx, *ky, *ksort;
    uint32_t *iota, *ord, *hs, *Gp;
    Rec *xl, *yl, *tmp;
    int* bad;
    unsigned long long* tstate;
    unsigned int* ticket;
    void* scratch = nullptr;
    size_t sort_bytes = 0, scan_bytes = 0;
    const int64_t npmax = (L > 0) ? 2 * nboxes(L - 1) : 1;        // parents of the widest step
    const int64_t ntiles = (n + PTILE - 1) / PTILE;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (uint64_t*)nullptr, (uint64_t*)nullptr,
                                    (uint32_t*)nullptr, (uint32_t*)nullptr, (int)n, 0, 64, st);
    cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)npmax, st);
    size_t cub_bytes = std::max(sort_bytes, scan_bytes);
    std::vector<void*> tmp_ptrs;
    auto talloc = [&](void** p, size_t b) -> int {
        cudaError_t e = cudaMallocAsync(p, b, st);
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
        if ((rc = talloc((void**)&xs, 8 * n))) break;
        if ((rc = talloc((void**)&ys, 8 * n))) break;
        if ((rc = talloc((void**)&kx, 8 * n))) break;
        if ((rc = talloc((void**)&ky, 8 * n))) break;
        if ((rc = talloc((void**)&ksort, 8 * n))) break;
        if ((rc = talloc((void**)&iota, 4 * n))) break;
        if ((rc = talloc((void**)&ord, 4 * n))) break;
        if ((rc = talloc((void**)&hs, 4 * npmax))) break;
        if ((rc = talloc((void**)&Gp, 4 * npmax))) break;
        if ((rc = talloc((void**)&tstate, 8 * ntiles))) break;
        if ((rc = talloc((void**)&ticket, 4))) break;
        if ((rc = talloc((void**)&xl, sizeof(Rec) * n))) break;
        if ((rc = talloc((void**)&yl, sizeof(Rec) * n))) break;
        if ((rc = talloc((void**)&tmp, sizeof(Rec) * n))) break;
        if ((rc = talloc((void**)&bad, sizeof(int)))) break;
        if ((rc = talloc(&scratch, cub_bytes))) break;
    } while (0);
    if (rc) { tfree(); return rc; }

    auto body = [&]() -> int {
        FMM2D_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), st));
        k_canon<<<grid_for(n, BS), BS, 0, st>>>(z, n, xs, ys, kx, ky, iota, bad);
        fmm2d::note_launch();
        FMM2D_CUDA_TRY(cudaGetLastError());
        int h_bad = 0;
        FMM2D_CUDA_TRY(cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
        FMM2D_CUDA_TRY(cudaStreamSynchronize(st));
        if (h_bad) return FMM2D_ENONFINITE;
        // presort (stable LSD radix: ties stay in index order)
        size_t sb = cub_bytes;
        FMM2D_CUDA_TRY(cub::DeviceRadixSort::SortPairs(scratch, sb, kx, ksort, iota, ord, (int)n, 0, 64, st));
        k_make_recs<<<grid_for(n, BS), BS, 0, st>>>(ksort, ord, ys, 0, n, xl);
        fmm2d::note_launch();
        sb = cub_bytes;
        FMM2D_CUDA_TRY(cub::DeviceRadixSort::SortPairs(scratch, sb, ky, ksort, iota, ord, (int)n, 0, 64, st));
        k_make_recs<<<grid_for(n, BS), BS, 0, st>>>(ksort, ord, xs, 1, n, yl);
        fmm2d::note_launch();
        FMM2D_CUDA_TRY(cudaGetLastError());
        k_bbox<<<1, 32, 0, st>>>(xl, yl, P->boff + P->obase[0], 1, P->cx + P->base[0], P->cy + P->base[0],
                                 P->r + P->base[0]);
        fmm2d::note_launch();
        // one split step: partition `list` inside the parent segments (par_off) into the
        // sub-segments sub_off, comparing against `split` on `axis`
        auto split_step = [&](const Rec* list, const Rec* split, const uint32_t* refine, const uint32_t* par_off,
                              const uint32_t* sub_off, int64_t np, int axis, Rec* out) -> int {
            k_high_sizes<<<grid_for(np, BS), BS, 0, st>>>(par_off, sub_off, np, hs);
            fmm2d::note_launch();
            size_t b2 = cub_bytes;
            FMM2D_CUDA_TRY(cub::DeviceScan::ExclusiveSum(scratch, b2, hs, Gp, (int)np, st));
            FMM2D_CUDA_TRY(cudaMemsetAsync(tstate, 0, 8 * ntiles, st));
            FMM2D_CUDA_TRY(cudaMemsetAsync(ticket, 0, 4, st));
            k_partition<<<(unsigned)ntiles, PT, 0, st>>>(list, split, refine, par_off, sub_off, Gp, axis, n, out,
                                                        tstate, ticket);
            fmm2d::note_launch();
            FMM2D_CUDA_TRY(cudaGetLastError());
            return 0;
        };
        for (int l = 0; l < L; ++l) {
            const uint32_t* O = P->boff + P->obase[l];
            const uint32_t* H = P->boff + hbase[l];
            const uint32_t* C = P->boff + P->obase[l + 1];
            // x-split: the y-list (ids: half-level l-1/2, refined by O) is partitioned by
            // (x, idx) against the x-list's first high record
            const uint32_t* yref = (l == 0) ? nullptr : O;
            FMM2D_TRY(split_step(yl, xl, yref, O, H, nboxes(l), 0, tmp));
            std::swap(yl, tmp);
            // y-split of each half: the x-list (ids: level l, refined by H) is partitioned
            // by (y, idx) against the y-list's first high record
            FMM2D_TRY(split_step(xl, yl, H, H, C, 2 * nboxes(l), 1, tmp));
            std::swap(xl, tmp);
            int64_t nb = nboxes(l + 1);
            k_bbox<<<grid_for(nb, BS), BS, 0, st>>>(xl, yl, C, nb, P->cx + P->base[l + 1], P->cy + P->base[l + 1],
                                                    P->r + P->base[l + 1]);
            fmm2d::note_launch();
            FMM2D_CUDA_TRY(cudaGetLastError());
        }
        RadArgs A;
        for (int l = 0; l <= L; ++l) {
            A.cx[l] = P->cx + P->base[l];
            A.cy[l] = P->cy + P->base[l];
            A.r[l] = P->r + P->base[l];
        }
        k_finish<<<grid_for(n, FIN_T), FIN_T, 0, st>>>(yl, n, L, P->boff + P->obase[L], P->perm, P->src, A);
        fmm2d::note_launch();
        k_sqrt<<<grid_for(P->nbox_total, BS), BS, 0, st>>>(P->r, P->nbox_total);
        fmm2d::note_launch();
        FMM2D_CUDA_TRY(cudaGetLastError());
        return 0;
    };
    rc = body();
    tfree();
    return rc;
}

}  // namespace fmm2d
