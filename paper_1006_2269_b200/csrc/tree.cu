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
// so the y-split is the same step with the axes swapped.  Box sizes are a pure
// function of N, so all offsets are computed on the host.  The presort is two
// stable radix sorts of orderable 64-bit keys (ties leave in index order).
#include <cub/cub.cuh>

#include "fmm2d_internal.cuh"

namespace fmm2d {

namespace {

__device__ __forceinline__ uint64_t orderable(double v)
{
    uint64_t u = (uint64_t)__double_as_longlong(v);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
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

__global__ void k_make_recs(const uint32_t* __restrict__ order, const double* __restrict__ xs,
                            const double* __restrict__ ys, int64_t n, Rec* __restrict__ out)
{
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    uint32_t i = order[k];
    Rec r;
    r.x = xs[i];
    r.y = ys[i];
    r.idx = i;
    r.box = 0;
    out[k] = r;
}

// (coord, idx) < (coord', idx') on axis 0 = x, 1 = y  (DESIGN R6)
__device__ __forceinline__ bool rec_less(const Rec& a, const Rec& b, int axis)
{
    double ca = axis ? a.y : a.x, cb = axis ? b.y : b.x;
    return (ca < cb) || (ca == cb && a.idx < b.idx);
}

// Split step, part 1: flag = 1 if the record belongs to the high side of its parent
// segment p (= rec.box).  The high side of p starts at sub_off[2p+1] in split_list.
__global__ void k_flag(const Rec* __restrict__ list, const Rec* __restrict__ split_list,
                       const uint32_t* __restrict__ par_off, const uint32_t* __restrict__ sub_off,
                       int axis, int64_t n, uint32_t* __restrict__ flag)
{
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    Rec r = list[k];
    uint32_t p = r.box;
    uint32_t sp = sub_off[2 * p + 1];
    uint32_t f = 0;
    if (sp < par_off[p + 1]) {
        Rec s = split_list[sp];
        f = rec_less(r, s, axis) ? 0u : 1u;
    }
    flag[k] = f;
}

// Split step, part 2: stable scatter inside each parent segment; new box = 2p + side.
__global__ void k_scatter(const Rec* __restrict__ list, const uint32_t* __restrict__ flag,
                          const uint32_t* __restrict__ pos, const uint32_t* __restrict__ par_off,
                          const uint32_t* __restrict__ sub_off, int64_t n, Rec* __restrict__ out)
{
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    Rec r = list[k];
    uint32_t p = r.box;
    uint32_t s = par_off[p];
    uint32_t hi_before = pos[k] - pos[s];
    uint32_t f = flag[k];
    uint32_t dst = f ? sub_off[2 * p + 1] + hi_before : (uint32_t)k - hi_before;
    r.box = 2 * p + f;
    out[dst] = r;
}

// The list sorted along the split axis is already partitioned: just relabel.
__global__ void k_relabel(Rec* __restrict__ list, const uint32_t* __restrict__ sub_off, int64_t n)
{
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    uint32_t p = list[k].box;
    list[k].box = 2 * p + ((uint32_t)k >= sub_off[2 * p + 1] ? 1u : 0u);
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

// Final order: perm and the leaf-ordered source rows {x, y, 0, 0}.
__global__ void k_finish(const Rec* __restrict__ yl, int64_t n, uint32_t* __restrict__ perm,
                         double4* __restrict__ src)
{
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    Rec r = yl[k];
    perm[k] = r.idx;
    src[k] = make_double4(r.x, r.y, 0.0, 0.0);
}

// A2 (part 2): r = exact max distance (correctly rounded sqrt, no FMA).  One warp per
// (box, chunk of up to 32*ITEMS points); warp max, then atomicMax on the bit pattern
// (non-negative doubles order like their uint64 bits).
constexpr int RAD_ITEMS = 32;
__global__ void k_radius(const double4* __restrict__ src, const uint32_t* __restrict__ off,
                         int64_t nb, int chunks_per_box, const double* __restrict__ cx,
                         const double* __restrict__ cy, double* __restrict__ r)
{
    int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    int64_t b = w / chunks_per_box;
    if (b >= nb) return;
    int ch = (int)(w - b * chunks_per_box);
    uint32_t s = off[b], e = off[b + 1];
    uint32_t cs = s + (uint32_t)ch * (32 * RAD_ITEMS);
    if (cs >= e) return;
    uint32_t ce = min(e, cs + 32 * RAD_ITEMS);
    double c0 = cx[b], c1 = cy[b];
    double m = 0.0;
    for (uint32_t k = cs + lane; k < ce; k += 32) {
        double4 v = src[k];
        m = fmax(m, rn_dist(v.x, v.y, c0, c1));
    }
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0)
        atomicMax((unsigned long long*)(r + b), (unsigned long long)__double_as_longlong(m));
}

inline unsigned grid_for(int64_t n, int bs) { return (unsigned)((n + bs - 1) / bs); }

}  // namespace

// Host: offsets of every level and half-level, a pure function of n (DESIGN R5):
// a box of size s splits into x-halves (ceil(s/2), floor(s/2)), each half into
// (ceil(h/2), floor(h/2)).
static void host_offsets(int64_t n, int L, std::vector<std::vector<uint32_t>>& lev,
                         std::vector<std::vector<uint32_t>>& half)
{
    lev.assign(L + 1, {});
    half.assign(L, {});
    lev[0] = {0u, (uint32_t)n};
    for (int l = 0; l < L; ++l) {
        const auto& o = lev[l];
        int64_t nb = nboxes(l);
        auto& h = half[l];
        auto& c = lev[l + 1];
        h.resize(2 * nb + 1);
        c.resize(4 * nb + 1);
        for (int64_t b = 0; b < nb; ++b) {
            uint32_t s = o[b], sz = o[b + 1] - o[b];
            uint32_t h0 = sz - sz / 2, h1 = sz / 2;
            h[2 * b] = s;
            h[2 * b + 1] = s + h0;
            c[4 * b] = s;
            c[4 * b + 1] = s + (h0 - h0 / 2);
            c[4 * b + 2] = s + h0;
            c[4 * b + 3] = s + h0 + (h1 - h1 / 2);
        }
        h[2 * nb] = (uint32_t)n;
        c[4 * nb] = (uint32_t)n;
    }
}

int build_tree(fmm2d_plan* P, const double2* z)
{
    const int64_t n = P->n;
    const int L = P->L;
    cudaStream_t st = P->stream;
    const int BS = 256;

    // ---- offsets (host) -> device: level l at obase[l]; half-levels after them
    std::vector<std::vector<uint32_t>> lev, half;
    host_offsets(n, L, lev, half);
    P->obase.assign(L + 1, 0);
    std::vector<int64_t> hbase(L, 0);
    int64_t tot = 0;
    for (int l = 0; l <= L; ++l) { P->obase[l] = tot; tot += (int64_t)lev[l].size(); }
    for (int l = 0; l < L; ++l) { hbase[l] = tot; tot += (int64_t)half[l].size(); }
    P->h_boff.resize(tot);
    for (int l = 0; l <= L; ++l) std::copy(lev[l].begin(), lev[l].end(), P->h_boff.begin() + P->obase[l]);
    for (int l = 0; l < L; ++l) std::copy(half[l].begin(), half[l].end(), P->h_boff.begin() + hbase[l]);
    FMM2D_TRY(dev_alloc(P, (void**)&P->boff, sizeof(uint32_t) * tot));
    FMM2D_CUDA_TRY(cudaMemcpyAsync(P->boff, P->h_boff.data(), sizeof(uint32_t) * tot,
                                   cudaMemcpyHostToDevice, st));
    {
        uint32_t mn = UINT32_MAX, mx = 0;
        const auto& o = lev[L];
        for (size_t b = 0; b + 1 < o.size(); ++b) {
            mn = std::min(mn, o[b + 1] - o[b]);
            mx = std::max(mx, o[b + 1] - o[b]);
        }
        P->stats.min_leaf = (int)mn;
        P->stats.max_leaf = (int)mx;
    }

    // ---- scratch
    double *xs, *ys;
    uint64_t *kx, *ky, *ksort;
    uint32_t *iota, *ord, *flag, *pos;
    Rec *xl, *yl, *tmp;
    int* bad;
    void* scratch = nullptr;
    size_t sort_bytes = 0, scan_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (uint64_t*)nullptr, (uint64_t*)nullptr,
                                    (uint32_t*)nullptr, (uint32_t*)nullptr, (int)n, 0, 64, st);
    cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)n, st);
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
        if ((rc = talloc((void**)&flag, 4 * n))) break;
        if ((rc = talloc((void**)&pos, 4 * n))) break;
        if ((rc = talloc((void**)&xl, sizeof(Rec) * n))) break;
        if ((rc = talloc((void**)&yl, sizeof(Rec) * n))) break;
        if ((rc = talloc((void**)&tmp, sizeof(Rec) * n))) break;
        if ((rc = talloc((void**)&bad, sizeof(int)))) break;
        if ((rc = talloc(&scratch, cub_bytes))) break;
    } while (0);
    if (rc) { tfree(); return rc; }

    auto body = [&]() -> int {
        FMM2D_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), st));
        k_canon<<<grid_for(n, BS), BS, 0, st>>>(z, n, xs, ys, kx, ky, iota, bad); fmm2d::note_launch();
        FMM2D_CUDA_TRY(cudaGetLastError());
        int h_bad = 0;
        FMM2D_CUDA_TRY(cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
        FMM2D_CUDA_TRY(cudaStreamSynchronize(st));
        if (h_bad) return FMM2D_ENONFINITE;
        // presort (stable LSD radix: ties stay in index order)
        size_t sb = cub_bytes;
        FMM2D_CUDA_TRY(cub::DeviceRadixSort::SortPairs(scratch, sb, kx, ksort, iota, ord, (int)n, 0, 64, st));
        k_make_recs<<<grid_for(n, BS), BS, 0, st>>>(ord, xs, ys, n, xl); fmm2d::note_launch();
        sb = cub_bytes;
        FMM2D_CUDA_TRY(cub::DeviceRadixSort::SortPairs(scratch, sb, ky, ksort, iota, ord, (int)n, 0, 64, st));
        k_make_recs<<<grid_for(n, BS), BS, 0, st>>>(ord, xs, ys, n, yl); fmm2d::note_launch();
        FMM2D_CUDA_TRY(cudaGetLastError());
        // level 0 bbox
        k_bbox<<<1, 32, 0, st>>>(xl, yl, P->boff + P->obase[0], 1, P->cx + P->base[0], P->cy + P->base[0],
                                 P->r + P->base[0]); fmm2d::note_launch();
        for (int l = 0; l < L; ++l) {
            const uint32_t* O = P->boff + P->obase[l];
            const uint32_t* H = P->boff + hbase[l];
            const uint32_t* C = P->boff + P->obase[l + 1];
            // x-split: y-list partitioned by (x, idx) against the x-list's first high record
            k_flag<<<grid_for(n, BS), BS, 0, st>>>(yl, xl, O, H, 0, n, flag); fmm2d::note_launch();
            sb = cub_bytes;
            FMM2D_CUDA_TRY(cub::DeviceScan::ExclusiveSum(scratch, sb, flag, pos, (int)n, st));
            k_scatter<<<grid_for(n, BS), BS, 0, st>>>(yl, flag, pos, O, H, n, tmp); fmm2d::note_launch();
            std::swap(yl, tmp);
            k_relabel<<<grid_for(n, BS), BS, 0, st>>>(xl, H, n); fmm2d::note_launch();
            // y-split of each half: x-list partitioned by (y, idx) against the y-list
            k_flag<<<grid_for(n, BS), BS, 0, st>>>(xl, yl, H, C, 1, n, flag); fmm2d::note_launch();
            sb = cub_bytes;
            FMM2D_CUDA_TRY(cub::DeviceScan::ExclusiveSum(scratch, sb, flag, pos, (int)n, st));
            k_scatter<<<grid_for(n, BS), BS, 0, st>>>(xl, flag, pos, H, C, n, tmp); fmm2d::note_launch();
            std::swap(xl, tmp);
            k_relabel<<<grid_for(n, BS), BS, 0, st>>>(yl, C, n); fmm2d::note_launch();
            int64_t nb = nboxes(l + 1);
            k_bbox<<<grid_for(nb, BS), BS, 0, st>>>(xl, yl, C, nb, P->cx + P->base[l + 1],
                                                    P->cy + P->base[l + 1], P->r + P->base[l + 1]); fmm2d::note_launch();
            FMM2D_CUDA_TRY(cudaGetLastError());
        }
        // leaf order = the final y-list (leaves in index order, (y, idx) inside, R13)
        k_finish<<<grid_for(n, BS), BS, 0, st>>>(yl, n, P->perm, P->src); fmm2d::note_launch();
        for (int l = 0; l <= L; ++l) {
            int64_t nb = nboxes(l);
            uint32_t maxsz = 0;
            const auto& o = lev[l];
            for (int64_t b = 0; b < std::min<int64_t>(nb, 2); ++b) maxsz = std::max(maxsz, o[b + 1] - o[b]);
            maxsz = (uint32_t)((n + nb - 1) / nb);
            int cpb = (int)((maxsz + 32 * RAD_ITEMS - 1) / (32 * RAD_ITEMS));
            int64_t warps = nb * cpb;
            k_radius<<<grid_for(warps * 32, BS), BS, 0, st>>>(P->src, P->boff + P->obase[l], nb, cpb,
                                                              P->cx + P->base[l], P->cy + P->base[l],
                                                              P->r + P->base[l]); fmm2d::note_launch();
        }
        FMM2D_CUDA_TRY(cudaGetLastError());
        return 0;
    };
    rc = body();
    tfree();
    return rc;
}

}  // namespace fmm2d
