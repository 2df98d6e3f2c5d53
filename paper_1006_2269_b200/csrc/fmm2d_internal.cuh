// fmm2d_internal.cuh -- plan layout and shared device helpers of libfmm2d.so.
//
// Product code (sm_100a).  Shares nothing with oracle/ (see DESIGN.md section 3).
// Layout in HBM:
//   boxes of all levels are numbered globally, level l occupying
//   [base[l], base[l] + 4^l) with base[l] = (4^l - 1)/3;
//   per-box SoA discs cx, cy, r (f64); expansions box-major double2[box][p+1];
//   leaf-ordered sources double4 {x, y, Re m, Im m} (32 B, one 256-bit row each);
//   lists per level as CSR (int64 offsets over the level's boxes, uint32 level-local ids).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <utility>
#include <vector>

#include "../../include/fmm2d.h"

#define FMM2D_MAXL 15
#ifndef FMM2D_NEAR_CHUNK
#define FMM2D_NEAR_CHUNK 384        // k_near: source rows staged per chunk (C5: one chunk per leaf)
#endif
#ifndef FMM2D_NEAR_SPLIT
#define FMM2D_NEAR_SPLIT 4096       // near lists with more source rows: split over several CTAs
#endif
#ifndef FMM2D_RR_SHORT
#define FMM2D_RR_SHORT 8            // r/R exchange: P2L / M2P lists up to this long take a warp, longer a block
#endif
#ifndef FMM2D_M2L_LONG
#define FMM2D_M2L_LONG 96           // weak lists longer than this: one warp per target (k_m2l_long)
#endif

namespace fmm2d {

static inline int64_t nboxes(int l) { return (int64_t)1 << (2 * l); }
static inline int64_t level_base(int l) { return (nboxes(l) - 1) / 3; }

struct Csr {
    int64_t* off = nullptr;   // device, 4^l + 1
    uint32_t* idx = nullptr;  // device, off[4^l] entries (level-local box ids)
    int64_t total = 0;
};

// a part of a long leaf strong list, evaluated by its own k_near CTA (partial sums)
struct NearSeg {
    int64_t qa, qb;      // list entries [qa, qb)
    uint32_t t, pad;     // target leaf
};

struct Stats {
    double t_build_ms = 0, t_tree_ms = 0, t_lists_ms = 0;
    int64_t weak_pairs = 0, strong_leaf_pairs = 0, p2p_pairs = 0;
    int max_leaf = 0, min_leaf = 0;
    int tree_key64 = 0;                // axes presorted with 64-bit keys (bit 0 x, bit 1 y)
    int64_t dev_bytes = 0;             // device memory the plan holds (its allocations)
};

}  // namespace fmm2d

namespace fmm2d {
struct Shard;   // shard.cu: exchange tables and buffers of a sharded plan
}

struct fmm2d_plan {
    int64_t n = 0;
    int L = 0, p = 0, flags = 0, device = 0;
    double theta = 0.5;
    cudaStream_t stream = nullptr;
    // partition: levels <= kpart are replicated on every rank,
    // levels > kpart hold the rank's own subtrees [rank 4^l / P, (rank+1) 4^l / P).
    // One GPU: nranks = 1, kpart = 0 (every box is "own").
    int nranks = 1, rank = 0, kpart = 0;
    uint32_t pos0 = 0, pos1 = 0;        // own source positions (leaf order)
    int64_t own_lo(int l) const { return (nboxes_(l) / nranks) * rank; }          // l >= kpart
    int64_t own_hi(int l) const { return (nboxes_(l) / nranks) * (rank + 1); }
    int64_t box_lo(int l) const { return (l <= kpart) ? 0 : own_lo(l); }           // boxes computed
    int64_t box_hi(int l) const { return (l <= kpart) ? nboxes_(l) : own_hi(l); }
    static int64_t nboxes_(int l) { return (int64_t)1 << (2 * l); }
    fmm2d::Shard* shard = nullptr;      // nranks > 1
    int64_t nbox_total = 0;
    std::vector<int64_t> base;          // base[l], l = 0..L+1
    // offsets of every level (uint32, n < 2^31), concatenated: level l at obase[l]
    uint32_t* boff = nullptr;
    std::vector<int64_t> obase;
    // tree outputs
    uint32_t* perm = nullptr;           // [n] leaf position -> input index
    double4* src = nullptr;             // [n] leaf-ordered {x, y, Re m, Im m}
    double *cx = nullptr, *cy = nullptr, *r = nullptr;   // [nbox_total]
    // connectivity
    std::vector<fmm2d::Csr> strong, weak;   // per level
    std::vector<fmm2d::Csr> xweak;          // per level: cross-level weak entries (parent merge; ids of level l-1)
    uint32_t* m2l_order = nullptr;      // M2L targets per level (levels 1..L concatenated), by list length
    uint32_t* m2l_long = nullptr;       // global ids of targets with more than FMM2D_M2L_LONG weak pairs
    int64_t m2l_nlong = 0;
    // leaf-level direct pairs: the strong lists, or with FMM2D_RR_EXCHANGE the strong lists less
    // the conversions: P2L into the smaller leaf, M2P of the smaller leaf
    fmm2d::Csr near, rr_p2l, rr_m2p;
    uint32_t* rr_p2l_leaves = nullptr;  // leaves with a non-empty P2L / M2P list
    uint32_t* rr_m2p_leaves = nullptr;
    int64_t rr_np2l = 0, rr_nm2p = 0;
    // short lists (<= FMM2D_RR_SHORT entries) at [0, *_short), long ones at [cap - (n - short), cap)
    int64_t rr_np2l_short = 0, rr_nm2p_short = 0, rr_leaf_cap = 0;
    double4* rr_acc = nullptr;          // [n] M2P sums (leaf order; valid on leaves with M2P work)
    // long near lists split into segments of at most FMM2D_NEAR_SPLIT source rows
    int64_t* near_seg_off = nullptr;    // [leaves + 1] segments of each leaf (empty: not split)
    fmm2d::NearSeg* near_segs = nullptr;
    uint32_t* near_split = nullptr;     // split leaves
    double4* near_part = nullptr;       // [segments][max_leaf] partial sums
    int64_t near_nseg = 0, near_nsplit = 0;
    // expansions.  Storage per level: every box of the replicated levels l <= kpart, the own
    // boxes [own_lo(l), own_hi(l)) of the levels below (one GPU: every box of every level, in
    // global box order, so mpole + g (p+1) is box g).  mpl[l] / lcl[l] point such that
    // mpl[l] + b (p+1) is level-l box b for every STORED b (a per-level virtual base).
    double2* mpole = nullptr;           // storage (one GPU: [nbox_total][p+1])
    double2* local = nullptr;
    double2* mpl[FMM2D_MAXL + 1] = {};
    double2* lcl[FMM2D_MAXL + 1] = {};
    // sharded plans: halo multipoles live in the import buffer (shard->mp.recv, slot = import
    // order); hmap[global box id] = the slot of an imported box
    const double2* mhalo = nullptr;
    uint32_t* hmap = nullptr;
    // sharded plans: source rows / input indices of the own positions only (src, perm are
    // virtual bases: src[k] valid for k in [pos0, pos1)); halo leaves' rows in hsrc / hperm,
    // leaf lf of the halo at hsrc + lmap[lf] (lmap = ~0 for every other leaf)
    double4* hsrc = nullptr;
    uint32_t* hperm = nullptr;
    uint32_t* lmap = nullptr;
    // staging for FMM2D_HOST_PTRS
    double2* mstage = nullptr;
    // strengths (input order) whose gather into the source rows is left to P2M, which reads
    // those rows anyway (set by eval_impl for one evaluation; nullptr: rows already hold m)
    const double2* m_fused = nullptr;
    double2* phistage = nullptr;
    double2* dphistage = nullptr;
    const void* tables = nullptr;       // fastmath tables (device, shared per device)
    // overlapped eval: the expansion chain on a high-priority side stream while k_near's
    // P2P runs on the plan's stream; k_near_final joins them
    bool overlap = false;
    int64_t m2l_cap = 0;                // > 0: M2L from this many single-warp blocks (overlap)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_gather = nullptr, ev_exp = nullptr;
    double4* nacc = nullptr;            // [n] P2P sums (leaf order)
    // symmetric near field (near.cu): each unordered leaf pair evaluated once
    bool sym = false;
    int sym_tile = 0, sym_npass = 0, sym_rows = 0, slot_w = 0;
    uint32_t* sym_mirror = nullptr;     // [strong leaf entries] position of t in row s
    uint32_t* sym_selfpos = nullptr;    // [leaves] position of t in its own row = |lower(t)|
    int64_t* sym_lower = nullptr;       // [leaves + 1] exclusive scan of sym_selfpos
    double4* sym_slot = nullptr;        // [lower entries][slot_w] partial sums (Phi, Phi')
    double4* sym_t = nullptr;           // [n] own-CTA sums + L2P, leaf order
    fmm2d::Stats stats;
    std::vector<void*> allocs;          // everything to free
};

// ---------------------------------------------------------------- helpers
namespace fmm2d {

int dev_alloc(fmm2d_plan* P, void** ptr, size_t bytes);
// Every device allocation of the library comes from ONE library-owned stream-ordered pool per
// device (created on first use, release threshold = keep everything), never from the device's
// default pool, whose attributes the library leaves alone (fmm2d_release_pool trims it).
cudaMemPool_t lib_pool(int device);
cudaError_t pool_malloc(void** ptr, size_t bytes, cudaStream_t st);

// build steps (tree.cu, lists.cu)
int build_tree(fmm2d_plan* P, const double2* z_dev);
int finish_radii(fmm2d_plan* P);
int build_lists(fmm2d_plan* P);
// eval steps (expansions.cu, near.cu)
int run_upward(fmm2d_plan* P);
int run_m2l(fmm2d_plan* P);
int run_downward(fmm2d_plan* P);
int run_near(fmm2d_plan* P, double2* phi, double2* dphi, int mode);
int prepare_near(fmm2d_plan* P);
int prepare_near_sym(fmm2d_plan* P);
int gather_strengths(fmm2d_plan* P, const double2* m);
int run_upward_top(fmm2d_plan* P);
int run_rr_p2l(fmm2d_plan* P);
// M2L kernel arguments (expansions.cu) and the log-term kernel (rr.cu, beside the table-driven
// log / Arg): adds sum_s a_0(s) Log(c_t - c_s) to coefficient 0 of every short-list target
struct M2LArgs {
    const int64_t* woff[FMM2D_MAXL + 1];
    const uint32_t* widx[FMM2D_MAXL + 1];
    const int64_t* xoff[FMM2D_MAXL + 1];     // cross-level entries (parent merge) or nullptr
    const uint32_t* xidx[FMM2D_MAXL + 1];
    int64_t base[FMM2D_MAXL + 2];
    int64_t lo[FMM2D_MAXL + 1];       // target boxes of level l: [lo[l], lo[l] + (pre[l+1] - pre[l]))
    int64_t pre[FMM2D_MAXL + 2];      // work prefix over levels 1..L
    const uint32_t* order;            // [pre[L+1]] target box of each work item (level-local id)
    int L;
    const double* cx;
    const double* cy;
    // per level: stored expansions (level-local box b at mpl[l] + b (p+1)) and the stored
    // range [slo, shi) -- one GPU: every box; other sources are imported (mhalo + hmap)
    const double2* mpl[FMM2D_MAXL + 1];
    double2* lcl[FMM2D_MAXL + 1];
    int64_t slo[FMM2D_MAXL + 1], shi[FMM2D_MAXL + 1];
    const double2* mhalo;
    const uint32_t* hmap;             // [global box id] import slot
};
int m2l_log_terms(fmm2d_plan* P, const M2LArgs& A, int p1);
int run_rr_m2p(fmm2d_plan* P);
// sharding (shard.cu)
int64_t box_start_host(int64_t n, int l, int64_t b);
int partition_level(int nranks);
int shard_setup(fmm2d_plan* P, int nranks, int rank, const void* nccl_id);
void shard_free(fmm2d_plan* P);
int shard_build_rest(fmm2d_plan* const* Ps, int np);
int shard_gather_halo(fmm2d_plan* P, const double2* m);
int shard_comm_top(fmm2d_plan* const* Ps, int np);
int shard_pack_mp(fmm2d_plan* P);
int shard_comm_mp(fmm2d_plan* const* Ps, int np);
int shard_unpack_mp(fmm2d_plan* P);
bool shard_has_comm(const fmm2d_plan* P);
int shard_allreduce_sum_u32(fmm2d_plan* P, unsigned int* buf, size_t count);
int shard_allgather_inplace(fmm2d_plan* P, void* base, size_t bytes_per_rank);
int shard_gather_output(fmm2d_plan* P, double2* phi, double2* dphi);
void shard_halo_sizes(const fmm2d_plan* P, int64_t* leaves, int64_t* mpoles, int64_t* exp_leaves, int64_t* exp_mp);
int nccl_unique_id(void* out);
int upload_binomials(int p);
// count of this library's own kernel launches (reported by bench.py as gpu_launches)
void note_launch();
int64_t launch_count();

// FMM2D_TREE_TRACE=1: event times of the build's phases on stderr (diagnostics only)
struct PhaseTrace {
    cudaStream_t st;
    bool on;
    std::vector<std::pair<std::string, cudaEvent_t>> ev;
    explicit PhaseTrace(cudaStream_t s) : st(s), on(std::getenv("FMM2D_TREE_TRACE") != nullptr) {}
    void mark(const std::string& name)
    {
        if (!on) return;
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return;
        cudaEventRecord(e, st);
        ev.emplace_back(name, e);
    }
    ~PhaseTrace()
    {
        if (!on || ev.empty()) return;
        cudaEventSynchronize(ev.back().second);
        for (size_t i = 1; i < ev.size(); ++i) {
            float ms = 0;
            cudaEventElapsedTime(&ms, ev[i - 1].second, ev[i].second);
            std::fprintf(stderr, "[fmm2d tree] %-28s %9.3f ms\n", ev[i].first.c_str(), ms);
        }
        for (auto& x : ev) cudaEventDestroy(x.second);
    }
};

}  // namespace fmm2d

#define FMM2D_CUDA_TRY(expr)                                  \
    do {                                                      \
        cudaError_t _e = (expr);                              \
        if (_e != cudaSuccess) {                              \
            fmm2d_set_last_cuda_error(_e, #expr, __FILE__, __LINE__); \
            return (_e == cudaErrorMemoryAllocation) ? FMM2D_ENOMEM : FMM2D_ECUDA; \
        }                                                     \
    } while (0)

#define FMM2D_TRY(expr)                                       \
    do {                                                      \
        int _rc = (expr);                                     \
        if (_rc) return _rc;                                  \
    } while (0)

void fmm2d_set_last_cuda_error(cudaError_t e, const char* what, const char* file, int line);
void fmm2d_set_last_error_text(const char* msg, const char* what, const char* file, int line);

// IEEE round-to-nearest helpers with no FMA contraction (DESIGN R11).  The squared
// distance is what the radius pass maximises: sqrt_rn is monotone, so
// sqrt_rn(max d^2) == max sqrt_rn(d^2) bit for bit (the oracle's order).
__device__ __forceinline__ double rn_dist2(double x, double y, double cx, double cy)
{
    double dx = __dsub_rn(x, cx);
    double dy = __dsub_rn(y, cy);
    return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
}
