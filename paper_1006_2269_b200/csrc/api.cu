// api.cu -- the C ABI of libfmm2d.so (include/fmm2d.h): plan life cycle and the
// orchestration of the build (A0-A3) and evaluation (A4-A11) passes on one stream.
//
// Paper order: mesh first, then connectivity, then upward shifts,
// far-to-local shifts along the weak pattern, downward shifts, and the direct
// near field at the finest level.
#include <atomic>
#include <mutex>
#include <cstdio>
#include <cstring>
#include <new>

#include "fmm2d_internal.cuh"

static thread_local char g_last_err[512] = "";

void fmm2d_set_last_cuda_error(cudaError_t e, const char* what, const char* file, int line)
{
    snprintf(g_last_err, sizeof(g_last_err), "%s: %s (%s:%d)", cudaGetErrorString(e), what, file, line);
}

void fmm2d_set_last_error_text(const char* msg, const char* what, const char* file, int line)
{
    snprintf(g_last_err, sizeof(g_last_err), "%s: %s (%s:%d)", msg ? msg : "", what, file, line);
}

namespace fmm2d {

static std::atomic<int64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
int64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

cudaMemPool_t lib_pool(int device)
{
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {nullptr};
    if (device < 0 || device >= 64) return nullptr;
    std::lock_guard<std::mutex> lk(mu);
    if (!pools[device]) {
        cudaMemPoolProps props;
        memset(&props, 0, sizeof(props));
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        cudaMemPool_t pool = nullptr;
        if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) return nullptr;
        // keep freed memory for the next build / evaluation (no page mapping in a timed path);
        // fmm2d_pool_trim gives it back
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        pools[device] = pool;
    }
    return pools[device];
}

cudaError_t pool_malloc(void** ptr, size_t bytes, cudaStream_t st)
{
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    cudaMemPool_t pool = lib_pool(dev);
    if (!pool) return cudaErrorMemoryAllocation;
    return cudaMallocFromPoolAsync(ptr, bytes ? bytes : 16, pool, st);
}

int dev_alloc(fmm2d_plan* P, void** ptr, size_t bytes)
{
    *ptr = nullptr;
    if (bytes == 0) bytes = 16;
    cudaError_t e = fmm2d::pool_malloc((void**)ptr, bytes, P->stream);
    if (e != cudaSuccess) {
        fmm2d_set_last_cuda_error(e, "cudaMallocAsync", __FILE__, __LINE__);
        *ptr = nullptr;
        return FMM2D_ENOMEM;
    }
    P->allocs.push_back(*ptr);
    P->stats.dev_bytes += (int64_t)bytes;
    return 0;
}

}  // namespace fmm2d

using namespace fmm2d;

extern "C" {

const char* fmm2d_last_error_detail(void) { return g_last_err; }

int fmm2d_default_options(fmm2d_options* opt)
{
    if (!opt) return FMM2D_EINVAL;
    memset(opt, 0, sizeof(*opt));
    opt->theta = 0.5;
    opt->p = 17;
    opt->leaf_target = 40;
    opt->nlevels = -1;
    opt->flags = 0;
    opt->device = 0;
    opt->stream = nullptr;
    opt->nranks = 1;
    opt->rank = 0;
    opt->nccl_id = nullptr;
    return 0;
}

const char* fmm2d_strerror(int code)
{
    switch (code) {
        case FMM2D_OK: return "ok";
        case FMM2D_EINVAL: return "invalid argument";
        case FMM2D_ENONFINITE: return "non-finite coordinate";
        case FMM2D_ENOMEM: return "out of memory";
        case FMM2D_ECUDA: return "CUDA error";
        case FMM2D_ENCCL: return "NCCL error";
        case FMM2D_ENOTSUP: return "unsupported option";
        default: return "unknown error";
    }
}

void fmm2d_free(fmm2d_plan* P)
{
    if (!P) return;
    cudaSetDevice(P->device);
    if (P->side) cudaStreamSynchronize(P->side);
    for (void* p : P->allocs) cudaFreeAsync(p, P->stream);
    cudaStreamSynchronize(P->stream);
    if (P->side) cudaStreamDestroy(P->side);
    if (P->ev_gather) cudaEventDestroy(P->ev_gather);
    if (P->ev_exp) cudaEventDestroy(P->ev_exp);
    shard_free(P);
    delete P;
}

// DESIGN R4: L = min L >= 0 with n <= 2 * leaf_target * 4^L.
static int depth_rule(int64_t n, int leaf_target)
{
    int L = 0;
    int64_t cap = 2 * (int64_t)leaf_target;
    while (n > cap && L < FMM2D_MAXL) { cap *= 4; ++L; }
    return L;
}

// validated depth of the tree for n points (or a negative error code)
static int plan_depth(int64_t n, const fmm2d_options* opt)
{
    if (!(opt->theta > 0.0 && opt->theta < 1.0)) return FMM2D_EINVAL;        // P:119, not clamped
    if (opt->p < 1 || opt->p > FMM2D_PMAX) return FMM2D_EINVAL;
    if (n < 1 || n >= ((int64_t)1 << 31)) return FMM2D_EINVAL;
    int L;
    if (opt->nlevels >= 0) {
        L = opt->nlevels;
        if (L > FMM2D_MAXL) return FMM2D_EINVAL;
        if (n < nboxes(L) && !(opt->flags & FMM2D_MIDPOINT)) return FMM2D_EINVAL;   // DESIGN R12
    } else {
        if (opt->leaf_target < 1) return FMM2D_EINVAL;
        L = depth_rule(n, opt->leaf_target);
        while (L > 0 && n < nboxes(L)) --L;
    }
    return L;
}

// Stage 1 of a build: plan fields, partition, allocations, the tree (A0-A2).  For one
// GPU it also runs the lists (A3).  Sharded plans continue in shard_build_rest.
static int build_stage_tree(const double* z, int64_t n, const fmm2d_options* opt, int nranks, int rank,
                            const void* nccl_id, fmm2d_plan** out, bool loopback = false)
{
    *out = nullptr;
    const int L = plan_depth(n, opt);
    if (L < 0) return L;
    if (nranks < 1 || rank < 0 || rank >= nranks) return FMM2D_EINVAL;
    if (nranks > 1 && (opt->flags & (FMM2D_RR_EXCHANGE | FMM2D_MIDPOINT))) return FMM2D_ENOTSUP;
    if ((opt->flags & FMM2D_MIDPOINT) && L > 15) return FMM2D_EINVAL;          // 30-bit leaf keys
    if (nranks > 1) {                                   // partitionable? (before any device work)
        const int k = partition_level(nranks);
        if (k < 0 || L <= k) return FMM2D_ENOTSUP;
    }
    if (cudaSetDevice(opt->device) != cudaSuccess) return FMM2D_ECUDA;
    fmm2d_plan* P = new (std::nothrow) fmm2d_plan();
    if (!P) return FMM2D_ENOMEM;
    P->n = n;
    P->L = L;
    P->p = opt->p;
    P->theta = opt->theta;
    P->flags = opt->flags;
    P->device = opt->device;
    P->stream = (cudaStream_t)opt->stream;
    P->base.resize(L + 2);
    for (int l = 0; l <= L + 1; ++l) P->base[l] = level_base(l);
    P->nbox_total = P->base[L + 1];
    P->pos0 = 0;
    P->pos1 = (uint32_t)n;

    auto body = [&]() -> int {
        FMM2D_TRY(shard_setup(P, nranks, rank, nccl_id));
        cudaEvent_t e0, e1, e2;
        FMM2D_CUDA_TRY(cudaEventCreate(&e0));
        FMM2D_CUDA_TRY(cudaEventCreate(&e1));
        FMM2D_CUDA_TRY(cudaEventCreate(&e2));
        FMM2D_CUDA_TRY(cudaEventRecord(e0, P->stream));
        FMM2D_TRY(upload_binomials(P->p));
        FMM2D_TRY(prepare_near(P));
        const int64_t nb = P->nbox_total;
        const int P1 = P->p + 1;
        // leaf-ordered rows and input indices of the own positions [pos0, pos1) only (one
        // GPU: all n); src / perm are virtual bases indexed by the global position
        const int64_t nown = (int64_t)P->pos1 - (int64_t)P->pos0;
        FMM2D_TRY(dev_alloc(P, (void**)&P->perm, sizeof(uint32_t) * nown));
        FMM2D_TRY(dev_alloc(P, (void**)&P->src, sizeof(double4) * nown));
        P->perm -= P->pos0;
        P->src -= P->pos0;
        FMM2D_TRY(dev_alloc(P, (void**)&P->cx, sizeof(double) * nb));
        FMM2D_TRY(dev_alloc(P, (void**)&P->cy, sizeof(double) * nb));
        FMM2D_TRY(dev_alloc(P, (void**)&P->r, sizeof(double) * nb));
        // expansions of the stored boxes of every level (replicated levels: all, below: own)
        int64_t sbase[FMM2D_MAXL + 2], stot = 0;
        for (int l = 0; l <= L; ++l) {
            sbase[l] = stot;
            stot += P->box_hi(l) - P->box_lo(l);
        }
        FMM2D_TRY(dev_alloc(P, (void**)&P->mpole, sizeof(double2) * stot * P1));
        FMM2D_TRY(dev_alloc(P, (void**)&P->local, sizeof(double2) * stot * P1));
        for (int l = 0; l <= L; ++l) {
            P->mpl[l] = P->mpole + (sbase[l] - P->box_lo(l)) * P1;
            P->lcl[l] = P->local + (sbase[l] - P->box_lo(l)) * P1;
        }
        const double2* zd = (const double2*)z;
        double2* zstage = nullptr;
        if (P->flags & FMM2D_HOST_PTRS) {
            FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&zstage, sizeof(double2) * n, P->stream));
            FMM2D_CUDA_TRY(cudaMemcpyAsync(zstage, z, sizeof(double2) * n, cudaMemcpyHostToDevice, P->stream));
            zd = zstage;
        }
        int rc = build_tree(P, zd);
        if (zstage) cudaFreeAsync(zstage, P->stream);
        if (rc) return rc;
        FMM2D_CUDA_TRY(cudaEventRecord(e1, P->stream));
        if (P->nranks == 1) {
            FMM2D_TRY(build_lists(P));
            FMM2D_TRY(prepare_near_sym(P));
        }
        // overlapped evaluation (DESIGN 6.4): not for loopback shards (one shared stream)
        if ((P->flags & FMM2D_OVERLAP) && !loopback && P->L >= 1 && !P->sym &&
            P->stats.max_leaf <= FMM2D_NEAR_CHUNK) {
            int lo = 0, hi = 0;
            FMM2D_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            FMM2D_CUDA_TRY(cudaStreamCreateWithPriority(&P->side, cudaStreamNonBlocking, hi));
            FMM2D_CUDA_TRY(cudaEventCreateWithFlags(&P->ev_gather, cudaEventDisableTiming));
            FMM2D_CUDA_TRY(cudaEventCreateWithFlags(&P->ev_exp, cudaEventDisableTiming));
            FMM2D_TRY(dev_alloc(P, (void**)&P->nacc, sizeof(double4) * ((int64_t)P->pos1 - P->pos0)));
            P->nacc -= P->pos0;                 // virtual base, like src
            P->overlap = true;
        }
        FMM2D_CUDA_TRY(cudaEventRecord(e2, P->stream));
        FMM2D_CUDA_TRY(cudaEventSynchronize(e2));
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, e0, e1);
        cudaEventElapsedTime(&b, e1, e2);
        P->stats.t_tree_ms = a;
        P->stats.t_lists_ms = b;
        P->stats.t_build_ms = a + b;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaEventDestroy(e2);
        return 0;
    };
    int rc = body();
    if (rc) {
        fmm2d_free(P);
        return rc;
    }
    *out = P;
    return 0;
}

int fmm2d_build(const double* z, int64_t n, const fmm2d_options* opt, fmm2d_plan** out)
{
    if (!out) return FMM2D_EINVAL;
    *out = nullptr;
    if (!z || !opt) return FMM2D_EINVAL;
    const int R = opt->nranks, r = opt->rank;
    if (R < 1 || r < 0 || r >= R) return FMM2D_EINVAL;
    if (R > 1 && !opt->nccl_id) return FMM2D_EINVAL;
    fmm2d_plan* P = nullptr;
    FMM2D_TRY(build_stage_tree(z, n, opt, R, r, opt->nccl_id, &P));
    if (R > 1) {
        const int rc = shard_build_rest(&P, 1);
        if (rc) {
            fmm2d_free(P);
            return rc;
        }
    }
    *out = P;
    return 0;
}

static int eval_impl(fmm2d_plan* const* Ps, int np, const double* m, double* phi, double* dphi, cudaEvent_t* ev);

int fmm2d_build_eval(const double* z, const double* m, int64_t n, const fmm2d_options* opt, double* phi,
                     double* dphi, fmm2d_plan** out)
{
    if (!out) return FMM2D_EINVAL;
    *out = nullptr;
    if (!z || !m || !opt) return FMM2D_EINVAL;
    if (opt->nranks != 1) return FMM2D_ENOTSUP;
    if (!(opt->flags & FMM2D_HOST_PTRS)) {
        FMM2D_TRY(fmm2d_build(z, n, opt, out));
        const int rc = fmm2d_eval(*out, m, phi, dphi);
        if (rc) {
            fmm2d_free(*out);
            *out = nullptr;
        }
        return rc;
    }
    if (n < 1) return FMM2D_EINVAL;
    FMM2D_CUDA_TRY(cudaSetDevice(opt->device));
    // streams: the build (positions' copy + build kernels) on a HIGH-priority stream of its
    // own, the strengths' copy on a second one behind the positions' copy, the evaluation
    // and the results' copies on the caller's stream.  With another problem's evaluation
    // in flight (FMM2D_ASYNC_HOST, two streams), the build's CTAs are dispatched ahead of
    // that evaluation's instead of queueing behind all of them.
    // The two internal streams are created once per device and kept: allocations made on
    // them are then reused from the memory pool call after call (a fresh stream per call
    // made the pool grow now and then, a host stall of tens of ms).
    cudaStream_t st = (cudaStream_t)opt->stream;
    cudaStream_t bst = nullptr, side = nullptr;
    cudaEvent_t ev_z = nullptr, ev_m = nullptr;
    double2 *dz = nullptr, *dm = nullptr;
    fmm2d_plan* P = nullptr;
    auto body = [&]() -> int {
        static std::mutex mu;
        static cudaStream_t cache_b[64] = {nullptr}, cache_s[64] = {nullptr};
        if (opt->device < 0 || opt->device >= 64) return FMM2D_EINVAL;
        {
            std::lock_guard<std::mutex> lk(mu);
            if (!cache_b[opt->device]) {
                int lo = 0, hi = 0;
                FMM2D_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
                FMM2D_CUDA_TRY(cudaStreamCreateWithPriority(&cache_b[opt->device], cudaStreamNonBlocking, hi));
                FMM2D_CUDA_TRY(cudaStreamCreateWithFlags(&cache_s[opt->device], cudaStreamNonBlocking));
            }
            bst = cache_b[opt->device];
            side = cache_s[opt->device];
        }
        FMM2D_CUDA_TRY(cudaEventCreateWithFlags(&ev_z, cudaEventDisableTiming));
        FMM2D_CUDA_TRY(cudaEventCreateWithFlags(&ev_m, cudaEventDisableTiming));
        FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&dz, sizeof(double2) * n, bst));
        FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&dm, sizeof(double2) * n, bst));
        // positions first (the build needs them), then the strengths behind them
        FMM2D_CUDA_TRY(cudaMemcpyAsync(dz, z, sizeof(double2) * n, cudaMemcpyHostToDevice, bst));
        FMM2D_CUDA_TRY(cudaEventRecord(ev_z, bst));
        FMM2D_CUDA_TRY(cudaStreamWaitEvent(side, ev_z, 0));
        FMM2D_CUDA_TRY(cudaMemcpyAsync(dm, m, sizeof(double2) * n, cudaMemcpyHostToDevice, side));
        FMM2D_CUDA_TRY(cudaEventRecord(ev_m, side));
        fmm2d_options o = *opt;
        o.flags &= ~FMM2D_HOST_PTRS;
        o.stream = bst;
        FMM2D_TRY(fmm2d_build((const double*)dz, n, &o, &P));   // synchronous
        // from here on the plan lives on the caller's stream, with host-pointer semantics;
        // the strengths already sit in its staging buffer
        P->stream = st;
        cudaFreeAsync(dz, bst);
        dz = nullptr;
        FMM2D_CUDA_TRY(cudaStreamSynchronize(bst));
        P->flags |= FMM2D_HOST_PTRS;
        P->allocs.push_back(dm);
        P->mstage = dm;
        dm = nullptr;
        FMM2D_TRY(dev_alloc(P, (void**)&P->phistage, sizeof(double2) * n));
        FMM2D_TRY(dev_alloc(P, (void**)&P->dphistage, sizeof(double2) * n));
        FMM2D_CUDA_TRY(cudaStreamWaitEvent(st, ev_m, 0));
        const int erc = eval_impl(&P, 1, nullptr, phi, dphi, nullptr);   // m == nullptr: already staged
        // FMM2D_ASYNC_HOST applies to this call's evaluation only: later fmm2d_eval calls on
        // the returned host plan are synchronous (their results are in phi / dphi on return)
        P->flags &= ~FMM2D_ASYNC_HOST;
        return erc;
    };
    int rc = body();
    if (dz) cudaFreeAsync(dz, bst ? bst : st);
    if (dm) cudaFreeAsync(dm, bst ? bst : st);
    if (side) cudaStreamSynchronize(side);               // the strengths' copy (kept streams)
    if (bst) cudaStreamSynchronize(bst);
    if (ev_z) cudaEventDestroy(ev_z);
    if (ev_m) cudaEventDestroy(ev_m);
    if (rc) {
        fmm2d_free(P);
        return rc;
    }
    *out = P;
    return 0;
}

int fmm2d_build_shards(const double* z, int64_t n, const fmm2d_options* opt, int nshards, fmm2d_plan** out)
{
    if (!out || !z || !opt || nshards < 1 || nshards > 64) return FMM2D_EINVAL;
    if (opt->flags & FMM2D_HOST_PTRS) return FMM2D_ENOTSUP;
    for (int i = 0; i < nshards; ++i) out[i] = nullptr;
    int rc = 0;
    for (int i = 0; i < nshards && !rc; ++i) rc = build_stage_tree(z, n, opt, nshards, i, nullptr, &out[i], true);
    if (!rc && nshards > 1) rc = shard_build_rest(out, nshards);
    if (rc) {
        for (int i = 0; i < nshards; ++i) {
            fmm2d_free(out[i]);
            out[i] = nullptr;
        }
    }
    return rc;
}

// One evaluation pass over the plans of this process: one plan (one GPU, or one
// rank of an NCCL-sharded build) or every rank of a loopback build, stage by stage.
static int eval_impl(fmm2d_plan* const* Ps, int np, const double* m, double* phi, double* dphi, cudaEvent_t* ev)
{
    // m == nullptr: host-pointer plan whose strengths are already in its staging buffer
    // (fmm2d_build_eval); the public entry points reject a null m before this
    if (!Ps || np < 1 || (!m && !(np == 1 && Ps[0] && Ps[0]->mstage))) return FMM2D_EINVAL;
    for (int i = 0; i < np; ++i)
        if (!Ps[i]) return FMM2D_EINVAL;
    fmm2d_plan* P0 = Ps[0];
    FMM2D_CUDA_TRY(cudaSetDevice(P0->device));
    const int64_t n = P0->n;
    const bool host = (P0->flags & FMM2D_HOST_PTRS) != 0;
    const bool sharded = P0->nranks > 1;
    const double2* md = (const double2*)m;
    double2* phid = (double2*)phi;
    double2* dphid = (double2*)dphi;
    if (host) {
        if (np != 1) return FMM2D_ENOTSUP;
        if (!P0->mstage) {
            FMM2D_TRY(dev_alloc(P0, (void**)&P0->mstage, sizeof(double2) * n));
            FMM2D_TRY(dev_alloc(P0, (void**)&P0->phistage, sizeof(double2) * n));
            FMM2D_TRY(dev_alloc(P0, (void**)&P0->dphistage, sizeof(double2) * n));
        }
        if (m) FMM2D_CUDA_TRY(cudaMemcpyAsync(P0->mstage, m, sizeof(double2) * n, cudaMemcpyHostToDevice, P0->stream));
        md = P0->mstage;
        phid = phi ? P0->phistage : nullptr;
        dphid = dphi ? P0->dphistage : nullptr;
    }
    const bool gather_out = sharded && np == 1 && (P0->flags & FMM2D_GATHER_OUTPUT) && shard_has_comm(P0);
    if (gather_out) {                                  // own entries written below, the rest summed in
        if (phid) FMM2D_CUDA_TRY(cudaMemsetAsync(phid, 0, sizeof(double2) * n, P0->stream));
        if (dphid) FMM2D_CUDA_TRY(cudaMemsetAsync(dphid, 0, sizeof(double2) * n, P0->stream));
    }
    if (ev) FMM2D_CUDA_TRY(cudaEventRecord(ev[0], P0->stream));
    // the own sources' strengths: gathered by P2M (which reads the same rows) unless the near
    // field runs concurrently with the expansions (overlap mode needs the rows first)
    const bool overlapped = np == 1 && P0->overlap && !ev;
    for (int i = 0; i < np; ++i) {
        Ps[i]->m_fused = overlapped ? nullptr : md;
        if (overlapped) FMM2D_TRY(gather_strengths(Ps[i], md));
        if (sharded) FMM2D_TRY(shard_gather_halo(Ps[i], md));
    }
    if (ev) FMM2D_CUDA_TRY(cudaEventRecord(ev[1], P0->stream));
    // the expansion chain: P2M, M2M (+ halo exchange), M2L, L2L, P2L, M2P
    auto expansions = [&]() -> int {
        for (int i = 0; i < np; ++i) FMM2D_TRY(run_upward(Ps[i]));
        if (sharded) {
            FMM2D_TRY(shard_comm_top(Ps, np));
            for (int i = 0; i < np; ++i) {
                FMM2D_TRY(run_upward_top(Ps[i]));
                FMM2D_TRY(shard_pack_mp(Ps[i]));
            }
            FMM2D_TRY(shard_comm_mp(Ps, np));
            for (int i = 0; i < np; ++i) FMM2D_TRY(shard_unpack_mp(Ps[i]));
        }
        if (ev) FMM2D_CUDA_TRY(cudaEventRecord(ev[2], P0->stream));
        for (int i = 0; i < np; ++i) FMM2D_TRY(run_m2l(Ps[i]));
        if (ev) FMM2D_CUDA_TRY(cudaEventRecord(ev[3], P0->stream));
        for (int i = 0; i < np; ++i) FMM2D_TRY(run_downward(Ps[i]));
        for (int i = 0; i < np; ++i) FMM2D_TRY(run_rr_p2l(Ps[i]));      // r/R exchange: into the locals
        for (int i = 0; i < np; ++i) FMM2D_TRY(run_rr_m2p(Ps[i]));      // r/R exchange: M2P sums
        if (ev) FMM2D_CUDA_TRY(cudaEventRecord(ev[4], P0->stream));     // stage 4 = the near field alone
        return 0;
    };
    if (np == 1 && P0->overlap && !ev) {
        // overlapped (DESIGN 6.4): the expansion chain on the high-priority side stream, the
        // P2P sums on the plan's stream at the same time, then L2P + output (k_near_final)
        cudaStream_t user = P0->stream;
        FMM2D_CUDA_TRY(cudaEventRecord(P0->ev_gather, user));
        FMM2D_CUDA_TRY(cudaStreamWaitEvent(P0->side, P0->ev_gather, 0));
        P0->stream = P0->side;
        // M2L keeps FMM2D_OVERLAP_M2L_WARPS warps per SM (default 2) so that the P2P CTAs
        // can co-reside with it
        {
            static int wps = [] {
                const char* e = getenv("FMM2D_OVERLAP_M2L_WARPS");
                return e ? atoi(e) : 2;
            }();
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P0->device);
            P0->m2l_cap = (int64_t)sms * std::max(1, wps);
        }
        const int rc = expansions();
        P0->m2l_cap = 0;
        P0->stream = user;
        FMM2D_TRY(rc);
        FMM2D_CUDA_TRY(cudaEventRecord(P0->ev_exp, P0->side));
        FMM2D_TRY(run_near(P0, phid, dphid, 1));
        FMM2D_CUDA_TRY(cudaStreamWaitEvent(user, P0->ev_exp, 0));
        FMM2D_TRY(run_near(P0, phid, dphid, 2));
    } else {
        FMM2D_TRY(expansions());
        for (int i = 0; i < np; ++i) FMM2D_TRY(run_near(Ps[i], phid, dphid, 0));
    }
    if (gather_out) FMM2D_TRY(shard_gather_output(P0, phid, dphid));
    if (ev) FMM2D_CUDA_TRY(cudaEventRecord(ev[5], P0->stream));
    if (host) {
        if (phi) FMM2D_CUDA_TRY(cudaMemcpyAsync(phi, phid, sizeof(double2) * n, cudaMemcpyDeviceToHost, P0->stream));
        if (dphi) FMM2D_CUDA_TRY(cudaMemcpyAsync(dphi, dphid, sizeof(double2) * n, cudaMemcpyDeviceToHost, P0->stream));
        if (!(P0->flags & FMM2D_ASYNC_HOST)) FMM2D_CUDA_TRY(cudaStreamSynchronize(P0->stream));
    }
    return 0;
}

int fmm2d_eval(fmm2d_plan* P, const double* m, double* phi, double* dphi)
{
    if (!m) return FMM2D_EINVAL;
    if (P && P->nranks > 1 && !shard_has_comm(P)) return FMM2D_EINVAL;   // loopback: eval_shards
    return eval_impl(&P, 1, m, phi, dphi, nullptr);
}

int fmm2d_eval_shards(fmm2d_plan* const* plans, int nshards, const double* m, double* phi, double* dphi)
{
    if (!plans || nshards < 1 || !m) return FMM2D_EINVAL;
    for (int i = 0; i < nshards; ++i)
        if (!plans[i] || plans[i]->nranks != nshards || plans[i]->rank != i || shard_has_comm(plans[i]))
            return FMM2D_EINVAL;
    return eval_impl(plans, nshards, m, phi, dphi, nullptr);
}

int fmm2d_eval_timed(fmm2d_plan* P, const double* m, double* phi, double* dphi, double* ms_out)
{
    if (!P || !m || !ms_out) return FMM2D_EINVAL;
    if (P->nranks > 1 && !shard_has_comm(P)) return FMM2D_EINVAL;
    FMM2D_CUDA_TRY(cudaSetDevice(P->device));
    cudaEvent_t ev[6];
    for (int i = 0; i < 6; ++i) FMM2D_CUDA_TRY(cudaEventCreate(&ev[i]));
    int rc = eval_impl(&P, 1, m, phi, dphi, ev);
    if (rc == 0) {
        cudaError_t e = cudaEventSynchronize(ev[5]);
        if (e != cudaSuccess) {
            fmm2d_set_last_cuda_error(e, "cudaEventSynchronize", __FILE__, __LINE__);
            rc = FMM2D_ECUDA;
        }
    }
    if (rc == 0) {
        for (int i = 0; i < 5; ++i) {
            float t = 0.f;
            cudaEventElapsedTime(&t, ev[i], ev[i + 1]);
            ms_out[i] = t;
        }
        float t = 0.f;
        cudaEventElapsedTime(&t, ev[0], ev[5]);
        ms_out[5] = t;
        ms_out[6] = ms_out[7] = 0.0;
    }
    for (int i = 0; i < 6; ++i) cudaEventDestroy(ev[i]);
    return rc;
}

int fmm2d_nccl_unique_id(void* out)
{
    if (!out) return FMM2D_EINVAL;
    return nccl_unique_id(out);
}

int fmm2d_partition_info(int64_t n, const fmm2d_options* opt, int nranks, int rank, int64_t* info)
{
    if (!opt || !info || nranks < 1 || rank < 0 || rank >= nranks) return FMM2D_EINVAL;
    const int L = plan_depth(n, opt);
    if (L < 0) return L;
    int k = 0;
    if (nranks > 1) {
        k = partition_level(nranks);
        if (k < 0 || L <= k) return FMM2D_ENOTSUP;
    }
    const int64_t nk = nboxes(k), nl = nboxes(L);
    info[0] = L;
    info[1] = k;
    info[2] = nl / nranks * rank;                       // own leaves [info2, info3)
    info[3] = nl / nranks * (rank + 1);
    info[4] = (nranks == 1) ? 0 : box_start_host(n, k, nk / nranks * rank);    // own positions
    info[5] = (nranks == 1 || rank + 1 == nranks) ? n : box_start_host(n, k, nk / nranks * (rank + 1));
    info[6] = nk / nranks * rank;                       // own level-k subtrees
    info[7] = nk / nranks * (rank + 1);
    return 0;
}

int64_t fmm2d_launch_count(void) { return launch_count(); }

int fmm2d_reserve(int device, size_t bytes)
{
    if (device < 0) return FMM2D_EINVAL;
    FMM2D_CUDA_TRY(cudaSetDevice(device));
    cudaMemPool_t pool = lib_pool(device);           // keeps freed memory (the library's own pool)
    if (!pool) return FMM2D_ECUDA;
    uint64_t have = 0;
    FMM2D_CUDA_TRY(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &have));
    if (have >= bytes) return 0;
    cudaStream_t st = nullptr;
    FMM2D_CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    void* p = nullptr;
    const cudaError_t e = fmm2d::pool_malloc((void**)&p, bytes, st);
    if (e == cudaSuccess) cudaFreeAsync(p, st);
    const cudaError_t e2 = cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        fmm2d_set_last_cuda_error(e, "cudaMallocAsync (reserve)", __FILE__, __LINE__);
        return FMM2D_ENOMEM;
    }
    if (e2 != cudaSuccess) {
        fmm2d_set_last_cuda_error(e2, "cudaStreamSynchronize (reserve)", __FILE__, __LINE__);
        return FMM2D_ECUDA;
    }
    return 0;
}

int fmm2d_pool_trim(int device, size_t keep_bytes)
{
    if (device < 0) return FMM2D_EINVAL;
    FMM2D_CUDA_TRY(cudaSetDevice(device));
    cudaMemPool_t pool = lib_pool(device);
    if (!pool) return FMM2D_ECUDA;
    FMM2D_CUDA_TRY(cudaDeviceSynchronize());        // frees enqueued on any stream have completed
    FMM2D_CUDA_TRY(cudaMemPoolTrimTo(pool, keep_bytes));
    return 0;
}

int fmm2d_pool_usage(int device, int64_t* used, int64_t* high, int reset)
{
    if (device < 0 || !used || !high) return FMM2D_EINVAL;
    FMM2D_CUDA_TRY(cudaSetDevice(device));
    cudaMemPool_t pool = lib_pool(device);
    if (!pool) return FMM2D_ECUDA;
    uint64_t u = 0, h = 0;
    FMM2D_CUDA_TRY(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &u));
    FMM2D_CUDA_TRY(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &h));
    *used = (int64_t)u;
    *high = (int64_t)h;
    if (reset) {
        uint64_t z = 0;
        FMM2D_CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &z));
    }
    return 0;
}

int fmm2d_halo_info(const fmm2d_plan* P, int64_t* info)
{
    if (!P || !info) return FMM2D_EINVAL;
    shard_halo_sizes(P, &info[0], &info[1], &info[2], &info[3]);
    info[4] = P->nranks;
    info[5] = P->rank;
    info[6] = P->kpart;
    info[7] = P->pos0;
    info[8] = P->pos1;
    return 0;
}

int fmm2d_plan_info(const fmm2d_plan* P, int64_t* n, int* nlevels, int* p, int64_t* weak_pairs,
                    int64_t* strong_leaf_pairs)
{
    if (!P) return FMM2D_EINVAL;
    if (n) *n = P->n;
    if (nlevels) *nlevels = P->L;
    if (p) *p = P->p;
    if (weak_pairs) *weak_pairs = P->stats.weak_pairs;
    if (strong_leaf_pairs) *strong_leaf_pairs = P->stats.strong_leaf_pairs;
    return 0;
}

static int copy_out(const void* dsrc, void* dst, size_t bytes, size_t* cap, size_t* off, cudaStream_t st)
{
    if (*off + bytes > *cap) return FMM2D_EINVAL;
    if (bytes) FMM2D_CUDA_TRY(cudaMemcpyAsync((char*)dst + *off, dsrc, bytes, cudaMemcpyDeviceToHost, st));
    *off += bytes;
    return 0;
}

/* STATS layout (double[16]): 0 n, 1 L, 2 p, 3 theta, 4 weak pairs (all levels),
 * 5 strong leaf pairs, 6 min leaf size, 7 max leaf size, 8 t_build_ms, 9 t_tree_ms,
 * 10 t_lists_ms, 11 number of boxes (all levels), 12 kernel launches of this library
 * since it was loaded (all plans), 13 ordered P2P pairs (j != i) of one eval, 14 axes presorted
 * with 64-bit keys (bit 0 x, bit 1 y), 15 device bytes the plan holds. */
int fmm2d_export(const fmm2d_plan* P, int what, int level, void* dst, size_t* bytes)
{
    if (!P || !bytes) return FMM2D_EINVAL;
    if (cudaSetDevice(P->device) != cudaSuccess) return FMM2D_ECUDA;
    const bool leaf_list = (what == FMM2D_EXPORT_NEAR || what == FMM2D_EXPORT_RR_P2L ||
                            what == FMM2D_EXPORT_RR_M2P);
    const bool per_level = (what == FMM2D_EXPORT_OFFSETS || what == FMM2D_EXPORT_DISCS ||
                            what == FMM2D_EXPORT_STRONG || what == FMM2D_EXPORT_WEAK ||
                            what == FMM2D_EXPORT_MPOLE || what == FMM2D_EXPORT_LOCAL || leaf_list ||
                            what == FMM2D_EXPORT_XWEAK);
    if (per_level && (level < 0 || level > P->L)) return FMM2D_EINVAL;
    if (leaf_list && level != P->L) return FMM2D_EINVAL;
    const int64_t nb = per_level ? nboxes(level) : 0;
    // leaf lists: without r/R exchange the conversion lists are empty
    Csr empty_csr;
    const Csr* LC = nullptr;
    if (leaf_list) {
        LC = (what == FMM2D_EXPORT_NEAR) ? &P->near : (what == FMM2D_EXPORT_RR_P2L ? &P->rr_p2l : &P->rr_m2p);
        if (!LC->off) LC = &empty_csr;
    }
    if (what == FMM2D_EXPORT_XWEAK) {
        LC = (level < (int)P->xweak.size()) ? &P->xweak[level] : &empty_csr;
        if (!LC->off) LC = &empty_csr;
    }
    size_t need = 0;
    switch (what) {
        case FMM2D_EXPORT_PERM: need = sizeof(uint32_t) * P->n; break;
        case FMM2D_EXPORT_OFFSETS: need = sizeof(int64_t) * (nb + 1); break;
        case FMM2D_EXPORT_DISCS: need = sizeof(double) * 3 * nb; break;
        case FMM2D_EXPORT_STRONG:
            need = sizeof(int64_t) * (nb + 1) + sizeof(uint32_t) * P->strong[level].total; break;
        case FMM2D_EXPORT_WEAK:
            need = sizeof(int64_t) * (nb + 1) + sizeof(uint32_t) * P->weak[level].total; break;
        case FMM2D_EXPORT_MPOLE:
        case FMM2D_EXPORT_LOCAL: need = sizeof(double2) * nb * (P->p + 1); break;
        case FMM2D_EXPORT_STATS: need = sizeof(double) * 16; break;
        case FMM2D_EXPORT_NEAR:
        case FMM2D_EXPORT_RR_P2L:
        case FMM2D_EXPORT_RR_M2P:
        case FMM2D_EXPORT_XWEAK: need = sizeof(int64_t) * (nb + 1) + sizeof(uint32_t) * LC->total; break;
        default: return FMM2D_EINVAL;
    }
    if (!dst) {
        *bytes = need;
        return 0;
    }
    if (*bytes < need) return FMM2D_EINVAL;
    size_t off = 0, cap = *bytes;
    cudaStream_t st = P->stream;
    switch (what) {
        case FMM2D_EXPORT_PERM:                  // sharded plans: the own positions (the rest 0)
            memset(dst, 0, need);
            FMM2D_CUDA_TRY(cudaMemcpyAsync((uint32_t*)dst + P->pos0, P->perm + P->pos0,
                                           sizeof(uint32_t) * (P->pos1 - P->pos0), cudaMemcpyDeviceToHost, st));
            off = need;
            break;
        case FMM2D_EXPORT_OFFSETS: {
            std::vector<uint32_t> h(nb + 1);
            FMM2D_CUDA_TRY(cudaMemcpyAsync(h.data(), P->boff + P->obase[level], sizeof(uint32_t) * (nb + 1),
                                           cudaMemcpyDeviceToHost, st));
            FMM2D_CUDA_TRY(cudaStreamSynchronize(st));
            int64_t* o = (int64_t*)dst;
            for (int64_t b = 0; b <= nb; ++b) o[b] = h[b];
            off = need;
            break;
        }
        case FMM2D_EXPORT_DISCS:
            FMM2D_TRY(copy_out(P->cx + P->base[level], dst, sizeof(double) * nb, &cap, &off, st));
            FMM2D_TRY(copy_out(P->cy + P->base[level], dst, sizeof(double) * nb, &cap, &off, st));
            FMM2D_TRY(copy_out(P->r + P->base[level], dst, sizeof(double) * nb, &cap, &off, st));
            break;
        case FMM2D_EXPORT_STRONG:
        case FMM2D_EXPORT_WEAK: {
            const Csr& C = (what == FMM2D_EXPORT_STRONG) ? P->strong[level] : P->weak[level];
            FMM2D_TRY(copy_out(C.off, dst, sizeof(int64_t) * (nb + 1), &cap, &off, st));
            FMM2D_TRY(copy_out(C.idx, dst, sizeof(uint32_t) * C.total, &cap, &off, st));
            break;
        }
        case FMM2D_EXPORT_NEAR:
        case FMM2D_EXPORT_RR_P2L:
        case FMM2D_EXPORT_RR_M2P:
        case FMM2D_EXPORT_XWEAK:
            if (LC->off) {
                FMM2D_TRY(copy_out(LC->off, dst, sizeof(int64_t) * (nb + 1), &cap, &off, st));
                FMM2D_TRY(copy_out(LC->idx, dst, sizeof(uint32_t) * LC->total, &cap, &off, st));
            } else {
                memset(dst, 0, sizeof(int64_t) * (nb + 1));
                off = sizeof(int64_t) * (nb + 1);
            }
            break;
        case FMM2D_EXPORT_MPOLE:
        case FMM2D_EXPORT_LOCAL: {              // sharded plans: the stored boxes (the rest 0)
            const double2* E = (what == FMM2D_EXPORT_MPOLE) ? P->mpl[level] : P->lcl[level];
            const int64_t b0 = P->box_lo(level), b1 = P->box_hi(level), P1 = P->p + 1;
            memset(dst, 0, need);
            FMM2D_CUDA_TRY(cudaMemcpyAsync((double2*)dst + b0 * P1, E + b0 * P1, sizeof(double2) * (b1 - b0) * P1,
                                           cudaMemcpyDeviceToHost, st));
            off = need;
            break;
        }
        case FMM2D_EXPORT_STATS: {
            double* s = (double*)dst;
            for (int i = 0; i < 16; ++i) s[i] = 0.0;
            s[0] = (double)P->n; s[1] = P->L; s[2] = P->p; s[3] = P->theta;
            s[4] = (double)P->stats.weak_pairs; s[5] = (double)P->stats.strong_leaf_pairs;
            s[6] = P->stats.min_leaf; s[7] = P->stats.max_leaf;
            s[8] = P->stats.t_build_ms; s[9] = P->stats.t_tree_ms; s[10] = P->stats.t_lists_ms;
            s[11] = (double)P->nbox_total;
            s[12] = (double)launch_count();
            s[13] = (double)P->stats.p2p_pairs;
            s[14] = (double)P->stats.tree_key64;
            s[15] = (double)P->stats.dev_bytes;
            off = need;
            break;
        }
    }
    FMM2D_CUDA_TRY(cudaStreamSynchronize(st));
    *bytes = off;
    return 0;
}

}  // extern "C"
