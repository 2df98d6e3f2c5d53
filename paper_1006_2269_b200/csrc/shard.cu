// shard.cu -- the evaluation pass partitioned across GPUs (
// SURVEY 8(e)).
//
// The balanced tree makes the partition natural: the 4^k boxes of level
// k hold equal point counts (+-1), so rank r of P owns the level-k subtrees
// [r 4^k / P, (r+1) 4^k / P), k the smallest level with P | 4^k.  At every level
// l >= k its boxes are the contiguous range [r 4^l / P, (r+1) 4^l / P) and its points
// the contiguous leaf-order positions [pos0, pos1).
//
//   build  every rank holds the full input z; levels 0..k are built on every rank
//          (replicated, deterministic), levels > k for the own subtrees only
//          (tree.cu).  Exchanges: max of the replicated top radii, all-gather of the
//          discs of levels > k (the theta-criterion needs the neighbours' discs),
//          lists of the own boxes (lists.cu), then the halo: remote leaves of the own
//          strong lists (their positions and input indices are imported once) and
//          remote boxes of the own weak lists (their multipoles are imported at every
//          evaluation).  Requests are per-owner sorted id lists; the owner keeps
//          them as export lists.
//   eval   every rank has the full strengths m (input order), so the halo sources
//          need no transfer: m is gathered locally through the imported indices.
//          P2M + M2M of the own subtrees, all-gather of the level-k multipoles, the
//          replicated M2M above k, export/import of the halo multipoles (grouped
//          send/recv), then M2L, L2L and L2P + P2P of the own boxes.  Every rank
//          writes the Phi, Phi' entries of its own sources (input positions).
// Results are independent of the partition: each own box sees the same lists,
// multipoles and locals as in a one-GPU run, in the same order, so the union of
// the ranks' outputs equals the one-GPU result bit for bit (tests).
//
// Transport: NCCL over NVLink/NVSwitch (one process per GPU; the library loads
// libnccl.so.2 on first use), or "loopback" -- all ranks as plans in one process on
// one device, the same stages run rank after rank and every transfer a device copy
// (tests of the partition on one GPU; no kernel ever waits on another rank's).
#include <dlfcn.h>
#include <nccl.h>

#include <cub/cub.cuh>
#include <map>
#include <mutex>
#include <string>

#include "fmm2d_internal.cuh"

namespace fmm2d {

// ------------------------------------------------------------------ NCCL (dlopen)
namespace {
struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi* nccl_api()
{
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        // FMM2D_NCCL_LIB: another library with NCCL's entry points (tests only: the
        // one-GPU multi-process shim tests/ncclshim); the product loads NCCL itself
        const char* alt = getenv("FMM2D_NCCL_LIB");
        void* h = (alt && *alt) ? dlopen(alt, RTLD_NOW | RTLD_GLOBAL) : dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h && !(alt && *alt)) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
#define FMM2D_SYM(f, name) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, name))
        FMM2D_SYM(GetUniqueId, "ncclGetUniqueId");
        FMM2D_SYM(CommInitRank, "ncclCommInitRank");
        FMM2D_SYM(CommDestroy, "ncclCommDestroy");
        FMM2D_SYM(AllReduce, "ncclAllReduce");
        FMM2D_SYM(AllGather, "ncclAllGather");
        FMM2D_SYM(Send, "ncclSend");
        FMM2D_SYM(Recv, "ncclRecv");
        FMM2D_SYM(GroupStart, "ncclGroupStart");
        FMM2D_SYM(GroupEnd, "ncclGroupEnd");
        FMM2D_SYM(GetErrorString, "ncclGetErrorString");
#undef FMM2D_SYM
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.AllGather &&
                 api.Send && api.Recv && api.GroupStart && api.GroupEnd && api.GetErrorString;
    });
    return api.ok ? &api : nullptr;
}
}  // namespace

#define FMM2D_NCCL_TRY(expr)                                                                \
    do {                                                                                    \
        ncclResult_t _r = (expr);                                                           \
        if (_r != ncclSuccess) {                                                            \
            fmm2d_set_last_error_text(nccl_api()->GetErrorString(_r), #expr, __FILE__, __LINE__); \
            return FMM2D_ENCCL;                                                             \
        }                                                                                   \
    } while (0)

// ------------------------------------------------------------------ partition
// Offsets are a pure function of n (DESIGN R5): walk the child digits from the root.
int64_t box_start_host(int64_t n, int l, int64_t b)
{
    int64_t off = 0, s = n;
    for (int j = l - 1; j >= 0; --j) {
        const int q = (int)((b >> (2 * j)) & 3);
        const int64_t h0 = s - s / 2, h1 = s / 2;
        const int64_t c[4] = {h0 - h0 / 2, h0 / 2, h1 - h1 / 2, h1 / 2};
        for (int i = 0; i < q; ++i) off += c[i];
        s = c[q];
    }
    return off;
}

// smallest k with P | 4^k (P must be a power of two), or -1
int partition_level(int nranks)
{
    if (nranks < 1) return -1;
    for (int k = 0; k <= FMM2D_MAXL; ++k)
        if ((((int64_t)1 << (2 * k)) % nranks) == 0) return k;
    return -1;
}

// exchange of one kind of halo data; ids are global box ids (mpoles) or leaf ids (rows)
struct XSet {
    int64_t es = 0;                                    // bytes per unit
    std::vector<int64_t> imp_cnt, imp_off, exp_cnt, exp_off;   // per peer, in units
    int64_t imp_tot = 0, exp_tot = 0;
    uint32_t* imp_ids = nullptr;                       // device, grouped by owner, ascending
    uint32_t* exp_ids = nullptr;                       // device, grouped by requester
    char* send = nullptr;                              // device, exp_tot * es
    char* recv = nullptr;                              // device, imp_tot * es
};

struct Shard {
    void* comm = nullptr;          // ncclComm_t, or nullptr for loopback
    XSet leaf;                     // unit: one leaf slot of `slot` rows {x, y, idx}
    XSet mp;                       // unit: one multipole, (p+1) complex
    int slot = 0;
    int64_t* d_counts = nullptr;   // device scratch for the count exchange (NCCL)
};

struct Row {
    double x, y;
    uint32_t idx, pad;
};

namespace {

inline unsigned grid_for(int64_t n, int bs) { return (unsigned)((n + bs - 1) / bs); }

// flag the remote entries of the own boxes' lists: need[gbase + s] = 1 + owner(s)
__global__ void k_flag_remote(int64_t b0, int64_t b1, const int64_t* __restrict__ off,
                              const uint32_t* __restrict__ idx, int64_t gbase, int64_t per_rank, int rank,
                              uint8_t* __restrict__ need)
{
    const int64_t b = b0 + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x & 31;
    if (b >= b1) return;
    for (int64_t q = off[b] + lane; q < off[b + 1]; q += 32) {
        const uint32_t s = idx[q];
        const int owner = (int)(s / per_rank);
        if (owner != rank) need[gbase + s] = (uint8_t)(owner + 1);
    }
}

struct OwnerIs {
    const uint8_t* need;
    uint8_t v;
    __device__ __forceinline__ bool operator()(const uint32_t& i) const { return need[i] == v; }
};

// owner: rows of the requested leaves, one slot of `slot` rows per leaf
__global__ void k_pack_rows(const uint32_t* __restrict__ ids, int64_t cnt, int slot, const uint32_t* __restrict__ off,
                            const double4* __restrict__ src, const uint32_t* __restrict__ perm, Row* __restrict__ out)
{
    const int64_t e = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (e >= cnt) return;
    const uint32_t s = ids[e], s0 = off[s], sz = off[s + 1] - s0;
    for (uint32_t j = lane; j < sz; j += 32) {
        const double4 v = src[s0 + j];
        Row r;
        r.x = v.x;
        r.y = v.y;
        r.idx = perm[s0 + j];
        r.pad = 0;
        out[e * slot + j] = r;
    }
}

// the imported rows of halo leaf e (slot e of `slot` rows) into the halo row store; the
// leaf's map entry lmap[leaf] = its first row there
__global__ void k_unpack_rows(const uint32_t* __restrict__ ids, int64_t cnt, int slot, const uint32_t* __restrict__ off,
                              const Row* __restrict__ in, double4* __restrict__ hsrc, uint32_t* __restrict__ hperm,
                              uint32_t* __restrict__ lmap)
{
    const int64_t e = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (e >= cnt) return;
    const uint32_t s = ids[e], sz = off[s + 1] - off[s];
    if (lane == 0) lmap[s] = (uint32_t)(e * slot);
    for (uint32_t j = lane; j < sz; j += 32) {
        const Row r = in[e * slot + j];
        hsrc[e * slot + j] = make_double4(r.x, r.y, 0.0, 0.0);
        hperm[e * slot + j] = r.idx;
    }
}

// strengths of the halo leaves, gathered locally through the imported input indices
__global__ void k_gather_halo(const uint32_t* __restrict__ ids, int64_t cnt, int slot, const uint32_t* __restrict__ off,
                              const uint32_t* __restrict__ hperm, const double2* __restrict__ m,
                              double4* __restrict__ hsrc)
{
    const int64_t e = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (e >= cnt) return;
    const uint32_t s = ids[e], sz = off[s + 1] - off[s];
    for (uint32_t j = lane; j < sz; j += 32) {
        const double2 v = m[hperm[e * slot + j]];
        double4 r = hsrc[e * slot + j];
        r.z = v.x;
        r.w = v.y;
        hsrc[e * slot + j] = r;
    }
}

// the stored expansions of every level (level l's box b at mp[l] + b P1) by global box id
struct LevelPtrs {
    const double2* mp[FMM2D_MAXL + 1];
    int64_t base[FMM2D_MAXL + 2];
    int L;
};

// exported multipoles (own boxes, P1 complex each) by global box id into the send buffer
__global__ void k_pack_mp(const uint32_t* __restrict__ ids, int64_t cnt, int P1, LevelPtrs M,
                          double2* __restrict__ out)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= cnt * P1) return;
    const int64_t e = t / P1;
    const int k = (int)(t - e * P1);
    const int64_t g = ids[e];
    int l = 0;
    while (l < M.L && g >= M.base[l + 1]) ++l;
    out[t] = M.mp[l][(g - M.base[l]) * P1 + k];
}

// import slot of every imported box (the receive buffer is the halo multipoles' store)
__global__ void k_halo_map(const uint32_t* __restrict__ ids, int64_t cnt, uint32_t* __restrict__ hmap)
{
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < cnt) hmap[ids[e]] = (uint32_t)e;
}

__global__ void k_max_into(double* __restrict__ dst, const double* __restrict__ src, int64_t n)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = fmax(dst[i], src[i]);
}

}  // namespace

// ------------------------------------------------------------------ transport
// All collectives take the plans of the calling process: one plan (NCCL) or all
// ranks' plans (loopback).  Buffers are described per plan by accessors.
static bool is_nccl(fmm2d_plan* const* Ps) { return Ps[0]->shard && Ps[0]->shard->comm; }

// in-place all-gather: rank r's part is bytes [r * part, (r+1) * part) of buf(plan)
template <class F>
static int allgather_inplace(fmm2d_plan* const* Ps, int np, size_t part, F buf)
{
    if (part == 0) return 0;
    if (is_nccl(Ps)) {
        fmm2d_plan* P = Ps[0];
        char* b = (char*)buf(P);
        FMM2D_NCCL_TRY(nccl_api()->AllGather(b + part * P->rank, b, part, ncclChar, (ncclComm_t)P->shard->comm,
                                             P->stream));
        return 0;
    }
    for (int r = 0; r < np; ++r)
        for (int q = 0; q < np; ++q)
            if (q != r)
                FMM2D_CUDA_TRY(cudaMemcpyAsync((char*)buf(Ps[q]) + part * r, (char*)buf(Ps[r]) + part * r, part,
                                               cudaMemcpyDeviceToDevice, Ps[r]->stream));
    return 0;
}

// in-place max all-reduce of n doubles
template <class F>
static int allreduce_max(fmm2d_plan* const* Ps, int np, int64_t n, F buf)
{
    if (n == 0) return 0;
    if (is_nccl(Ps)) {
        fmm2d_plan* P = Ps[0];
        FMM2D_NCCL_TRY(nccl_api()->AllReduce(buf(P), buf(P), (size_t)n, ncclDouble, ncclMax,
                                             (ncclComm_t)P->shard->comm, P->stream));
        return 0;
    }
    cudaStream_t st = Ps[0]->stream;
    for (int q = 1; q < np; ++q) {
        k_max_into<<<grid_for(n, 256), 256, 0, st>>>(buf(Ps[0]), buf(Ps[q]), n);
        note_launch();
    }
    for (int q = 1; q < np; ++q)
        FMM2D_CUDA_TRY(cudaMemcpyAsync(buf(Ps[q]), buf(Ps[0]), sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    return 0;
}

// point-to-point exchange of an XSet.  forward: requester -> owner (id lists,
// imp_ids -> exp_ids); otherwise owner -> requester (payload, send -> recv).
static int exchange(fmm2d_plan* const* Ps, int np, XSet Shard::*which, bool ids_forward)
{
    if (is_nccl(Ps)) {
        fmm2d_plan* P = Ps[0];
        const XSet& X = P->shard->*which;
        ncclComm_t c = (ncclComm_t)P->shard->comm;
        NcclApi* A = nccl_api();
        FMM2D_NCCL_TRY(A->GroupStart());
        for (int q = 0; q < P->nranks; ++q) {
            if (q == P->rank) continue;
            if (ids_forward) {
                if (X.imp_cnt[q]) FMM2D_NCCL_TRY(A->Send(X.imp_ids + X.imp_off[q], X.imp_cnt[q], ncclUint32, q, c, P->stream));
                if (X.exp_cnt[q]) FMM2D_NCCL_TRY(A->Recv(X.exp_ids + X.exp_off[q], X.exp_cnt[q], ncclUint32, q, c, P->stream));
            } else {
                if (X.exp_cnt[q])
                    FMM2D_NCCL_TRY(A->Send(X.send + X.exp_off[q] * X.es, X.exp_cnt[q] * X.es, ncclChar, q, c, P->stream));
                if (X.imp_cnt[q])
                    FMM2D_NCCL_TRY(A->Recv(X.recv + X.imp_off[q] * X.es, X.imp_cnt[q] * X.es, ncclChar, q, c, P->stream));
            }
        }
        FMM2D_NCCL_TRY(A->GroupEnd());
        return 0;
    }
    for (int r = 0; r < np; ++r) {
        const XSet& R = Ps[r]->shard->*which;
        for (int q = 0; q < np; ++q) {
            if (q == r) continue;
            const XSet& Q = Ps[q]->shard->*which;
            if (ids_forward) {            // r requests from q: r.imp(q) -> q.exp(r)
                if (R.imp_cnt[q])
                    FMM2D_CUDA_TRY(cudaMemcpyAsync(Q.exp_ids + Q.exp_off[r], R.imp_ids + R.imp_off[q],
                                                   sizeof(uint32_t) * R.imp_cnt[q], cudaMemcpyDeviceToDevice,
                                                   Ps[r]->stream));
            } else {                      // r serves q: r.send(q) -> q.recv(r)
                if (R.exp_cnt[q])
                    FMM2D_CUDA_TRY(cudaMemcpyAsync(Q.recv + Q.imp_off[r] * Q.es, R.send + R.exp_off[q] * R.es,
                                                   R.exp_cnt[q] * R.es, cudaMemcpyDeviceToDevice, Ps[r]->stream));
            }
        }
    }
    return 0;
}

// ------------------------------------------------------------------ build stages
// Stage B1 (after build_tree): discs of every level on every rank.
static int comm_discs(fmm2d_plan* const* Ps, int np)
{
    fmm2d_plan* P0 = Ps[0];
    const int k = P0->kpart, L = P0->L;
    // replicated levels 0..k: max of the squared radii over the ranks' points
    FMM2D_TRY(allreduce_max(Ps, np, P0->base[k + 1], [](fmm2d_plan* P) { return P->r; }));
    // own levels: all-gather centres and (squared) radii
    for (int l = k + 1; l <= L; ++l) {
        const size_t part = sizeof(double) * (size_t)(nboxes(l) / P0->nranks);
        const int64_t b = P0->base[l];
        FMM2D_TRY(allgather_inplace(Ps, np, part, [b](fmm2d_plan* P) { return (void*)(P->cx + b); }));
        FMM2D_TRY(allgather_inplace(Ps, np, part, [b](fmm2d_plan* P) { return (void*)(P->cy + b); }));
        FMM2D_TRY(allgather_inplace(Ps, np, part, [b](fmm2d_plan* P) { return (void*)(P->r + b); }));
    }
    return 0;
}

// compact the ids flagged 1 + q into X.imp_ids, grouped by owner q (ascending inside)
static int compact_requests(fmm2d_plan* P, const uint8_t* need, int64_t nitems, XSet& X)
{
    cudaStream_t st = P->stream;
    const int R = P->nranks;
    X.imp_cnt.assign(R, 0);
    X.imp_off.assign(R, 0);
    uint32_t* tmp = nullptr;
    int64_t* d_num = nullptr;
    void* scratch = nullptr;
    size_t sb = 0;
    cub::CountingInputIterator<uint32_t> it(0);
    OwnerIs pred{need, 1};
    cub::DeviceSelect::If(nullptr, sb, it, (uint32_t*)nullptr, (int64_t*)nullptr, (int64_t)nitems, pred, st);
    FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&tmp, sizeof(uint32_t) * std::max<int64_t>(nitems, 1), st));
    FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&d_num, sizeof(int64_t) * R, st));
    FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&scratch, std::max<size_t>(sb, 16), st));
    int64_t tot = 0;
    std::vector<int64_t> h(R, 0);
    auto body = [&]() -> int {
        for (int q = 0; q < R; ++q) {
            if (q == P->rank) continue;
            size_t b = sb;
            OwnerIs pq{need, (uint8_t)(q + 1)};
            FMM2D_CUDA_TRY(cub::DeviceSelect::If(scratch, b, it, tmp + tot, d_num + q, (int64_t)nitems, pq, st));
            FMM2D_CUDA_TRY(cudaMemcpyAsync(&h[q], d_num + q, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
            FMM2D_CUDA_TRY(cudaStreamSynchronize(st));
            X.imp_off[q] = tot;
            X.imp_cnt[q] = h[q];
            tot += h[q];
        }
        X.imp_tot = tot;
        FMM2D_TRY(dev_alloc(P, (void**)&X.imp_ids, sizeof(uint32_t) * std::max<int64_t>(tot, 1)));
        if (tot)
            FMM2D_CUDA_TRY(cudaMemcpyAsync(X.imp_ids, tmp, sizeof(uint32_t) * tot, cudaMemcpyDeviceToDevice, st));
        return 0;
    };
    const int rc = body();
    cudaFreeAsync(tmp, st);
    cudaFreeAsync(d_num, st);
    cudaFreeAsync(scratch, st);
    return rc;
}

// Stage B2 (after the lists): the halo requests of this rank.
static int halo_requests(fmm2d_plan* P)
{
    cudaStream_t st = P->stream;
    const int L = P->L, k = P->kpart;
    Shard* S = P->shard;
    const int64_t nl = nboxes(L);
    uint8_t* need = nullptr;
    FMM2D_CUDA_TRY(fmm2d::pool_malloc((void**)&need, std::max<int64_t>(P->nbox_total, nl), st));
    auto body = [&]() -> int {
        // leaves of the own strong lists (level L)
        FMM2D_CUDA_TRY(cudaMemsetAsync(need, 0, nl, st));
        {
            const int64_t b0 = P->box_lo(L), b1 = P->box_hi(L);
            k_flag_remote<<<grid_for((b1 - b0) * 32, 256), 256, 0, st>>>(b0, b1, P->strong[L].off, P->strong[L].idx, 0,
                                                                        nl / P->nranks, P->rank, need);
            note_launch();
            FMM2D_CUDA_TRY(cudaGetLastError());
        }
        FMM2D_TRY(compact_requests(P, need, nl, S->leaf));
        // boxes of the own weak lists, levels k+1..L (global box ids)
        FMM2D_CUDA_TRY(cudaMemsetAsync(need, 0, P->nbox_total, st));
        for (int l = k + 1; l <= L; ++l) {
            const int64_t b0 = P->box_lo(l), b1 = P->box_hi(l);
            k_flag_remote<<<grid_for((b1 - b0) * 32, 256), 256, 0, st>>>(b0, b1, P->weak[l].off, P->weak[l].idx,
                                                                        P->base[l], nboxes(l) / P->nranks, P->rank,
                                                                        need);
            note_launch();
            // parent merge: cross-level sources at level l-1 (remote only below the
            // replicated levels; level k's multipoles are all-gathered)
            if (P->xweak[l].off && l - 1 > k) {
                k_flag_remote<<<grid_for((b1 - b0) * 32, 256), 256, 0, st>>>(b0, b1, P->xweak[l].off,
                                                                            P->xweak[l].idx, P->base[l - 1],
                                                                            nboxes(l - 1) / P->nranks, P->rank, need);
                note_launch();
            }
            FMM2D_CUDA_TRY(cudaGetLastError());
        }
        FMM2D_TRY(compact_requests(P, need, P->nbox_total, S->mp));
        return 0;
    };
    const int rc = body();
    cudaFreeAsync(need, st);
    return rc;
}

// Stage B3: counts -> export lists and buffers.
static int comm_counts(fmm2d_plan* const* Ps, int np)
{
    const int R = Ps[0]->nranks;
    std::vector<int64_t> M((size_t)R * 2 * R, 0);      // M[r][2q + c]: rank r imports from q
    if (is_nccl(Ps)) {
        fmm2d_plan* P = Ps[0];
        Shard* S = P->shard;
        std::vector<int64_t> mine(2 * R);
        for (int q = 0; q < R; ++q) {
            mine[2 * q] = S->leaf.imp_cnt[q];
            mine[2 * q + 1] = S->mp.imp_cnt[q];
        }
        FMM2D_CUDA_TRY(cudaMemcpyAsync(S->d_counts + (size_t)P->rank * 2 * R, mine.data(), sizeof(int64_t) * 2 * R,
                                       cudaMemcpyHostToDevice, P->stream));
        FMM2D_NCCL_TRY(nccl_api()->AllGather(S->d_counts + (size_t)P->rank * 2 * R, S->d_counts, 2 * R, ncclInt64,
                                             (ncclComm_t)S->comm, P->stream));
        FMM2D_CUDA_TRY(cudaMemcpyAsync(M.data(), S->d_counts, sizeof(int64_t) * M.size(), cudaMemcpyDeviceToHost,
                                       P->stream));
        FMM2D_CUDA_TRY(cudaStreamSynchronize(P->stream));
    } else {
        for (int r = 0; r < np; ++r)
            for (int q = 0; q < R; ++q) {
                M[(size_t)r * 2 * R + 2 * q] = Ps[r]->shard->leaf.imp_cnt[q];
                M[(size_t)r * 2 * R + 2 * q + 1] = Ps[r]->shard->mp.imp_cnt[q];
            }
    }
    for (int i = 0; i < np; ++i) {
        fmm2d_plan* P = Ps[i];
        Shard* S = P->shard;
        XSet* xs[2] = {&S->leaf, &S->mp};
        for (int c = 0; c < 2; ++c) {
            XSet& X = *xs[c];
            X.exp_cnt.assign(R, 0);
            X.exp_off.assign(R, 0);
            int64_t tot = 0;
            for (int q = 0; q < R; ++q) {
                X.exp_off[q] = tot;
                X.exp_cnt[q] = (q == P->rank) ? 0 : M[(size_t)q * 2 * R + 2 * P->rank + c];
                tot += X.exp_cnt[q];
            }
            X.exp_tot = tot;
            FMM2D_TRY(dev_alloc(P, (void**)&X.exp_ids, sizeof(uint32_t) * std::max<int64_t>(tot, 1)));
            FMM2D_TRY(dev_alloc(P, (void**)&X.send, (size_t)std::max<int64_t>(tot * X.es, 16)));
            FMM2D_TRY(dev_alloc(P, (void**)&X.recv, (size_t)std::max<int64_t>(X.imp_tot * X.es, 16)));
        }
    }
    return 0;
}

static int pack_rows(fmm2d_plan* P)
{
    const XSet& X = P->shard->leaf;
    if (X.exp_tot == 0) return 0;
    const uint32_t* off = P->boff + P->obase[P->L];
    k_pack_rows<<<grid_for(X.exp_tot * 32, 256), 256, 0, P->stream>>>(X.exp_ids, X.exp_tot, P->shard->slot, off,
                                                                     P->src, P->perm, (Row*)X.send);
    note_launch();
    FMM2D_CUDA_TRY(cudaGetLastError());
    return 0;
}

// the halo stores (rows + input indices of the imported leaves, the imported multipoles'
// slots) -- allocated for the import counts only, never for all n points / all boxes
static int unpack_rows(fmm2d_plan* P)
{
    const XSet& X = P->shard->leaf;
    const int slot = P->shard->slot;
    const int64_t nl = nboxes(P->L);
    FMM2D_TRY(dev_alloc(P, (void**)&P->lmap, sizeof(uint32_t) * nl));
    FMM2D_CUDA_TRY(cudaMemsetAsync(P->lmap, 0xFF, sizeof(uint32_t) * nl, P->stream));
    FMM2D_TRY(dev_alloc(P, (void**)&P->hsrc, sizeof(double4) * std::max<int64_t>(X.imp_tot * slot, 1)));
    FMM2D_TRY(dev_alloc(P, (void**)&P->hperm, sizeof(uint32_t) * std::max<int64_t>(X.imp_tot * slot, 1)));
    if (X.imp_tot > 0) {
        const uint32_t* off = P->boff + P->obase[P->L];
        k_unpack_rows<<<grid_for(X.imp_tot * 32, 256), 256, 0, P->stream>>>(X.imp_ids, X.imp_tot, slot, off,
                                                                           (const Row*)X.recv, P->hsrc, P->hperm,
                                                                           P->lmap);
        note_launch();
        FMM2D_CUDA_TRY(cudaGetLastError());
    }
    const XSet& Y = P->shard->mp;
    FMM2D_TRY(dev_alloc(P, (void**)&P->hmap, sizeof(uint32_t) * std::max<int64_t>(P->nbox_total, 1)));
    if (Y.imp_tot > 0) {
        k_halo_map<<<grid_for(Y.imp_tot, 256), 256, 0, P->stream>>>(Y.imp_ids, Y.imp_tot, P->hmap);
        note_launch();
        FMM2D_CUDA_TRY(cudaGetLastError());
    }
    P->mhalo = (const double2*)Y.recv;
    return 0;
}

// ------------------------------------------------------------------ plan set-up
int shard_setup(fmm2d_plan* P, int nranks, int rank, const void* nccl_id)
{
    P->nranks = nranks;
    P->rank = rank;
    if (nranks == 1) return 0;
    const int k = partition_level(nranks);
    if (k < 0) return FMM2D_ENOTSUP;                   // P must be a power of two
    if (P->L <= k) return FMM2D_ENOTSUP;               // too small to partition
    P->kpart = k;
    const int64_t nk = nboxes(k);
    P->pos0 = (uint32_t)box_start_host(P->n, k, nk / nranks * rank);
    P->pos1 = (rank + 1 == nranks) ? (uint32_t)P->n : (uint32_t)box_start_host(P->n, k, nk / nranks * (rank + 1));
    Shard* S = new (std::nothrow) Shard();
    if (!S) return FMM2D_ENOMEM;
    P->shard = S;
    S->slot = (int)((P->n + nboxes(P->L) - 1) / nboxes(P->L));     // largest leaf (DESIGN R5)
    S->leaf.es = (int64_t)sizeof(Row) * S->slot;
    S->mp.es = (int64_t)sizeof(double2) * (P->p + 1);
    if (nccl_id) {
        NcclApi* A = nccl_api();
        if (!A) {
            fmm2d_set_last_error_text("libnccl.so.2 could not be loaded", "dlopen", __FILE__, __LINE__);
            return FMM2D_ENCCL;
        }
        // one communicator per unique id, kept for the life of the process: every plan
        // built with the same id (e.g. one per step of a benchmark) reuses it
        static std::mutex mu;
        static std::map<std::string, ncclComm_t> cache;
        std::lock_guard<std::mutex> lock(mu);
        const std::string key((const char*)nccl_id, sizeof(ncclUniqueId));
        auto it = cache.find(key);
        if (it == cache.end()) {
            ncclUniqueId id;
            memcpy(&id, nccl_id, sizeof(id));
            ncclComm_t c = nullptr;
            FMM2D_NCCL_TRY(A->CommInitRank(&c, nranks, id, rank));
            it = cache.emplace(key, c).first;
        }
        S->comm = it->second;
        FMM2D_TRY(dev_alloc(P, (void**)&S->d_counts, sizeof(int64_t) * 2 * nranks * nranks));
    }
    return 0;
}

void shard_free(fmm2d_plan* P)
{
    if (!P->shard) return;
    delete P->shard;                   // the communicator stays cached (shard_setup)
    P->shard = nullptr;
}

int nccl_unique_id(void* out)
{
    NcclApi* A = nccl_api();
    if (!A) {
        fmm2d_set_last_error_text("libnccl.so.2 could not be loaded", "dlopen", __FILE__, __LINE__);
        return FMM2D_ENCCL;
    }
    ncclUniqueId id;
    FMM2D_NCCL_TRY(A->GetUniqueId(&id));
    memcpy(out, &id, sizeof(id));
    return 0;
}

// ------------------------------------------------------------------ staged drivers
// build_stage_tree (api.cu) has run on every plan; the remaining build stages.
int shard_build_rest(fmm2d_plan* const* Ps, int np)
{
    FMM2D_TRY(comm_discs(Ps, np));
    for (int i = 0; i < np; ++i) {
        FMM2D_TRY(finish_radii(Ps[i]));
        FMM2D_TRY(build_lists(Ps[i]));
        FMM2D_TRY(halo_requests(Ps[i]));
    }
    FMM2D_TRY(comm_counts(Ps, np));
    FMM2D_TRY(exchange(Ps, np, &Shard::leaf, true));
    FMM2D_TRY(exchange(Ps, np, &Shard::mp, true));
    for (int i = 0; i < np; ++i) FMM2D_TRY(pack_rows(Ps[i]));
    FMM2D_TRY(exchange(Ps, np, &Shard::leaf, false));
    for (int i = 0; i < np; ++i) {
        FMM2D_TRY(unpack_rows(Ps[i]));
        FMM2D_CUDA_TRY(cudaStreamSynchronize(Ps[i]->stream));
    }
    return 0;
}

int shard_gather_halo(fmm2d_plan* P, const double2* m)
{
    const XSet& X = P->shard->leaf;
    if (X.imp_tot == 0) return 0;
    const uint32_t* off = P->boff + P->obase[P->L];
    k_gather_halo<<<grid_for(X.imp_tot * 32, 256), 256, 0, P->stream>>>(X.imp_ids, X.imp_tot, P->shard->slot, off,
                                                                       P->hperm, m, P->hsrc);
    note_launch();
    FMM2D_CUDA_TRY(cudaGetLastError());
    return 0;
}

// eval: level-k multipoles to every rank
int shard_comm_top(fmm2d_plan* const* Ps, int np)
{
    fmm2d_plan* P0 = Ps[0];
    const int k = P0->kpart;
    const size_t part = sizeof(double2) * (P0->p + 1) * (size_t)(nboxes(k) / P0->nranks);
    return allgather_inplace(Ps, np, part, [k](fmm2d_plan* P) { return (void*)P->mpl[k]; });   // level k: all boxes stored
}

int shard_pack_mp(fmm2d_plan* P)
{
    const XSet& X = P->shard->mp;
    if (X.exp_tot == 0) return 0;
    const int P1 = P->p + 1;
    LevelPtrs M;
    M.L = P->L;
    for (int l = 0; l <= P->L; ++l) M.mp[l] = P->mpl[l];
    for (int l = 0; l <= P->L + 1; ++l) M.base[l] = P->base[l];
    k_pack_mp<<<grid_for(X.exp_tot * P1, 256), 256, 0, P->stream>>>(X.exp_ids, X.exp_tot, P1, M, (double2*)X.send);
    note_launch();
    FMM2D_CUDA_TRY(cudaGetLastError());
    return 0;
}

int shard_comm_mp(fmm2d_plan* const* Ps, int np) { return exchange(Ps, np, &Shard::mp, false); }

// the imported multipoles stay in the receive buffer, which M2L reads through hmap
int shard_unpack_mp(fmm2d_plan* P)
{
    (void)P;
    return 0;
}

bool shard_has_comm(const fmm2d_plan* P) { return P->shard && P->shard->comm; }

// Collectives of the partitioned build's top-level selection (tree.cu) on the plan's stream.
int shard_allreduce_sum_u32(fmm2d_plan* P, unsigned int* buf, size_t count)
{
    if (!shard_has_comm(P)) return 0;
    FMM2D_NCCL_TRY(nccl_api()->AllReduce(buf, buf, count, ncclUint32, ncclSum, (ncclComm_t)P->shard->comm,
                                         P->stream));
    return 0;
}

// block r (bytes_per_rank bytes at base + r bytes_per_rank) of every rank to every rank;
// the caller's own block is already in place
int shard_allgather_inplace(fmm2d_plan* P, void* base, size_t bytes_per_rank)
{
    if (!shard_has_comm(P)) return 0;
    char* b = static_cast<char*>(base);
    FMM2D_NCCL_TRY(nccl_api()->AllGather(b + bytes_per_rank * P->rank, b, bytes_per_rank, ncclChar,
                                         (ncclComm_t)P->shard->comm, P->stream));
    return 0;
}

// FMM2D_GATHER_OUTPUT: every rank wrote its own sources' entries into zeroed outputs;
// a sum all-reduce completes them on every rank (x + 0 = x exactly).  Loopback shards
// already share one output array: nothing to do.
int shard_gather_output(fmm2d_plan* P, double2* phi, double2* dphi)
{
    if (!shard_has_comm(P)) return 0;
    NcclApi* A = nccl_api();
    ncclComm_t c = (ncclComm_t)P->shard->comm;
    FMM2D_NCCL_TRY(A->GroupStart());
    if (phi) FMM2D_NCCL_TRY(A->AllReduce(phi, phi, 2 * (size_t)P->n, ncclDouble, ncclSum, c, P->stream));
    if (dphi) FMM2D_NCCL_TRY(A->AllReduce(dphi, dphi, 2 * (size_t)P->n, ncclDouble, ncclSum, c, P->stream));
    FMM2D_NCCL_TRY(A->GroupEnd());
    return 0;
}

void shard_halo_sizes(const fmm2d_plan* P, int64_t* leaves, int64_t* mpoles, int64_t* exp_leaves, int64_t* exp_mp)
{
    *leaves = P->shard ? P->shard->leaf.imp_tot : 0;
    *mpoles = P->shard ? P->shard->mp.imp_tot : 0;
    *exp_leaves = P->shard ? P->shard->leaf.exp_tot : 0;
    *exp_mp = P->shard ? P->shard->mp.exp_tot : 0;
}

}  // namespace fmm2d
