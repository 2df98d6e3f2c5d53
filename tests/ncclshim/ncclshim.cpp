/*
 * ncclshim.cpp -- TEST INFRASTRUCTURE.  A stand-in for libnccl.so.2 that lets several
 * processes share ONE GPU, so that the NCCL transport of shard.cu (the exact code path
 * the multi-GPU bench runs: ncclCommInitRank, AllGather, AllReduce, grouped Send/Recv)
 * can execute with more than one process in an environment that has one GPU.  Real
 * NCCL refuses two ranks on one device.
 *
 * libfmm2d.so dlopens it instead of libnccl.so.2 when FMM2D_NCCL_LIB names it
 * (tests/test_gpu_nccl_shim.py only).  It implements the ten entry points shard.cu binds
 * with the CUDA runtime: every rank owns a cudaMalloc'd staging buffer whose IPC handle
 * it publishes in a shared-memory segment (/dev/shm) named after the unique id; an
 * operation is a DEPOSIT (wait for the rank's stream, copy the send buffer into its own
 * staging) and a WITHDRAW (after a host barrier, copy from the peers' mapped staging
 * into the receive buffer; all-reduce: reduce on the host in rank order), then a second
 * host barrier.  Inside ncclGroupStart/End the deposits of all queued operations precede
 * the withdrawals, as NCCL's grouped semantics require.  Every wait is on the host: no
 * kernel ever waits on another process's kernel (B200_PROFILING: one GPU must not stand
 * in for several concurrently running GPUs; this checks the protocol, not the speed).
 */
#include <cuda_runtime.h>
#include <fcntl.h>
#include <nccl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

namespace {

constexpr int kMaxRanks = 16;

struct Shm {
    std::atomic<int> count;
    std::atomic<int> generation;
    std::atomic<int> joined;
    cudaIpcMemHandle_t handle[kMaxRanks];
};

struct Comm {
    int nranks = 0, rank = 0;
    Shm* shm = nullptr;
    char name[64] = {0};
    char* mine = nullptr;                 // own staging (device)
    char* peer[kMaxRanks] = {nullptr};    // mapped staging of every rank (own included)
    size_t bcast_bytes = 0, p2p_bytes = 0;  // staging = [bcast][nranks x p2p]
};

struct Op {
    enum Kind { SEND, RECV, ALLGATHER, ALLREDUCE } kind;
    const void* sbuf;
    void* rbuf;
    size_t bytes;                         // per rank
    int peer;
    ncclDataType_t type;
    ncclRedOp_t op;
    Comm* comm;
    cudaStream_t stream;
};

int g_group = 0;
std::vector<Op> g_ops;
Comm* g_comm = nullptr;                   // the process's communicator (one per process here)
std::atomic<long> g_calls{0};

size_t type_size(ncclDataType_t t)
{
    switch (t) {
        case ncclInt8: case ncclUint8: return 1;
        case ncclFloat16: case ncclBfloat16: return 2;
        case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
        default: return 8;
    }
}

void barrier(Comm* c)
{
    Shm* s = c->shm;
    const int gen = s->generation.load();
    if (s->count.fetch_add(1) == c->nranks - 1) {
        s->count.store(0);
        s->generation.fetch_add(1);
    } else {
        while (s->generation.load() == gen) sched_yield();
    }
}

template <class T>
void reduce_into(T* acc, const T* v, size_t n, ncclRedOp_t op)
{
    for (size_t i = 0; i < n; ++i) {
        if (op == ncclSum) acc[i] += v[i];
        else if (op == ncclMax) acc[i] = v[i] > acc[i] ? v[i] : acc[i];
        else if (op == ncclMin) acc[i] = v[i] < acc[i] ? v[i] : acc[i];
        else acc[i] *= v[i];
    }
}

void reduce_typed(void* acc, const void* v, size_t bytes, ncclDataType_t t, ncclRedOp_t op)
{
    switch (t) {
        case ncclFloat64: reduce_into((double*)acc, (const double*)v, bytes / 8, op); break;
        case ncclFloat32: reduce_into((float*)acc, (const float*)v, bytes / 4, op); break;
        case ncclInt32: reduce_into((int32_t*)acc, (const int32_t*)v, bytes / 4, op); break;
        case ncclUint32: reduce_into((uint32_t*)acc, (const uint32_t*)v, bytes / 4, op); break;
        case ncclInt64: reduce_into((int64_t*)acc, (const int64_t*)v, bytes / 8, op); break;
        case ncclUint64: reduce_into((uint64_t*)acc, (const uint64_t*)v, bytes / 8, op); break;
        default: reduce_into((uint8_t*)acc, (const uint8_t*)v, bytes, op); break;
    }
}

#define SHIM_CUDA(x)                                                                  \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            fprintf(stderr, "ncclshim: %s: %s\n", #x, cudaGetErrorString(e_));        \
            return ncclUnhandledCudaError;                                            \
        }                                                                             \
    } while (0)

// run a batch of operations of one communicator: deposits, barrier, withdrawals, barrier
ncclResult_t run_ops(std::vector<Op>& ops)
{
    // an empty group still takes part in both barriers (the peers' groups may not be empty)
    Comm* c = ops.empty() ? g_comm : ops[0].comm;
    if (!c) return ncclSuccess;
    for (const Op& o : ops)
        if (o.comm != c) return ncclInvalidUsage;        // one communicator per group here
    const int R = c->nranks, me = c->rank;
    // deposits (own staging), in call order
    size_t boff = 0;
    std::vector<size_t> soff(R, 0);
    for (const Op& o : ops) {
        SHIM_CUDA(cudaStreamSynchronize(o.stream));       // the producer's work is done
        if (o.kind == Op::ALLGATHER || o.kind == Op::ALLREDUCE) {
            if (boff + o.bytes > c->bcast_bytes) return ncclInvalidArgument;
            SHIM_CUDA(cudaMemcpy(c->mine + boff, o.sbuf, o.bytes, cudaMemcpyDeviceToDevice));
            boff += o.bytes;
        } else if (o.kind == Op::SEND) {
            if (soff[o.peer] + o.bytes > c->p2p_bytes) return ncclInvalidArgument;
            SHIM_CUDA(cudaMemcpy(c->mine + c->bcast_bytes + c->p2p_bytes * o.peer + soff[o.peer], o.sbuf, o.bytes,
                                 cudaMemcpyDeviceToDevice));
            soff[o.peer] += o.bytes;
        }
    }
    SHIM_CUDA(cudaDeviceSynchronize());                   // device-to-device cudaMemcpy may return early
    barrier(c);
    // withdrawals from the peers' staging
    boff = 0;
    std::vector<size_t> roff(R, 0);
    std::vector<char> acc, tmp;
    for (const Op& o : ops) {
        if (o.kind == Op::ALLGATHER) {
            for (int q = 0; q < R; ++q)
                SHIM_CUDA(cudaMemcpy((char*)o.rbuf + o.bytes * q, c->peer[q] + boff, o.bytes,
                                     cudaMemcpyDeviceToDevice));
            boff += o.bytes;
        } else if (o.kind == Op::ALLREDUCE) {
            acc.resize(o.bytes);
            tmp.resize(o.bytes);
            SHIM_CUDA(cudaMemcpy(acc.data(), c->peer[0] + boff, o.bytes, cudaMemcpyDeviceToHost));
            for (int q = 1; q < R; ++q) {                 // rank order: the same sum on every rank
                SHIM_CUDA(cudaMemcpy(tmp.data(), c->peer[q] + boff, o.bytes, cudaMemcpyDeviceToHost));
                reduce_typed(acc.data(), tmp.data(), o.bytes, o.type, o.op);
            }
            SHIM_CUDA(cudaMemcpy(o.rbuf, acc.data(), o.bytes, cudaMemcpyHostToDevice));
            boff += o.bytes;
        } else if (o.kind == Op::RECV) {
            SHIM_CUDA(cudaMemcpy(o.rbuf, c->peer[o.peer] + c->bcast_bytes + c->p2p_bytes * me + roff[o.peer],
                                 o.bytes, cudaMemcpyDeviceToDevice));
            roff[o.peer] += o.bytes;
        }
    }
    SHIM_CUDA(cudaDeviceSynchronize());
    barrier(c);                                           // nobody reuses staging early
    return ncclSuccess;
}

ncclResult_t submit(const Op& o)
{
    g_calls.fetch_add(1);
    if (g_group > 0) {
        g_ops.push_back(o);
        return ncclSuccess;
    }
    std::vector<Op> one{o};
    return run_ops(one);
}

}  // namespace

extern "C" {

long ncclShimCallCount(void) { return g_calls.load(); }

ncclResult_t ncclGetUniqueId(ncclUniqueId* id)
{
    std::random_device rd;
    memset(id, 0, sizeof(*id));
    for (int i = 0; i < 16; ++i) id->internal[i] = (char)("0123456789abcdef"[rd() & 15]);
    return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* out, int nranks, ncclUniqueId id, int rank)
{
    if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks) return ncclInvalidArgument;
    if (getenv("FMM2D_NCCLSHIM_DEBUG")) fprintf(stderr, "ncclshim: init rank %d of %d\n", rank, nranks);
    Comm* c = new Comm();
    c->nranks = nranks;
    c->rank = rank;
    char tag[17] = {0};
    for (int i = 0; i < 16; ++i) {
        const char ch = id.internal[i];
        tag[i] = ((ch >= '0' && ch <= '9') || (ch >= 'a' && ch <= 'f')) ? ch : 'x';
    }
    snprintf(c->name, sizeof(c->name), "/fmm2d_ncclshim_%s", tag);
    const int fd = shm_open(c->name, O_CREAT | O_RDWR, 0600);
    if (fd < 0 || ftruncate(fd, sizeof(Shm)) != 0) return ncclSystemError;
    c->shm = (Shm*)mmap(nullptr, sizeof(Shm), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (c->shm == MAP_FAILED) return ncclSystemError;
    const char* e = getenv("FMM2D_NCCLSHIM_MB");
    const size_t mb = e ? (size_t)atol(e) : 256;
    c->bcast_bytes = mb << 19;                            // half for broadcasts / reductions
    c->p2p_bytes = (mb << 19) / nranks;                   // half split over the peers
    SHIM_CUDA(cudaMalloc((void**)&c->mine, c->bcast_bytes + c->p2p_bytes * nranks));
    SHIM_CUDA(cudaIpcGetMemHandle(&c->shm->handle[rank], c->mine));
    // wait until every rank has published its handle (the segment starts zeroed)
    c->shm->joined.fetch_add(1);
    while (c->shm->joined.load() < nranks) sched_yield();
    for (int q = 0; q < nranks; ++q) {
        if (q == rank) {
            c->peer[q] = c->mine;
        } else {
            SHIM_CUDA(cudaIpcOpenMemHandle((void**)&c->peer[q], c->shm->handle[q], cudaIpcMemLazyEnablePeerAccess));
        }
    }
    barrier(c);
    g_calls.fetch_add(1);
    g_comm = c;
    *out = (ncclComm_t)c;
    return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm)
{
    Comm* c = (Comm*)comm;
    if (!c) return ncclSuccess;
    barrier(c);
    for (int q = 0; q < c->nranks; ++q)
        if (q != c->rank && c->peer[q]) cudaIpcCloseMemHandle(c->peer[q]);
    barrier(c);
    cudaFree(c->mine);
    munmap(c->shm, sizeof(Shm));
    if (c->rank == 0) shm_unlink(c->name);
    delete c;
    return ncclSuccess;
}

ncclResult_t ncclAllReduce(const void* s, void* r, size_t count, ncclDataType_t t, ncclRedOp_t op, ncclComm_t comm,
                           cudaStream_t st)
{
    return submit(Op{Op::ALLREDUCE, s, r, count * type_size(t), -1, t, op, (Comm*)comm, st});
}

ncclResult_t ncclAllGather(const void* s, void* r, size_t count, ncclDataType_t t, ncclComm_t comm, cudaStream_t st)
{
    return submit(Op{Op::ALLGATHER, s, r, count * type_size(t), -1, t, ncclSum, (Comm*)comm, st});
}

ncclResult_t ncclSend(const void* s, size_t count, ncclDataType_t t, int peer, ncclComm_t comm, cudaStream_t st)
{
    return submit(Op{Op::SEND, s, nullptr, count * type_size(t), peer, t, ncclSum, (Comm*)comm, st});
}

ncclResult_t ncclRecv(void* r, size_t count, ncclDataType_t t, int peer, ncclComm_t comm, cudaStream_t st)
{
    return submit(Op{Op::RECV, nullptr, r, count * type_size(t), peer, t, ncclSum, (Comm*)comm, st});
}

ncclResult_t ncclGroupStart(void)
{
    ++g_group;
    return ncclSuccess;
}

ncclResult_t ncclGroupEnd(void)
{
    if (g_group <= 0) return ncclInvalidUsage;
    if (--g_group > 0) return ncclSuccess;
    std::vector<Op> ops;
    ops.swap(g_ops);
    return run_ops(ops);
}

const char* ncclGetErrorString(ncclResult_t r)
{
    switch (r) {
        case ncclSuccess: return "ncclshim: success";
        case ncclInvalidArgument: return "ncclshim: invalid argument (staging too small? FMM2D_NCCLSHIM_MB)";
        case ncclInvalidUsage: return "ncclshim: invalid usage";
        case ncclUnhandledCudaError: return "ncclshim: CUDA error";
        default: return "ncclshim: error";
    }
}

}  // extern "C"
