/*
 * fmm2d.h -- C ABI of libfmm2d.so, the B200-native (sm_100a) evaluation pass of
 * the asymmetric adaptive 2D fast multipole method of
 *   S. Engblom, "On well-separated sets and fast multipole methods",
 *   arXiv 1006.2269  (cited as P:<line> of its text).
 *
 * What it computes (Eq. 1, with the log kernel):
 *     Phi(z_i)  = sum_{j != i} m_j * Log(z_i - z_j)
 *     Phi'(z_i) = sum_{j != i} m_j / (z_i - z_j)
 * at every source z_i, by the paper's FMM: a balanced 4-ary tree of median
 * splits, theta-criterion connectivity (Criterion 1, P:115-123;
 * rule P:343-353), upward P2M/M2M, M2L along the weak lists, downward L2L,
 * and L2P + direct P2P along the strong leaf lists.  Readings of
 * points the paper leaves open are DESIGN.md section 2 (R1..R26).
 *
 * Conventions for every entry point:
 *   - Complex arrays are interleaved float64 pairs (re, im), length 2*n doubles,
 *     in INPUT order (index j of z, m, phi, dphi refers to the same source).
 *   - Pointers are CUDA device pointers on opt.stream unless FMM2D_HOST_PTRS is set
 *     in opt.flags, in which case they are host pointers (pinned memory gives the
 *     fastest copies) and the call returns after the results are in host memory
 *     (with FMM2D_ASYNC_HOST: once their copies are enqueued on opt.stream).
 *   - Return 0 on success, a negative FMM2D_E* code on error; nothing aborts or
 *     exits.  On error the outputs are unspecified and an existing plan is unchanged.
 *   - There is no CPU fallback: every numeric step runs in the library's CUDA kernels.
 */
#ifndef FMM2D_H
#define FMM2D_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define FMM2D_API __attribute__((visibility("default")))
#else
#define FMM2D_API
#endif

#define FMM2D_PMAX 32            /* largest supported truncation order p          */
#define FMM2D_ABI_VERSION 1

/* error codes */
#define FMM2D_OK          0
#define FMM2D_EINVAL     -1      /* theta outside (0,1), p outside 1..PMAX, n < 1,
                                    n >= 2^31, forced nlevels with n < 4^L, NULL args */
#define FMM2D_ENONFINITE -2      /* a coordinate is NaN or +-inf                        */
#define FMM2D_ENOMEM     -3      /* device or host allocation failed                    */
#define FMM2D_ECUDA      -4      /* a CUDA runtime / kernel error                       */
#define FMM2D_ENCCL      -5      /* a NCCL error (multi-rank builds)                    */
#define FMM2D_ENOTSUP    -6      /* unsupported option combination                      */

/* opt.flags */
#define FMM2D_HOST_PTRS       0x1  /* z, m, phi, dphi are host pointers               */
#define FMM2D_REAL_STRENGTHS  0x2  /* caller promises Im m_j == 0 (kernel may skip it) */
#define FMM2D_SYMMETRIC_P2P   0x4  /* evaluate each unordered pair of distinct near leaves
                                      once, feeding both directions (same results up to
                                      rounding; needs a slot buffer; leaves <= 64 points).
                                      Default: every ordered pair separately (measured
                                      faster on B200)            */
#define FMM2D_TREE_KEY64      0x8  /* diagnostic: presort both axes with full 64-bit keys
                                      instead of 32-bit keys + run fix-up (same tree,
                                      DESIGN.md section 6.1)                            */
#define FMM2D_RR_EXCHANGE     0x20  /* the finest-level r/R exchange of P:370-377: strongly
                                      coupled leaves of radii r < R with r + theta R <= theta d
                                      interact by P2L (larger leaf's sources into the
                                      smaller leaf's local) and M2P (smaller leaf's multipole
                                      at the larger leaf's points) instead of the direct
                                      sum (R23).  One GPU only (nranks > 1: ENOTSUP) */
#define FMM2D_PARENT_MERGE    0x40  /* the parent merge of P:364-370: a box weakly coupled to
                                      all four children of a box q interacts with q itself
                                      (cross-level M2L from level l-1) when Criterion 1
                                      holds for the pair (R25)                 */
#define FMM2D_OVERLAP         0x80  /* evaluate the expansion chain (high-priority side stream)
                                      concurrently with the P2P sums, then L2P + output; same
                                      results bit for bit.  Measured slower on B200 (the
                                      kernels' register footprints do not co-reside; DESIGN
                                      6.4), so off by default                            */
#define FMM2D_GATHER_OUTPUT  0x100  /* multi-rank (NCCL) plans: every rank receives ALL entries
                                      of Phi and Phi' (a sum all-reduce over the outputs,
                                      each rank contributing its own sources; 2 x 16 n
                                      bytes per evaluation).  One GPU / loopback: no effect */
#define FMM2D_MIDPOINT       0x200  /* the uniform baseline of Fig. 4: the bounding square split
                                      at geometric midpoints ("standard midpoint
                                      adaptivity", Fig. 2) instead of source medians; empty
                                      boxes allowed (R26).  One GPU only        */
#define FMM2D_ASYNC_HOST     0x400  /* with FMM2D_HOST_PTRS: fmm2d_eval / fmm2d_build_eval
                                      return once the results' device->host copies are
                                      enqueued on opt->stream instead of waiting for them;
                                      the caller synchronises that stream before reading
                                      phi / dphi (fmm2d_free does).  Lets a caller keep two
                                      problems in flight on two streams (the copies of one
                                      overlap the kernels of the other).  On a plan made by
                                      fmm2d_build_eval it covers that call's evaluation
                                      only: later fmm2d_eval calls are synchronous      */
#define FMM2D_TREE_GLOBAL_ONLY 0x10 /* diagnostic: every split step in global memory (no
                                      on-chip finish of the deepest levels; same tree)  */

typedef struct fmm2d_plan fmm2d_plan;   /* opaque; owns all device memory */

typedef struct {
    double theta;        /* Criterion 1 parameter, (0,1) exclusive; rejected (not
                            clamped) otherwise.                              */
    int    p;            /* truncation order: multipole a_0..a_p, local b_0..b_p
                            (DESIGN R1); 1..FMM2D_PMAX.                              */
    int    leaf_target;  /* used when nlevels < 0: L = min L >= 0 with
                            n <= 2*leaf_target*4^L (DESIGN R4).          */
    int    nlevels;      /* >= 0 forces L (requires n >= 4^L); < 0 = automatic.     */
    int    flags;        /* FMM2D_HOST_PTRS | FMM2D_REAL_STRENGTHS | ...             */
    int    device;       /* CUDA device ordinal                                      */
    void*  stream;       /* cudaStream_t for every kernel and copy (NULL = legacy
                            default stream)                                          */
    int    nranks;       /* 1 for one GPU                                            */
    int    rank;         /* 0 for one GPU                                            */
    const void* nccl_id; /* 128-byte ncclUniqueId for nranks > 1, else NULL          */
} fmm2d_options;

/* Fill *opt with defaults: theta 0.5, p 17, leaf_target 40, nlevels -1, flags 0,
 * device 0, stream NULL, nranks 1, rank 0, nccl_id NULL (P:426-430 defaults). */
FMM2D_API int fmm2d_default_options(fmm2d_options* opt);

/* Build the plan for n source positions z (A0-A3 of DESIGN.md: validate, median-split
 * tree P:333-341, box discs, theta-criterion lists P:343-353) and allocate the
 * expansions for order opt->p.  z: n complex positions (interleaved), read during
 * the call only.  Synchronous: returns after the plan is complete (the list sizes
 * are read back to size the allocations).  *out receives the new plan (NULL on
 * error).  Errors: EINVAL, ENONFINITE, ENOMEM, ECUDA. */
FMM2D_API int fmm2d_build(const double* z, int64_t n, const fmm2d_options* opt, fmm2d_plan** out);

/* One evaluation pass for strengths m (A4-A11: P2M, M2M, M2L on every level's weak
 * lists, L2L, L2P + P2P on the strong leaf lists).
 * m:    n complex strengths in input order (read only).
 * phi:  n complex outputs Phi(z_i) in input order, or NULL to skip.
 * dphi: n complex outputs Phi'(z_i) in input order, or NULL to skip.
 * Device pointers: asynchronous on the plan's stream (the caller synchronises).
 * FMM2D_HOST_PTRS: synchronous.  Errors: EINVAL, ECUDA. */
FMM2D_API int fmm2d_eval(fmm2d_plan* plan, const double* m, double* phi, double* dphi);

/* fmm2d_build followed by one fmm2d_eval, for a caller that holds z and m together
 * (same arguments and meaning as those two calls; *out receives the plan, which later
 * fmm2d_eval calls may reuse).  With FMM2D_HOST_PTRS the positions' copy and the build
 * run on an internal high-priority stream, the strengths' host->device copy on a second
 * one as soon as the positions' copy has finished (it overlaps the tree build), and the
 * evaluation and the results' copies on opt->stream; the strengths are then staged in the
 * plan's own buffer.  With FMM2D_ASYNC_HOST as well, two problems can be kept in flight on
 * two caller streams: the next build's kernels are dispatched ahead of the running
 * evaluation's, and each problem's copies overlap the other's kernels.  Synchronous with
 * FMM2D_HOST_PTRS, else stream-ordered like fmm2d_eval.  Multi-GPU plans: not
 * supported (ENOTSUP).  Errors: those of fmm2d_build and fmm2d_eval. */
FMM2D_API int fmm2d_build_eval(const double* z, const double* m, int64_t n, const fmm2d_options* opt,
                               double* phi, double* dphi, fmm2d_plan** out);

/* fmm2d_eval, then synchronise and report the device time of each phase in
 * ms_out[0..7] (CUDA events on the plan's stream): 0 strength gather, 1 P2M+M2M,
 * 2 M2L (all levels), 3 L2L (+ r/R exchange: P2L, M2P), 4 L2P+P2P+output (k_near),
 * 5 total, 6..7 reserved.
 * The phases are run one after the other here (no overlap), so that each is timed alone.
 * Same arguments and errors as fmm2d_eval; ms_out may not be NULL. */
FMM2D_API int fmm2d_eval_timed(fmm2d_plan* plan, const double* m, double* phi, double* dphi,
                               double* ms_out);

/* Grow the library's stream-ordered memory pool on `device` to hold at least `bytes`, once,
 * outside any timed or latency-critical section.  Every plan and every temporary buffer of
 * this library is allocated from this pool: one per device, owned by the library (never the
 * device's default pool, whose attributes are left alone), created on first use, and it keeps
 * freed memory, so later builds reuse it instead of mapping fresh pages (hundreds of ms for
 * tens of GB).  A serving setup step; optional.  Synchronous.  Errors: EINVAL, ENOMEM, ECUDA. */
FMM2D_API int fmm2d_reserve(int device, size_t bytes);

/* Give the memory the library's pool on `device` holds but no live plan uses back to the
 * device, down to keep_bytes (cudaMemPoolTrimTo), e.g. before handing the GPU to another
 * allocator.  Synchronises the device first.  Errors: EINVAL, ECUDA. */
FMM2D_API int fmm2d_pool_trim(int device, size_t keep_bytes);

/* The library pool's device memory in use now and its high-water mark since the last reset
 * (cudaMemPoolAttrUsedMemCurrent / UsedMemHigh), in bytes; reset != 0 restarts the
 * high-water mark.  Diagnostics (per-rank memory of a partitioned build).  Errors: EINVAL,
 * ECUDA. */
FMM2D_API int fmm2d_pool_usage(int device, int64_t* used, int64_t* high, int reset);

/* Number of kernels this library has launched since it was loaded (all plans and
 * threads; CUB's internal launches are not counted). */
FMM2D_API int64_t fmm2d_launch_count(void);

/* ---- several GPUs ------------------------------------------
 * The pass is partitioned by the balanced tree's level-k subtrees: with
 * P ranks (a power of two), k is the smallest level with P | 4^k and rank r owns the
 * level-k subtrees [r 4^k/P, (r+1) 4^k/P) -- equal point counts up to 1 per box.
 * Multi-process (one process per GPU, NCCL): every rank calls fmm2d_build with the
 * SAME full z, n and options except opt.rank, with opt.nranks = P and opt.nccl_id =
 * the 128-byte ncclUniqueId made by fmm2d_nccl_unique_id on one rank and broadcast
 * (e.g. torch.distributed).  fmm2d_build is then collective (all ranks must call it),
 * and so is every fmm2d_eval: each rank passes the same full m and receives Phi, Phi'
 * at the input positions of the sources it owns (other entries are not written, unless
 * FMM2D_GATHER_OUTPUT is set: then every rank receives all entries).
 * The library creates one NCCL communicator per distinct id and keeps it for the
 * life of the process; later builds with the same id (same nranks, same rank) reuse it.
 * The union over ranks equals the one-GPU result.  Errors: ENOTSUP (P not a power of
 * two, or the tree has no level below k), ENCCL (libnccl.so.2 missing or a NCCL
 * failure). */

/* Create a NCCL unique id (128 bytes at out) for a multi-process build. */
FMM2D_API int fmm2d_nccl_unique_id(void* out);

/* Partition facts without a GPU (host arithmetic only; offsets are a function of n):
 * info[0] L, [1] partition level k, [2..3] own leaves [lo, hi), [4..5] own source
 * positions in leaf order [lo, hi), [6..7] own level-k subtrees [lo, hi).
 * opt supplies theta, p, leaf_target and nlevels (validated as in fmm2d_build). */
FMM2D_API int fmm2d_partition_info(int64_t n, const fmm2d_options* opt, int nranks, int rank, int64_t* info);

/* Loopback partition on ONE device (tests of the partitioned path): builds nshards
 * plans, plans[i] being rank i of nshards, in one process on opt->device and
 * opt->stream; every transfer between ranks is a device copy.  Device pointers only
 * (FMM2D_HOST_PTRS: ENOTSUP).  out: array of nshards plan pointers (each freed with
 * fmm2d_free). */
FMM2D_API int fmm2d_build_shards(const double* z, int64_t n, const fmm2d_options* opt, int nshards,
                                 fmm2d_plan** out);
/* Evaluate all shards of a loopback build; every rank writes its own entries of phi
 * and dphi, so on return (stream-ordered) they hold the complete result. */
FMM2D_API int fmm2d_eval_shards(fmm2d_plan* const* plans, int nshards, const double* m, double* phi,
                                double* dphi);

/* Halo facts of a plan: info[0] imported leaves, [1] imported multipoles (per eval),
 * [2] exported leaves, [3] exported multipoles, [4] nranks, [5] rank, [6] k,
 * [7..8] own positions [lo, hi). */
FMM2D_API int fmm2d_halo_info(const fmm2d_plan* plan, int64_t* info);

/* Free the plan and all its device memory.  NULL-safe. */
FMM2D_API void fmm2d_free(fmm2d_plan* plan);

/* Static string for an error code. */
FMM2D_API const char* fmm2d_strerror(int code);

/* Detail of the last CUDA failure seen by this thread ("" if none): the CUDA error
 * string, the failing call and its source location.  Thread-local storage. */
FMM2D_API const char* fmm2d_last_error_detail(void);

/* Plan facts: n, L, p, theta-independent sizes.  Any out pointer may be NULL. */
FMM2D_API int fmm2d_plan_info(const fmm2d_plan* plan, int64_t* n, int* nlevels, int* p,
                    int64_t* weak_pairs, int64_t* strong_leaf_pairs);

/* ---- test / diagnostic exports (copy plan data to HOST memory dst) ----------
 * what:                                 level   dst layout                      */
#define FMM2D_EXPORT_PERM        1  /* -      uint32[n]: leaf position -> input index */
#define FMM2D_EXPORT_OFFSETS     2  /* l      int64[4^l+1]: box ranges in leaf order  */
#define FMM2D_EXPORT_DISCS       3  /* l      double[3*4^l]: cx[], cy[], r[]          */
#define FMM2D_EXPORT_STRONG      4  /* l      int64[4^l+1] offsets then uint32[] idx  */
#define FMM2D_EXPORT_WEAK        5  /* l      int64[4^l+1] offsets then uint32[] idx  */
#define FMM2D_EXPORT_MPOLE       6  /* l      complex128[4^l][p+1] (after an eval)    */
#define FMM2D_EXPORT_LOCAL       7  /* l      complex128[4^l][p+1] (after an eval)    */
#define FMM2D_EXPORT_STATS       8  /* -      double[16]: see api.cu (15: device bytes held) */
#define FMM2D_EXPORT_NEAR        9  /* L      int64[4^L+1] offsets then uint32[]: direct pairs */
#define FMM2D_EXPORT_RR_P2L     10  /* L      same layout: P2L sources of each leaf (r/R exch.) */
#define FMM2D_EXPORT_RR_M2P     11  /* L      same layout: M2P sources of each leaf (r/R exch.) */
#define FMM2D_EXPORT_XWEAK      12  /* l      same layout: cross-level weak entries (ids of level
                                       l-1; parent merge; empty when off)               */
/* If dst is NULL, *bytes receives the required size.  Otherwise *bytes must hold
 * the capacity of dst; on success it receives the bytes written.  Synchronises the
 * plan's stream.  Errors: EINVAL (bad what/level/capacity), ECUDA. */
FMM2D_API int fmm2d_export(const fmm2d_plan* plan, int what, int level, void* dst, size_t* bytes);

#ifdef __cplusplus
}
#endif
#endif /* FMM2D_H */
