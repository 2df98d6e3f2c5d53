// rr.cu -- the r/R exchange of the paper (DESIGN R23): P2L of the larger leaves'
// sources into a leaf's local expansion and M2P of the smaller leaves' multipoles at its
// points, for the leaf pairs k_rr_lists moved out of the near field.  (Own translation unit:
// the table-driven FP64 routines of fastmath.cuh carry __constant__ data that would share the
// constant bank with M2L's transition matrix.)
#include <algorithm>

#include "fmm2d_internal.cuh"
#include "fastmath.cuh"

namespace fmm2d {

namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b)
{
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// ---------------------------------------------------------------- r/R exchange (DESIGN R23)
// P2L: the sources of the larger leaves in a leaf's P2L list go straight into
// its local expansion: b_0 += m Log(c - z_j), b_l += -m / (l (z_j - c)^l) (c - z_j and
// z_j - c each formed componentwise, R2).  One block of RR_T threads per leaf with P2L
// work: warp w takes list entries w, w + RR_W, ...; lanes over each entry's sources;
// coefficients in registers, a fixed-order shuffle reduction per warp, the warps'
// partials summed in warp order in shared memory and added to the local.  Per source:
// log|.|, Arg and 1/|.|^2 by the table-driven routines of fastmath.cuh (tables in shared
// memory, as in k_near), t_l = m iv^l by one complex product per l, b_l -= t_l / l.
constexpr int RR_T = 128, RR_W = RR_T / 32;
// Leaves with at most FMM2D_RR_SHORT list entries (most leaves; k_rr_lists' leaf arrays
// hold them at the front): P2L a thread per leaf (k_rr_p2l_t), M2P a warp per leaf
// (k_rr_m2p_w); longer lists (non-uniform inputs: up to thousands of entries, at the back
// of the arrays): a block each (k_rr_p2l, k_rr_m2p).  C5 with the exchange: P2L + M2P
// 16.3 -> 4.4 ms (a block per leaf left most warps idle and reloaded 8 KB of tables per leaf).
#ifndef FMM2D_RR_WARP
#define FMM2D_RR_WARP 1
#endif
#ifndef FMM2D_RR_P2L_THREAD
#define FMM2D_RR_P2L_THREAD 1           // short P2L lists: a thread per leaf (else a warp)
#endif

__device__ __forceinline__ void rr_load_tables(fm::Tables& T, const fm::Tables* __restrict__ g)
{
    const double2* gs = reinterpret_cast<const double2*>(g);
    double2* ss = reinterpret_cast<double2*>(&T);
    for (int k = threadIdx.x; k < (int)(sizeof(fm::Tables) / 16); k += blockDim.x) ss[k] = gs[k];
}

template <int P>
__global__ void __launch_bounds__(RR_T) k_rr_p2l(const uint32_t* __restrict__ leaves,
                                                 const int64_t* __restrict__ off, const uint32_t* __restrict__ idx,
                                                 const uint32_t* __restrict__ boff, const double4* __restrict__ src,
                                                 const double* __restrict__ cx, const double* __restrict__ cy,
                                                 double2* __restrict__ loc, const fm::Tables* __restrict__ gtab)
{
    __shared__ double2 part[RR_W][P + 1];
    __shared__ fm::Tables T;
    const uint32_t t = leaves[blockIdx.x];
    rr_load_tables(T, gtab);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double ctx = cx[t], cty = cy[t];
    double2 b[P + 1];
#pragma unroll
    for (int l = 0; l <= P; ++l) b[l] = make_double2(0.0, 0.0);
    for (int64_t q = off[t] + warp; q < off[t + 1]; q += RR_W) {
        const uint32_t s = idx[q];
        for (uint32_t j = boff[s] + lane; j < boff[s + 1]; j += 32) {
            const double4 z = src[j];
            const double2 m = make_double2(z.z, z.w);
            const double ux = ctx - z.x, uy = cty - z.y;              // c - z_j
            const double r2 = fma(ux, ux, uy * uy);
            const double2 lg = make_double2(0.5 * fm::log_pos(r2, T.lg), fm::arg_t(ux, uy, T.at));
            b[0] = cadd(b[0], cmul(m, lg));
            const double vx = z.x - ctx, vy = z.y - cty;              // z_j - c
            const double iv2 = fm::rcp(fma(vx, vx, vy * vy));
            const double2 iv = make_double2(vx * iv2, -vy * iv2);
            double2 tl = m;
#pragma unroll
            for (int l = 1; l <= P; ++l) {
                tl = cmul(tl, iv);                                     // m iv^l
                const double c = -1.0 / l;
                b[l].x = fma(c, tl.x, b[l].x);
                b[l].y = fma(c, tl.y, b[l].y);
            }
        }
    }
#pragma unroll
    for (int l = 0; l <= P; ++l) {
        for (int o = 16; o; o >>= 1) {
            b[l].x += __shfl_xor_sync(0xffffffffu, b[l].x, o);
            b[l].y += __shfl_xor_sync(0xffffffffu, b[l].y, o);
        }
    }
    if (lane == 0) {
#pragma unroll
        for (int l = 0; l <= P; ++l) part[warp][l] = b[l];
    }
    __syncthreads();
    if (threadIdx.x <= P) {
        const int l = threadIdx.x;
        double2 v = part[0][l];
        for (int w = 1; w < RR_W; ++w) v = cadd(v, part[w][l]);
        double2* Lc = loc + (int64_t)t * (P + 1);
        Lc[l] = cadd(Lc[l], v);
    }
}

// M2P: the multipoles of the smaller leaves in a leaf's M2P list evaluated at
// each of its points: Phi += a_0 Log(w) + sum_k a_k x^k and Phi' += a_0 x - x^2 sum_k k a_k
// x^(k-1), w = z_i - c_s (componentwise), x = 1/w.  Both sums from one Horner pass over
// H(x) = sum_k a_k x^(k-1) and its derivative (sum_k k a_k x^(k-1) = H + x H').  One
// block per leaf with M2P work: the list's multipoles and centres are staged in shared
// memory in chunks of RR_CH entries (coalesced loads by the whole block); thread (point i,
// group g) takes the chunk's entries g, g + G, ...; the G partial sums of a point are
// added in group order; the sums go to acc[i] (leaf order), k_near adds them.  log|w|,
// Arg w, 1/|w|^2: fastmath.cuh, tables in shared memory.
constexpr int RR_CH = 32;
template <int P>
__global__ void __launch_bounds__(RR_T) k_rr_m2p(const uint32_t* __restrict__ leaves, const int64_t* __restrict__ off,
                                                 const uint32_t* __restrict__ idx, const uint32_t* __restrict__ boff,
                                                 const double4* __restrict__ src, const double* __restrict__ cx,
                                                 const double* __restrict__ cy, const double2* __restrict__ mp,
                                                 double4* __restrict__ acc, const fm::Tables* __restrict__ gtab)
{
    constexpr int E = P + 2;                        // per entry: P + 1 coefficients, the centre
    __shared__ double4 part[RR_T];
    __shared__ double2 sA[RR_CH * E];
    __shared__ fm::Tables T;
    const uint32_t t = leaves[blockIdx.x];
    rr_load_tables(T, gtab);
    const uint32_t ts = boff[t];
    const int nt = (int)(boff[t + 1] - ts);
    const int64_t q0 = off[t], q1 = off[t + 1];
    const int per = min(nt, RR_T);                  // points per pass
    const int G = RR_T / per;                       // list groups
    const int ip = threadIdx.x % per, g = threadIdx.x / per;
    for (int i0 = 0; i0 < nt; i0 += per) {
        const int i = i0 + ip;
        const bool act = g < G && i < nt;
        double2 f = make_double2(0.0, 0.0), df = make_double2(0.0, 0.0);
        double4 z = make_double4(0.0, 0.0, 0.0, 0.0);
        if (act) z = src[ts + i];
        for (int64_t qc = q0; qc < q1; qc += RR_CH) {
            const int nch = (int)min((int64_t)RR_CH, q1 - qc);
            __syncthreads();                        // previous chunk consumed (and the tables)
            for (int e = threadIdx.x; e < nch * E; e += RR_T) {
                const int j = e / E, k = e - j * E;
                const uint32_t s = idx[qc + j];
                sA[e] = (k <= P) ? mp[(int64_t)s * (P + 1) + k] : make_double2(cx[s], cy[s]);
            }
            __syncthreads();
            if (act) {
                for (int j = g; j < nch; j += G) {
                    const double2* A = sA + j * E;
                    const double2 c = A[P + 1];
                    const double wx = z.x - c.x, wy = z.y - c.y;
                    const double r2 = fma(wx, wx, wy * wy);
                    const double iw2 = fm::rcp(r2);
                    const double2 x = make_double2(wx * iw2, -wy * iw2);
                    double2 h = A[P], dh = make_double2(0.0, 0.0);
#pragma unroll
                    for (int k = P - 1; k >= 1; --k) {
                        dh = cadd(cmul(dh, x), h);          // H'
                        h = cadd(cmul(h, x), A[k]);         // H
                    }
                    const double2 d = cadd(h, cmul(x, dh)); // sum_k k a_k x^(k-1)
                    const double2 lg = make_double2(0.5 * fm::log_pos(r2, T.lg), fm::arg_t(wx, wy, T.at));
                    f = cadd(f, cadd(cmul(A[0], lg), cmul(h, x)));
                    df = cadd(df, csub(cmul(A[0], x), cmul(d, cmul(x, x))));
                }
            }
        }
        __syncthreads();
        part[threadIdx.x] = make_double4(f.x, f.y, df.x, df.y);
        __syncthreads();
        if (g == 0 && i < nt) {
            double4 v = part[ip];
            for (int gg = 1; gg < G; ++gg) {
                const double4 u = part[gg * per + ip];
                v.x += u.x;
                v.y += u.y;
                v.z += u.z;
                v.w += u.w;
            }
            acc[ts + i] = v;
        }
    }
}

// Warp-per-leaf forms (FMM2D_RR_WARP, default): most leaves have one or two P2L / M2P
// entries of ~24 sources, so a block per leaf left most of its warps idle and reloaded the
// 8 KB of tables per leaf.  Here persistent blocks load the tables once and each warp takes
// leaves in a grid-stride loop.  P2L: lanes over each entry's sources, the coefficients in
// registers, one fixed-order shuffle reduction per leaf.  M2P: lanes over the leaf's points,
// the entries in list order (multipole coefficients are warp-uniform loads).
template <int P>
__global__ void __launch_bounds__(RR_T) k_rr_p2l_w(const uint32_t* __restrict__ leaves, int64_t nleaves,
                                                   const int64_t* __restrict__ off, const uint32_t* __restrict__ idx,
                                                   const uint32_t* __restrict__ boff, const double4* __restrict__ src,
                                                   const double* __restrict__ cx, const double* __restrict__ cy,
                                                   double2* __restrict__ loc, const fm::Tables* __restrict__ gtab)
{
    __shared__ fm::Tables T;
    rr_load_tables(T, gtab);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * RR_W;
    for (int64_t li = (int64_t)blockIdx.x * RR_W + (threadIdx.x >> 5); li < nleaves; li += nw) {
        const uint32_t t = leaves[li];
        const double ctx = cx[t], cty = cy[t];
        double2 b[P + 1];
#pragma unroll
        for (int l = 0; l <= P; ++l) b[l] = make_double2(0.0, 0.0);
        for (int64_t q = off[t]; q < off[t + 1]; ++q) {
            const uint32_t s = idx[q];
            for (uint32_t j = boff[s] + lane; j < boff[s + 1]; j += 32) {
                const double4 z = src[j];
                const double2 m = make_double2(z.z, z.w);
                const double ux = ctx - z.x, uy = cty - z.y;          // c - z_j
                const double r2 = fma(ux, ux, uy * uy);
                const double2 lg = make_double2(0.5 * fm::log_pos(r2, T.lg), fm::arg_t(ux, uy, T.at));
                b[0] = cadd(b[0], cmul(m, lg));
                const double vx = z.x - ctx, vy = z.y - cty;          // z_j - c
                const double iv2 = fm::rcp(fma(vx, vx, vy * vy));
                const double2 iv = make_double2(vx * iv2, -vy * iv2);
                double2 tl = m;
#pragma unroll
                for (int l = 1; l <= P; ++l) {
                    tl = cmul(tl, iv);                                 // m iv^l
                    const double c = -1.0 / l;
                    b[l].x = fma(c, tl.x, b[l].x);
                    b[l].y = fma(c, tl.y, b[l].y);
                }
            }
        }
#pragma unroll
        for (int l = 0; l <= P; ++l) {
            for (int o = 16; o; o >>= 1) {
                b[l].x += __shfl_xor_sync(0xffffffffu, b[l].x, o);
                b[l].y += __shfl_xor_sync(0xffffffffu, b[l].y, o);
            }
        }
        double2* Lc = loc + (int64_t)t * (P + 1);
#pragma unroll
        for (int l = 0; l <= P; ++l)
            if (lane == (l & 31)) Lc[l] = cadd(Lc[l], b[l]);
    }
}

// P2L, thread per leaf (short lists): the leaf's coefficients stay in the thread's registers
// over all its entries' sources -- no cross-lane reduction (which cost more than the P2L
// arithmetic of a leaf's one or two entries in the warp-per-leaf form).
template <int P>
__global__ void __launch_bounds__(RR_T) k_rr_p2l_t(const uint32_t* __restrict__ leaves, int64_t nleaves,
                                                   const int64_t* __restrict__ off, const uint32_t* __restrict__ idx,
                                                   const uint32_t* __restrict__ boff, const double4* __restrict__ src,
                                                   const double* __restrict__ cx, const double* __restrict__ cy,
                                                   double2* __restrict__ loc, const fm::Tables* __restrict__ gtab)
{
    __shared__ fm::Tables T;
    rr_load_tables(T, gtab);
    __syncthreads();
    const int64_t li = (int64_t)blockIdx.x * RR_T + threadIdx.x;
    if (li >= nleaves) return;
    const uint32_t t = leaves[li];
    const double ctx = cx[t], cty = cy[t];
    double2 b[P + 1];
#pragma unroll
    for (int l = 0; l <= P; ++l) b[l] = make_double2(0.0, 0.0);
    for (int64_t q = off[t]; q < off[t + 1]; ++q) {
        const uint32_t s = idx[q];
        for (uint32_t j = boff[s]; j < boff[s + 1]; ++j) {
            const double4 z = src[j];
            const double2 m = make_double2(z.z, z.w);
            const double ux = ctx - z.x, uy = cty - z.y;              // c - z_j
            const double r2 = fma(ux, ux, uy * uy);
            const double2 lg = make_double2(0.5 * fm::log_pos(r2, T.lg), fm::arg_t(ux, uy, T.at));
            b[0] = cadd(b[0], cmul(m, lg));
            const double vx = z.x - ctx, vy = z.y - cty;              // z_j - c
            const double iv2 = fm::rcp(fma(vx, vx, vy * vy));
            const double2 iv = make_double2(vx * iv2, -vy * iv2);
            double2 tl = m;
#pragma unroll
            for (int l = 1; l <= P; ++l) {
                tl = cmul(tl, iv);                                     // m iv^l
                const double c = -1.0 / l;
                b[l].x = fma(c, tl.x, b[l].x);
                b[l].y = fma(c, tl.y, b[l].y);
            }
        }
    }
    double2* Lc = loc + (int64_t)t * (P + 1);
#pragma unroll
    for (int l = 0; l <= P; ++l) Lc[l] = cadd(Lc[l], b[l]);
}

template <int P>
__global__ void __launch_bounds__(RR_T) k_rr_m2p_w(const uint32_t* __restrict__ leaves, int64_t nleaves,
                                                   const int64_t* __restrict__ off, const uint32_t* __restrict__ idx,
                                                   const uint32_t* __restrict__ boff, const double4* __restrict__ src,
                                                   const double* __restrict__ cx, const double* __restrict__ cy,
                                                   const double2* __restrict__ mp, double4* __restrict__ acc,
                                                   const fm::Tables* __restrict__ gtab)
{
    __shared__ fm::Tables T;
    rr_load_tables(T, gtab);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * RR_W;
    for (int64_t li = (int64_t)blockIdx.x * RR_W + (threadIdx.x >> 5); li < nleaves; li += nw) {
        const uint32_t t = leaves[li];
        const uint32_t ts = boff[t], te = boff[t + 1];
        const int64_t q0 = off[t], q1 = off[t + 1];
        for (uint32_t i = ts + lane; i < te; i += 32) {
            const double4 z = src[i];
            double2 f = make_double2(0.0, 0.0), df = make_double2(0.0, 0.0);
            for (int64_t q = q0; q < q1; ++q) {
                const uint32_t s = idx[q];
                const double2* __restrict__ A = mp + (int64_t)s * (P + 1);
                const double wx = z.x - cx[s], wy = z.y - cy[s];     // w = z_i - c_s
                const double r2 = fma(wx, wx, wy * wy);
                const double iw2 = fm::rcp(r2);
                const double2 x = make_double2(wx * iw2, -wy * iw2);
                double2 h = A[P], dh = make_double2(0.0, 0.0);
#pragma unroll
                for (int k = P - 1; k >= 1; --k) {
                    dh = cadd(cmul(dh, x), h);          // H'
                    h = cadd(cmul(h, x), A[k]);         // H
                }
                const double2 d = cadd(h, cmul(x, dh)); // sum_k k a_k x^(k-1)
                const double2 a0 = A[0];
                const double2 lg = make_double2(0.5 * fm::log_pos(r2, T.lg), fm::arg_t(wx, wy, T.at));
                f = cadd(f, cadd(cmul(a0, lg), cmul(h, x)));
                df = cadd(df, csub(cmul(a0, x), cmul(d, cmul(x, x))));
            }
            acc[i] = make_double4(f.x, f.y, df.x, df.y);
        }
    }
}

// persistent grid: as many blocks as fit on the device at once (no second wave)
template <typename K>
static unsigned rr_grid(K kernel, int64_t nleaves)
{
    int dev = 0, sms = 148, nb = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, RR_T, 0) != cudaSuccess || nb < 1) nb = 1;
    const int64_t need = (nleaves + RR_W - 1) / RR_W;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)sms * nb));
}

template <int P>
int rr_p2l_p(fmm2d_plan* Pl)
{
    if (Pl->rr_np2l == 0) return 0;
    const int L = Pl->L;
    // short lists: a warp per leaf; long lists (at the back of the leaf array): a block each
    const int64_t ns = FMM2D_RR_WARP ? Pl->rr_np2l_short : 0, nl = Pl->rr_np2l - Pl->rr_np2l_short;
    if (ns > 0 && FMM2D_RR_P2L_THREAD) {
        k_rr_p2l_t<P><<<(unsigned)((ns + RR_T - 1) / RR_T), RR_T, 0, Pl->stream>>>(
            Pl->rr_p2l_leaves, ns, Pl->rr_p2l.off, Pl->rr_p2l.idx, Pl->boff + Pl->obase[L], Pl->src,
            Pl->cx + Pl->base[L], Pl->cy + Pl->base[L], Pl->lcl[L], static_cast<const fm::Tables*>(Pl->tables));
        fmm2d::note_launch();
        FMM2D_CUDA_TRY(cudaGetLastError());
    } else if (ns > 0) {
        k_rr_p2l_w<P><<<rr_grid(k_rr_p2l_w<P>, ns), RR_T, 0, Pl->stream>>>(
            Pl->rr_p2l_leaves, ns, Pl->rr_p2l.off, Pl->rr_p2l.idx, Pl->boff + Pl->obase[L], Pl->src,
            Pl->cx + Pl->base[L], Pl->cy + Pl->base[L], Pl->lcl[L], static_cast<const fm::Tables*>(Pl->tables));
        fmm2d::note_launch();
        FMM2D_CUDA_TRY(cudaGetLastError());
    }
    if (!FMM2D_RR_WARP && Pl->rr_np2l_short > 0) {
        k_rr_p2l<P><<<(unsigned)Pl->rr_np2l_short, RR_T, 0, Pl->stream>>>(
            Pl->rr_p2l_leaves, Pl->rr_p2l.off, Pl->rr_p2l.idx, Pl->boff + Pl->obase[L], Pl->src, Pl->cx + Pl->base[L],
            Pl->cy + Pl->base[L], Pl->lcl[L], static_cast<const fm::Tables*>(Pl->tables));
        fmm2d::note_launch();
        FMM2D_CUDA_TRY(cudaGetLastError());
    }
    if (nl > 0) {
        k_rr_p2l<P><<<(unsigned)nl, RR_T, 0, Pl->stream>>>(
            Pl->rr_p2l_leaves + (Pl->rr_leaf_cap - nl), Pl->rr_p2l.off, Pl->rr_p2l.idx, Pl->boff + Pl->obase[L],
            Pl->src, Pl->cx + Pl->base[L], Pl->cy + Pl->base[L], Pl->lcl[L], static_cast<const fm::Tables*>(Pl->tables));
        fmm2d::note_launch();
        FMM2D_CUDA_TRY(cudaGetLastError());
    }
    return 0;
}

template <int P>
int rr_m2p_p(fmm2d_plan* Pl)
{
    if (Pl->rr_nm2p == 0) return 0;
    const int L = Pl->L;
    const int64_t ns = FMM2D_RR_WARP ? Pl->rr_nm2p_short : 0, nl = Pl->rr_nm2p - Pl->rr_nm2p_short;
    if (ns > 0) {
        k_rr_m2p_w<P><<<rr_grid(k_rr_m2p_w<P>, ns), RR_T, 0, Pl->stream>>>(
            Pl->rr_m2p_leaves, ns, Pl->rr_m2p.off, Pl->rr_m2p.idx, Pl->boff + Pl->obase[L], Pl->src,
            Pl->cx + Pl->base[L], Pl->cy + Pl->base[L], Pl->mpl[L], Pl->rr_acc,
            static_cast<const fm::Tables*>(Pl->tables));
        fmm2d::note_launch();
        FMM2D_CUDA_TRY(cudaGetLastError());
    }
    if (!FMM2D_RR_WARP && Pl->rr_nm2p_short > 0) {
        k_rr_m2p<P><<<(unsigned)Pl->rr_nm2p_short, RR_T, 0, Pl->stream>>>(
            Pl->rr_m2p_leaves, Pl->rr_m2p.off, Pl->rr_m2p.idx, Pl->boff + Pl->obase[L], Pl->src, Pl->cx + Pl->base[L],
            Pl->cy + Pl->base[L], Pl->mpl[L], Pl->rr_acc, static_cast<const fm::Tables*>(Pl->tables));
        fmm2d::note_launch();
        FMM2D_CUDA_TRY(cudaGetLastError());
    }
    if (nl > 0) {
        k_rr_m2p<P><<<(unsigned)nl, RR_T, 0, Pl->stream>>>(
            Pl->rr_m2p_leaves + (Pl->rr_leaf_cap - nl), Pl->rr_m2p.off, Pl->rr_m2p.idx, Pl->boff + Pl->obase[L],
            Pl->src, Pl->cx + Pl->base[L], Pl->cy + Pl->base[L], Pl->mpl[L], Pl->rr_acc,
            static_cast<const fm::Tables*>(Pl->tables));
        fmm2d::note_launch();
        FMM2D_CUDA_TRY(cudaGetLastError());
    }
    return 0;
}


// ---------------------------------------------------------------- M2L: the log terms
// Coefficient 0 of the M2L shift carries a_0 Log(c_t - c_s) (DESIGN R2: the
// componentwise difference).  k_m2l (255 registers, 2 warps per sub-partition) leaves it out; here
// one thread per target box walks the same weak (+ cross-level) list with the table-driven
// log / Arg (<= 2 ulp) at full occupancy and adds the sum to the stored coefficient.  Same work
// order as k_m2l; long-list targets are k_m2l_long's (which keeps the term).
__global__ void __launch_bounds__(128) k_m2l_log(M2LArgs A, int p1, const fm::Tables* __restrict__ gtab)
{
    __shared__ fm::Tables T;
    rr_load_tables(T, gtab);
    __syncthreads();
    const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= A.pre[A.L + 1]) return;
    int lev = 1;
    while (lev < A.L && w >= A.pre[lev + 1]) ++lev;
    const int64_t b = A.order[w];
    const int64_t g = A.base[lev] + b;
    const int64_t w0 = A.woff[lev][b], nw = A.woff[lev][b + 1] - w0;
    const int64_t x0 = A.xoff[lev] ? A.xoff[lev][b] : 0;
    const int64_t jb = nw + (A.xoff[lev] ? A.xoff[lev][b + 1] - x0 : 0);
    if (jb > FMM2D_M2L_LONG || jb == 0) return;
    const uint32_t* __restrict__ widx = A.widx[lev];
    const uint32_t* __restrict__ xidx = A.xidx[lev];
    const int64_t wbase = A.base[lev], xbase = lev > 0 ? A.base[lev - 1] : 0;
    const double ctx = A.cx[g], cty = A.cy[g];
    double sr = 0.0, si = 0.0;
    for (int64_t j = 0; j < jb; ++j) {
        const bool cross = j >= nw;
        const int sl = cross ? lev - 1 : lev;
        const uint32_t bs = cross ? xidx[x0 + (j - nw)] : widx[w0 + j];
        const int64_t s = (cross ? xbase : wbase) + bs;
        const double2* M = (bs >= A.slo[sl] && bs < A.shi[sl]) ? A.mpl[sl] + (int64_t)bs * p1
                                                              : A.mhalo + (int64_t)A.hmap[s] * p1;
        const double2 a0 = M[0];
        const double tx = ctx - A.cx[s], ty = cty - A.cy[s];
        const double r2 = fma(tx, tx, ty * ty);
        const double lr = 0.5 * fm::log_pos(r2, T.lg), li = fm::arg_t(tx, ty, T.at);
        sr += a0.x * lr - a0.y * li;
        si += a0.x * li + a0.y * lr;
    }
    double2* out = A.lcl[lev] + b * p1;
    const double2 o = out[0];
    out[0] = make_double2(o.x + sr, o.y + si);
}

}  // namespace

int m2l_log_terms(fmm2d_plan* P, const M2LArgs& A, int p1)
{
    const int64_t work = A.pre[A.L + 1];
    if (work <= 0) return 0;
    k_m2l_log<<<(unsigned)((work + 127) / 128), 128, 0, P->stream>>>(A, p1, static_cast<const fm::Tables*>(P->tables));
    fmm2d::note_launch();
    FMM2D_CUDA_TRY(cudaGetLastError());
    return 0;
}

#define FMM2D_P_CASES(F)                                                                      \
    case 1: return F<1>(P); case 2: return F<2>(P); case 3: return F<3>(P);                   \
    case 4: return F<4>(P); case 5: return F<5>(P); case 6: return F<6>(P);                   \
    case 7: return F<7>(P); case 8: return F<8>(P); case 9: return F<9>(P);                   \
    case 10: return F<10>(P); case 11: return F<11>(P); case 12: return F<12>(P);             \
    case 13: return F<13>(P); case 14: return F<14>(P); case 15: return F<15>(P);             \
    case 16: return F<16>(P); case 17: return F<17>(P); case 18: return F<18>(P);             \
    case 19: return F<19>(P); case 20: return F<20>(P); case 21: return F<21>(P);             \
    case 22: return F<22>(P); case 23: return F<23>(P); case 24: return F<24>(P);             \
    case 25: return F<25>(P); case 26: return F<26>(P); case 27: return F<27>(P);             \
    case 28: return F<28>(P); case 29: return F<29>(P); case 30: return F<30>(P);             \
    case 31: return F<31>(P); case 32: return F<32>(P);

int run_rr_p2l(fmm2d_plan* P)
{
    if (!(P->flags & FMM2D_RR_EXCHANGE)) return 0;
    switch (P->p) { FMM2D_P_CASES(rr_p2l_p) default: return FMM2D_EINVAL; }
}

int run_rr_m2p(fmm2d_plan* P)
{
    if (!(P->flags & FMM2D_RR_EXCHANGE)) return 0;
    switch (P->p) { FMM2D_P_CASES(rr_m2p_p) default: return FMM2D_EINVAL; }
}

}  // namespace fmm2d
