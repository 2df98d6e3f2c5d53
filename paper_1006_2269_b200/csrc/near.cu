// near.cu -- A9-A11: L2P + P2P over the strong leaf lists, written back in input order.
//
// Paper: "at the finest level, the remaining strong connections are evaluated
// directly"; the pairwise term is m_j log(z_i - z_j) of Eq. 1
// with j != i by index; the result is returned in input order.
//
// GPU formulation: one CTA of 128 threads per target leaf t.
// The sources of t's strong list are staged through shared memory in chunks of up
// to NEAR_CHUNK 32-byte rows {x, y, Re m, Im m} (whole leaves, at most 32 per chunk;
// warp 0 scans the leaf sizes, all four warps copy).  Each thread owns TWO targets
// (register blocking: every source row loaded from shared memory feeds two pairs)
// and one of G source groups; group g walks chunk rows g, g+G, ...  Rows of t's own
// leaf are walked in a separate short range where the self pair j == i is neutralised
// (dz := 1, m := 0), so the main loop carries no per-pair test.  Log(dz) and 1/dz use
// the table-driven FP64 routines of fastmath.cuh (tables in shared memory).  The G
// partial sums per target are reduced in shared memory in fixed group order
// (deterministic), the L2P Horner evaluation of t's local expansion is added, and the
// result is stored at the input position perm[i].
// Leaves larger than NEAR_CHUNK (only when nlevels forces a shallow tree) take
// k_near_wide, which reads sources straight from global memory.
#include "fastmath.cuh"
#include "fmm2d_internal.cuh"

namespace fmm2d {

namespace {

constexpr int NEAR_T = 128;
#ifndef FMM2D_NEAR_CHUNK
#define FMM2D_NEAR_CHUNK 256
#endif
#ifndef FMM2D_NEAR_MINB
#define FMM2D_NEAR_MINB 8
#endif
constexpr int NEAR_CHUNK = FMM2D_NEAR_CHUNK;    // >= 256: the chunk buffer doubles as reduction space
static_assert(NEAR_CHUNK >= 2 * NEAR_T, "chunk buffer too small for the reduction");

__global__ void k_gather_m(const double2* __restrict__ m, const uint32_t* __restrict__ perm, int64_t n,
                           double4* __restrict__ src)
{
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    double2 v = m[perm[k]];
    double4 s = src[k];
    s.z = v.x;
    s.w = v.y;
    src[k] = s;
}

// Sums of one target: A = sum m log|dz|^2, B = sum m Arg dz, D = sum m conj(dz)/|dz|^2,
// so that Phi = A/2 + i B and Phi' = D (the halving is done once, at the end).
struct PairAcc {
    double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0, dr = 0.0, di = 0.0;
    __device__ __forceinline__ double2 phi() const { return make_double2(0.5 * ar - bi, 0.5 * ai + br); }
    __device__ __forceinline__ double2 dphi() const { return make_double2(dr, di); }
};

// one ordered pair: Phi_i += m Log(dz), Phi'_i += m / dz  (REAL: Im m = 0)
template <bool REAL>
__device__ __forceinline__ void pair(PairAcc& a, double dx, double dy, double mr, double mi,
                                     const fm::Tables& T)
{
    const double r2 = fma(dx, dx, dy * dy);
    const double l2 = fm::log_pos(r2, T.lg);                          // log |dz|^2
    const double th = fm::arg(dx, dy, T.at);                          // Arg dz
    const double ir2 = fm::rcp(r2);
    const double mr2 = mr * ir2;
    a.ar = fma(mr, l2, a.ar);
    a.br = fma(mr, th, a.br);
    a.dr = fma(mr2, dx, a.dr);                                        // m conj(dz) / |dz|^2
    a.di = fma(-mr2, dy, a.di);
    if (!REAL) {
        const double mi2 = mi * ir2;
        a.ai = fma(mi, l2, a.ai);
        a.bi = fma(mi, th, a.bi);
        a.dr = fma(mi2, dy, a.dr);
        a.di = fma(mi2, dx, a.di);
    }
}

__device__ __forceinline__ double4 pack(const PairAcc& a)
{
    const double2 f = a.phi(), g = a.dphi();
    return make_double4(f.x, f.y, g.x, g.y);
}

// L2P (Horner): Phi = sum b_l w^l, Phi' = sum l b_l w^{l-1}, w = z_i - c
__device__ __forceinline__ void l2p(const double2* __restrict__ B, int p, double wx, double wy, double& fr,
                                    double& fi, double& gr, double& gi)
{
    fr = B[p].x;
    fi = B[p].y;
    gr = p * B[p].x;
    gi = p * B[p].y;
    for (int l = p - 1; l >= 0; --l) {
        const double2 b = B[l];
        double nr = fr * wx - fi * wy + b.x;
        double ni = fr * wy + fi * wx + b.y;
        fr = nr;
        fi = ni;
        if (l >= 1) {
            nr = gr * wx - gi * wy + l * b.x;
            ni = gr * wy + gi * wx + l * b.y;
            gr = nr;
            gi = ni;
        }
    }
}

__device__ __forceinline__ void load_tables(fm::Tables& T, const fm::Tables* __restrict__ g)
{
    const double2* gs = (const double2*)g;
    double2* ss = (double2*)&T;
    for (int k = threadIdx.x; k < (int)(sizeof(fm::Tables) / 16); k += blockDim.x) ss[k] = gs[k];
}

// first k >= b with k == g (mod G)
__device__ __forceinline__ int first_in_class(int b, int g, int G)
{
    int r = (g - b) % G;
    return b + (r < 0 ? r + G : r);
}

template <bool REAL>
__global__ void __launch_bounds__(NEAR_T, FMM2D_NEAR_MINB) k_near(int G, int p, const uint32_t* __restrict__ off,
                                                 const int64_t* __restrict__ soff, const uint32_t* __restrict__ sidx,
                                                 const double4* __restrict__ src, const double* __restrict__ cx,
                                                 const double* __restrict__ cy, const double2* __restrict__ loc,
                                                 const uint32_t* __restrict__ perm, const fm::Tables* __restrict__ gtab,
                                                 double2* __restrict__ phi, double2* __restrict__ dphi)
{
    __shared__ double4 S[NEAR_CHUNK];
    __shared__ fm::Tables T;
    double4(*red)[NEAR_T] = reinterpret_cast<double4(*)[NEAR_T]>(S);   // after the last chunk
    __shared__ int cstart[33];
    __shared__ int cinfo[2];                 // [0] leaves in chunk, [1] chunk row of leaf t (-1)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    load_tables(T, gtab);
    const int64_t t = blockIdx.x;
    const uint32_t ts = off[t], te = off[t + 1];
    const int nt = (int)(te - ts);
    const int64_t q0 = soff[t], q1 = soff[t + 1];
    const int tile = NEAR_T / G;                 // target pairs per pass
    for (int i0 = 0; i0 < nt; i0 += 2 * tile) {
        const int tp = tid % tile;
        const int g = tid / tile;
        const int ni = min(2 * tile, nt - i0);   // targets in this pass
        const bool active = (g < G) && (2 * tp < ni);
        const int la = min(2 * tp, ni - 1), lb = min(2 * tp + 1, ni - 1);
        const double4 A = src[ts + i0 + la];
        const double4 B = src[ts + i0 + lb];
        PairAcc aa, ab;
        for (int64_t q = q0; q < q1;) {
            __syncthreads();                      // previous chunk consumed
            if (warp == 0) {
                const int64_t qq = q + lane;
                int sz = 0;
                uint32_t lf = 0;
                if (qq < q1) {
                    lf = sidx[qq];
                    sz = (int)(off[lf + 1] - off[lf]);
                }
                int incl = sz;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    int v = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += v;
                }
                const unsigned fit = __ballot_sync(0xffffffffu, qq < q1 && incl <= NEAR_CHUNK);
                const int nl = __popc(fit);       // leaves in this chunk (prefix property)
                if (lane < nl) cstart[lane + 1] = incl;
                if (lane == 0) {
                    cstart[0] = 0;
                    cinfo[0] = nl;
                    cinfo[1] = -1;
                }
                __syncwarp();
                if (lane < nl && lf == (uint32_t)t) cinfo[1] = incl - sz;
            }
            __syncthreads();
            const int nl = cinfo[0];
            for (int l = warp; l < nl; l += NEAR_T / 32) {
                const uint32_t lf = sidx[q + l];
                const uint32_t s0 = off[lf];
                const int c0 = cstart[l], sz = cstart[l + 1] - c0;
                for (int e = lane; e < sz; e += 32) S[c0 + e] = src[s0 + e];
            }
            __syncthreads();
            const int total = cstart[nl];
            const int kown = (cinfo[1] >= 0) ? cinfo[1] : total;       // own leaf rows [kown, kown+nt)
            const int kend = min(total, kown + nt);
            if (active) {
                // rows before the own leaf, then after it: no self pair possible
#pragma unroll 2
                for (int k = g; k < kown; k += G) {
                    const double4 s = S[k];
                    pair<REAL>(aa, A.x - s.x, A.y - s.y, s.z, s.w, T);
                    pair<REAL>(ab, B.x - s.x, B.y - s.y, s.z, s.w, T);
                }
#pragma unroll 2
                for (int k = first_in_class(kend, g, G); k < total; k += G) {
                    const double4 s = S[k];
                    pair<REAL>(aa, A.x - s.x, A.y - s.y, s.z, s.w, T);
                    pair<REAL>(ab, B.x - s.x, B.y - s.y, s.z, s.w, T);
                }
                // own leaf: neutralise j == i
                const int sa = kown + i0 + la, sb = kown + i0 + lb;
                for (int k = first_in_class(kown, g, G); k < kend; k += G) {
                    const double4 s = S[k];
                    const bool xa = (k == sa), xb = (k == sb);
                    pair<REAL>(aa, xa ? 1.0 : A.x - s.x, xa ? 0.0 : A.y - s.y, xa ? 0.0 : s.z, xa ? 0.0 : s.w, T);
                    pair<REAL>(ab, xb ? 1.0 : B.x - s.x, xb ? 0.0 : B.y - s.y, xb ? 0.0 : s.z, xb ? 0.0 : s.w, T);
                }
            }
            q += nl;
        }
        __syncthreads();                          // chunk buffer free: reuse it for partial sums
        red[0][tid] = pack(aa);
        red[1][tid] = pack(ab);
        __syncthreads();
        // finalize: 2*tile targets, thread k < ni handles target k (pair tp = k/2, slot k&1)
        for (int kk = tid; kk < ni; kk += NEAR_T) {
            const int ptp = kk >> 1, slot = kk & 1;
            double4 acc = red[slot][ptp];
            for (int gg = 1; gg < G; ++gg) {
                const double4 v = red[slot][gg * tile + ptp];
                acc.x += v.x;
                acc.y += v.y;
                acc.z += v.z;
                acc.w += v.w;
            }
            const uint32_t i = ts + i0 + kk;
            const double4 me = src[i];
            double fr, fi, gr, gi;
            l2p(loc + t * (p + 1), p, me.x - cx[t], me.y - cy[t], fr, fi, gr, gi);
            const uint32_t o = perm[i];
            if (phi) phi[o] = make_double2(acc.x + fr, acc.y + fi);
            if (dphi) dphi[o] = make_double2(acc.z + gr, acc.w + gi);
        }
        __syncthreads();
    }
}

// Wide leaves (> NEAR_CHUNK points): sources straight from global memory.
template <bool REAL>
__global__ void __launch_bounds__(NEAR_T) k_near_wide(int p, const uint32_t* __restrict__ off,
                                                      const int64_t* __restrict__ soff,
                                                      const uint32_t* __restrict__ sidx,
                                                      const double4* __restrict__ src, const double* __restrict__ cx,
                                                      const double* __restrict__ cy, const double2* __restrict__ loc,
                                                      const uint32_t* __restrict__ perm,
                                                      const fm::Tables* __restrict__ gtab, double2* __restrict__ phi,
                                                      double2* __restrict__ dphi)
{
    __shared__ fm::Tables T;
    load_tables(T, gtab);
    __syncthreads();
    const int64_t t = blockIdx.x;
    const uint32_t ts = off[t], te = off[t + 1];
    for (uint32_t i = ts + threadIdx.x; i < te; i += NEAR_T) {
        const double4 me = src[i];
        PairAcc acc;
        for (int64_t q = soff[t]; q < soff[t + 1]; ++q) {
            const uint32_t lf = sidx[q];
            for (uint32_t j = off[lf]; j < off[lf + 1]; ++j) {
                const double4 s = src[j];
                const bool self = (j == i);
                pair<REAL>(acc, self ? 1.0 : me.x - s.x, self ? 0.0 : me.y - s.y, self ? 0.0 : s.z,
                           self ? 0.0 : s.w, T);
            }
        }
        double fr, fi, gr, gi;
        l2p(loc + t * (p + 1), p, me.x - cx[t], me.y - cy[t], fr, fi, gr, gi);
        const uint32_t o = perm[i];
        const double2 f = acc.phi(), d = acc.dphi();
        if (phi) phi[o] = make_double2(f.x + fr, f.y + fi);
        if (dphi) dphi[o] = make_double2(d.x + gr, d.y + gi);
    }
}

inline unsigned grid_for(int64_t n, int bs) { return (unsigned)((n + bs - 1) / bs); }

// per-device table copy (built once on the host, long double evaluation)
const fm::Tables* device_tables(int dev, int* rc)
{
    static const fm::Tables* cache[64] = {nullptr};
    *rc = 0;
    if (dev < 0 || dev >= 64) {
        *rc = FMM2D_EINVAL;
        return nullptr;
    }
    if (cache[dev]) return cache[dev];
    static fm::Tables h;
    fm::make_tables(&h);
    fm::Tables* d = nullptr;
    cudaError_t e = cudaMalloc((void**)&d, sizeof(fm::Tables));
    if (e == cudaSuccess) e = cudaMemcpy(d, &h, sizeof(h), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        fmm2d_set_last_cuda_error(e, "device_tables", __FILE__, __LINE__);
        *rc = FMM2D_ECUDA;
        return nullptr;
    }
    cache[dev] = d;
    return d;
}

}  // namespace

int gather_strengths(fmm2d_plan* P, const double2* m)
{
    k_gather_m<<<grid_for(P->n, 256), 256, 0, P->stream>>>(m, P->perm, P->n, P->src);
    fmm2d::note_launch();
    FMM2D_CUDA_TRY(cudaGetLastError());
    return 0;
}

int prepare_near(fmm2d_plan* P)
{
    int rc = 0;
    P->tables = device_tables(P->device, &rc);
    return rc;
}

int run_near(fmm2d_plan* P, double2* phi, double2* dphi)
{
    const int L = P->L;
    const int64_t nl = nboxes(L);
    const double* cx = P->cx + P->base[L];
    const double* cy = P->cy + P->base[L];
    const double2* loc = P->local + P->base[L] * (P->p + 1);
    const uint32_t* off = P->boff + P->obase[L];
    const bool real = (P->flags & FMM2D_REAL_STRENGTHS) != 0;
    const fm::Tables* tab = (const fm::Tables*)P->tables;
    if (P->stats.max_leaf <= NEAR_CHUNK) {
        // target pairs per leaf, groups so that pairs * G <= 128
        const int pairs = (std::max(1, P->stats.max_leaf) + 1) / 2;
        int G = NEAR_T / std::min(pairs, NEAR_T);
        if (G < 1) G = 1;
        if (real)
            k_near<true><<<(unsigned)nl, NEAR_T, 0, P->stream>>>(G, P->p, off, P->strong[L].off, P->strong[L].idx,
                                                                P->src, cx, cy, loc, P->perm, tab, phi, dphi);
        else
            k_near<false><<<(unsigned)nl, NEAR_T, 0, P->stream>>>(G, P->p, off, P->strong[L].off, P->strong[L].idx,
                                                                 P->src, cx, cy, loc, P->perm, tab, phi, dphi);
    } else {
        if (real)
            k_near_wide<true><<<(unsigned)nl, NEAR_T, 0, P->stream>>>(P->p, off, P->strong[L].off, P->strong[L].idx,
                                                                     P->src, cx, cy, loc, P->perm, tab, phi, dphi);
        else
            k_near_wide<false><<<(unsigned)nl, NEAR_T, 0, P->stream>>>(P->p, off, P->strong[L].off,
                                                                      P->strong[L].idx, P->src, cx, cy, loc,
                                                                      P->perm, tab, phi, dphi);
    }
    fmm2d::note_launch();
    FMM2D_CUDA_TRY(cudaGetLastError());
    return 0;
}

}  // namespace fmm2d
