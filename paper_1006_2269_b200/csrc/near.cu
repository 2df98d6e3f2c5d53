// near.cu -- A9-A11: L2P + P2P over the strong leaf lists, written back in input order.
//
// Paper: "at the finest level, the remaining strong connections are evaluated
// directly"; the pairwise term is m_j log(z_i - z_j) of Eq. 1
// with j != i by index; the result is returned in input order.
//
// GPU formulation: one CTA of 128 threads per target leaf.
// Thread t owns target i = t mod n_t and source group g = t / n_t (G groups,
// G * n_t <= 128); group g walks sources j = g, g+G, ... of every leaf in the
// target's strong list.  All threads of a CTA read the same source leaf at the same
// time (broadcast loads of 32-byte rows through L1).  The G partial sums per target
// are reduced in shared memory in fixed group order (deterministic), the L2P
// Horner evaluation of the leaf's local expansion is added, and the result is
// stored at the input position perm[i].
#include "fmm2d_internal.cuh"

namespace fmm2d {

namespace {

constexpr int NEAR_T = 128;

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

template <bool REAL>
__global__ void __launch_bounds__(NEAR_T) k_near(int G, int p, const uint32_t* __restrict__ off,
                                                 const int64_t* __restrict__ soff,
                                                 const uint32_t* __restrict__ sidx,
                                                 const double4* __restrict__ src, const double* __restrict__ cx,
                                                 const double* __restrict__ cy, const double2* __restrict__ loc,
                                                 const uint32_t* __restrict__ perm, double2* __restrict__ phi,
                                                 double2* __restrict__ dphi)
{
    __shared__ double4 red[NEAR_T];
    const int64_t t = blockIdx.x;
    const uint32_t ts = off[t], te = off[t + 1];
    const int nt = (int)(te - ts);
    const int64_t q0 = soff[t], q1 = soff[t + 1];
    // tile the leaf's targets by NEAR_T / G (only one tile unless the leaf is large)
    const int tile = NEAR_T / G;
    for (int i0 = 0; i0 < nt; i0 += tile) {
        const int li = threadIdx.x % tile;
        const int g = threadIdx.x / tile;
        const int ni = min(tile, nt - i0);
        const bool active = (g < G) && (li < ni);
        const uint32_t i = ts + i0 + li;
        double xi = 0.0, yi = 0.0;
        if (active) {
            double4 s = src[i];
            xi = s.x;
            yi = s.y;
        }
        double pr = 0.0, pi = 0.0, dr = 0.0, di = 0.0;
        for (int64_t q = q0; q < q1; ++q) {
            const uint32_t sb = sidx[q];
            const uint32_t js = off[sb], je = off[sb + 1];
            if (!active) continue;
            for (uint32_t j = js + g; j < je; j += G) {
                if (j == i) continue;                                   // j != i (Eq. 1)
                const double4 s = src[j];
                const double dx = xi - s.x, dy = yi - s.y;
                const double r2 = dx * dx + dy * dy;
                const double lr = 0.5 * log(r2);                        // log|z_i - z_j|
                const double th = atan2(dy, dx);                         // Arg, principal
                const double ir2 = 1.0 / r2;
                const double ux = dx * ir2, uy = -dy * ir2;              // 1/(z_i - z_j)
                if (REAL) {
                    pr = fma(s.z, lr, pr);
                    pi = fma(s.z, th, pi);
                    dr = fma(s.z, ux, dr);
                    di = fma(s.z, uy, di);
                } else {
                    pr += s.z * lr - s.w * th;
                    pi += s.z * th + s.w * lr;
                    dr += s.z * ux - s.w * uy;
                    di += s.z * uy + s.w * ux;
                }
            }
        }
        red[threadIdx.x] = make_double4(pr, pi, dr, di);
        __syncthreads();
        if (g == 0 && li < ni) {
            for (int gg = 1; gg < G; ++gg) {
                double4 v = red[gg * tile + li];
                pr += v.x;
                pi += v.y;
                dr += v.z;
                di += v.w;
            }
            // L2P: Phi += sum b_l w^l, Phi' += sum l b_l w^{l-1} (Horner), w = z_i - c
            const double2* B = loc + (int64_t)t * (p + 1);
            const double wx = xi - cx[t], wy = yi - cy[t];
            double fr = B[p].x, fi = B[p].y;
            double gr = p * B[p].x, gi = p * B[p].y;
            for (int l = p - 1; l >= 0; --l) {
                const double2 b = B[l];
                double nr = fr * wx - fi * wy + b.x;
                double ni2 = fr * wy + fi * wx + b.y;
                fr = nr;
                fi = ni2;
                if (l >= 1) {
                    nr = gr * wx - gi * wy + l * b.x;
                    ni2 = gr * wy + gi * wx + l * b.y;
                    gr = nr;
                    gi = ni2;
                }
            }
            const uint32_t o = perm[i];
            if (phi) phi[o] = make_double2(pr + fr, pi + fi);
            if (dphi) dphi[o] = make_double2(dr + gr, di + gi);
        }
        __syncthreads();
    }
}

inline unsigned grid_for(int64_t n, int bs) { return (unsigned)((n + bs - 1) / bs); }

}  // namespace

int gather_strengths(fmm2d_plan* P, const double2* m)
{
    k_gather_m<<<grid_for(P->n, 256), 256, 0, P->stream>>>(m, P->perm, P->n, P->src); fmm2d::note_launch();
    FMM2D_CUDA_TRY(cudaGetLastError());
    return 0;
}

int run_near(fmm2d_plan* P, double2* phi, double2* dphi)
{
    const int L = P->L;
    int G = NEAR_T / std::max(1, P->stats.max_leaf);
    if (G < 1) G = 1;
    int64_t nl = nboxes(L);
    const double* cx = P->cx + P->base[L];
    const double* cy = P->cy + P->base[L];
    const double2* loc = P->local + P->base[L] * (P->p + 1);
    if (P->flags & FMM2D_REAL_STRENGTHS)
        k_near<true><<<(unsigned)nl, NEAR_T, 0, P->stream>>>(G, P->p, P->boff + P->obase[L], P->strong[L].off,
                                                            P->strong[L].idx, P->src, cx, cy, loc, P->perm,
                                                            phi, dphi);
    else
        k_near<false><<<(unsigned)nl, NEAR_T, 0, P->stream>>>(G, P->p, P->boff + P->obase[L], P->strong[L].off,
                                                             P->strong[L].idx, P->src, cx, cy, loc, P->perm,
                                                             phi, dphi);
    fmm2d::note_launch();
    FMM2D_CUDA_TRY(cudaGetLastError());
    return 0;
}

}  // namespace fmm2d
