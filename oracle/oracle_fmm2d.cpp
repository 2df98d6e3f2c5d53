/*
 * oracle_fmm2d.cpp -- plain, slow CPU oracle for the asymmetric adaptive 2D FMM
 * of S. Engblom, "On well-separated sets and fast multipole methods"
 * (arXiv 1006.2269; cited as P:<line> of /root/reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * under paper_1006_2269_b200/ and neither side includes the other.
 *
 * Everything here follows the paper's definitions in the paper's order, with
 * the readings recorded in DESIGN.md section "Readings" (R1..R22):
 *   O0 direct sum            P:57-60 (Eq. 1)
 *   O1 depth rule            P:426-430 (~20 sources per box) + DESIGN R4
 *   O2 median-split tree     P:333-341, Fig. 1 caption P:97-100
 *   O3 box discs             Criterion 1, P:115-123 (spheres containing the sets)
 *   O4 connectivity
 *   O5 expansions / shifts   P:355-362, classical complex forms P:436-440
 *   O6 branch conventions    DESIGN R2
 *   O7 r/R exchange          P:370-377 (optional; leaf level: P2L + M2P instead of P2P)
 *   O8 parent merge          P:364-370 (optional; cross-level M2L from a parent box)
 *   O9 midpoint tree         Fig. 2, Fig. 4 baseline: geometric
 *                            midpoint splits of the bounding square, empty boxes allowed
 * Floating point: compiled with -O2 -ffp-contract=off (no FMA contraction), no
 * fast-math; sqrt is IEEE correctly rounded.  OpenMP is used only across
 * independent boxes / targets, each of which is summed in a fixed order, so
 * the results are bitwise identical for any thread count.
 */
#include <algorithm>
#include <omp.h>
#include <parallel/algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <new>
#include <vector>

typedef std::complex<double> cplx;
typedef std::complex<long double> cplxl;

extern "C" {

/* ------------------------------------------------------------------------- */
/* O0: direct sum, P:57-60 (Eq. 1) with G(z_i,z_j) = m_j log(z_i - z_j).       */
/* Phi_i  = sum_{j != i} m_j Log(z_i - z_j)   (principal Log, Arg in (-pi,pi]) */
/* dPhi_i = sum_{j != i} m_j / (z_i - z_j)                                      */
/* Evaluated in long double.  targets == NULL means all i = 0..n-1.            */
/* z, m: interleaved complex (re, im) arrays of length n.                      */
/* ------------------------------------------------------------------------- */
int oracle_direct(const double* z, const double* m, int64_t n,
                  const int64_t* targets, int64_t ntargets,
                  double* phi, double* dphi)
{
    if (n < 1) return -1;
    int64_t nt = targets ? ntargets : n;
    /* one target per work item: sampled direct sums have few targets and long rows */
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t t = 0; t < nt; ++t) {
        int64_t i = targets ? targets[t] : t;
        cplxl s(0.0L, 0.0L), ds(0.0L, 0.0L);
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;                       /* j != i by index, Eq. 1 */
            /* -0 -> +0 first (DESIGN R6), then componentwise differences */
            long double dx = ((long double)z[2 * i] + 0.0L) - ((long double)z[2 * j] + 0.0L);
            long double dy = ((long double)z[2 * i + 1] + 0.0L) - ((long double)z[2 * j + 1] + 0.0L);
            cplxl dz(dx, dy);
            cplxl mj((long double)m[2 * j], (long double)m[2 * j + 1]);
            s += mj * std::log(dz);                    /* principal Log */
            ds += mj / dz;
        }
        if (phi)  { phi[2 * t] = (double)s.real();  phi[2 * t + 1] = (double)s.imag(); }
        if (dphi) { dphi[2 * t] = (double)ds.real(); dphi[2 * t + 1] = (double)ds.imag(); }
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* O4 predicate: Criterion 1 (theta-criterion).                     */
/*   well separated  <=>  R + theta r <= theta d,                               */
/* d = centre distance, R = max radius, r = min radius.  Evaluated in exactly  */
/* this operation order (DESIGN R10/R11).  The d > 0 guard is DESIGN R9.       */
/* ------------------------------------------------------------------------- */
int oracle_well_separated(double cbx, double cby, double rb,
                          double ccx, double ccy, double rc, double theta)
{
    double dx = cbx - ccx;
    double dy = cby - ccy;
    double d = std::sqrt(dx * dx + dy * dy);
    double R = std::max(rb, rc);
    double r = std::min(rb, rc);
    return (d > 0.0) && (R + theta * r <= theta * d);
}

/* O1: depth rule (DESIGN R4): smallest L >= 0 with n <= 2 * leaf_target * 4^L. */
/* ------------------------------------------------------------------------- */
/* O7 predicate: Criterion 1 "when the roles of r and R are exchanged"          */
/* (P:370-377): for boxes of radii r < R (strictly; equal radii make the two   */
/* criteria identical), r + theta R <= theta d.  Same operation order as the   */
/* criterion (DESIGN R11); d > 0 as R9.  Returns 1 when the exchanged criterion */
/* holds (the caller asks only about pairs that failed Criterion 1).           */
/* ------------------------------------------------------------------------- */
int oracle_rr_exchange(double cbx, double cby, double rb, double ccx, double ccy, double rc, double theta)
{
    double dx = cbx - ccx;
    double dy = cby - ccy;
    double d = std::sqrt(dx * dx + dy * dy);
    double R = std::max(rb, rc);
    double r = std::min(rb, rc);
    return (r < R) && (d > 0.0) && (r + theta * R <= theta * d);
}

int oracle_nlevels(int64_t n, int leaf_target)
{
    if (n < 1 || leaf_target < 1) return -1;
    int L = 0;
    int64_t cap = 2 * (int64_t)leaf_target;
    while (n > cap) { cap *= 4; ++L; }
    return L;
}

/* ------------------------------------------------------------------------- */
/* The plan: tree (O2), discs (O3), connectivity (O4), expansions (O5).        */
/* ------------------------------------------------------------------------- */
struct oracle_plan {
    int64_t n;
    int L;
    double theta;
    std::vector<double> x, y;                        /* canonical coords, input order */
    std::vector<uint32_t> perm;                      /* leaf position -> input index  */
    std::vector<std::vector<int64_t>> off;           /* per level: 4^l + 1 offsets    */
    std::vector<std::vector<double>> cx, cy, rad;    /* per level: 4^l discs          */
    std::vector<std::vector<std::vector<uint32_t>>> strong, weak; /* per level, box */
    /* O7 (rr exchange on): the leaf strong list split into P2P (near), P2L into
     * this smaller box from a larger one (p2l_in), M2P of a smaller box at this
     * larger box's points (m2p_in).  Off: near = strong[L], the others empty. */
    int rr;
    std::vector<std::vector<uint32_t>> near, p2l_in, m2p_in;
    /* O8 (parent merge on): per level l >= 2, box b's cross-level weak list: boxes q of
     * level l-1 whose four children were all weak to b and that are themselves well
     * separated from b; those children are then not in weak[l][b]. */
    int pm;
    std::vector<std::vector<std::vector<uint32_t>>> xweak;
    /* O9: midpoint split policy (empty boxes possible: disc r = -1, centre 0) */
    int midpoint;
    /* expansions from the last oracle_eval (diagnostics) */
    int p;
    std::vector<std::vector<cplx>> mpole, local;     /* per level: 4^l * (p+1)        */
};

static inline int64_t nboxes(int l) { return (int64_t)1 << (2 * l); }

/* total order of DESIGN R6: (coordinate, input index), -0 already mapped to +0 */
struct ByX {
    const oracle_plan* P;
    bool operator()(uint32_t a, uint32_t b) const {
        if (P->x[a] != P->x[b]) return P->x[a] < P->x[b];
        return a < b;
    }
};
struct ByY {
    const oracle_plan* P;
    bool operator()(uint32_t a, uint32_t b) const {
        if (P->y[a] != P->y[b]) return P->y[a] < P->y[b];
        return a < b;
    }
};

static int64_t ceil_half(int64_t n) { return n - n / 2; }

/* A library sort under a STRICT total order (ties broken by the input index, R6), so the
 * result is unique: the OpenMP-parallel GNU sort is used for the few huge segments of the
 * top levels (one box spans all points at level 0), std::sort elsewhere. */
extern "C++" {
template <class Cmp>
static void sort_seg(uint32_t* a, int64_t n, Cmp c)
{
    if (n > (1 << 16) && !omp_in_parallel()) __gnu_parallel::sort(a, a + n, c);
    else std::sort(a, a + n, c);
}
}

/* O2: "recursively splitting the source points at or near their median in each
 * coordinate direction".  DESIGN R5/R7: x first, low side gets the
 * first ceil(n/2) points in (x, idx) order; each half is then split in y the
 * same way.  Children: 4b+0 x-low/y-low, 4b+1 x-low/y-high, 4b+2 x-high/y-low,
 * 4b+3 x-high/y-high ("2^d-tree cut at a certain maximum level").
 * A library sort stands in for the paper's median-of-three quickselect: both
 * produce the same sets under the total order. */
static void build_tree(oracle_plan* P)
{
    const int64_t n = P->n;
    P->perm.resize(n);
    for (int64_t i = 0; i < n; ++i) P->perm[i] = (uint32_t)i;
    P->off.assign(P->L + 1, std::vector<int64_t>());
    P->off[0] = {0, n};
    ByX byx{P};
    ByY byy{P};
    for (int l = 0; l < P->L; ++l) {
        const std::vector<int64_t>& o = P->off[l];
        std::vector<int64_t>& oc = P->off[l + 1];
        oc.assign(4 * nboxes(l) + 1, 0);
        /* few huge boxes: one at a time, each sort parallel inside (sort_seg) */
#pragma omp parallel for schedule(dynamic, 64) if (nboxes(l) >= 256)
        for (int64_t b = 0; b < nboxes(l); ++b) {
            int64_t s = o[b], e = o[b + 1], nb = e - s;
            uint32_t* seg = P->perm.data() + s;
            sort_seg(seg, nb, byx);                            /* x-split */
            int64_t h0 = ceil_half(nb), h1 = nb - h0;
            sort_seg(seg, h0, byy);                            /* y-split of x-low  */
            sort_seg(seg + h0, nb - h0, byy);                  /* y-split of x-high */
            oc[4 * b + 0] = s;
            oc[4 * b + 1] = s + ceil_half(h0);
            oc[4 * b + 2] = s + h0;
            oc[4 * b + 3] = s + h0 + ceil_half(h1);
        }
        oc[4 * nboxes(l)] = n;
    }
    /* DESIGN R13: inside a leaf, ascending (y, idx). */
    const std::vector<int64_t>& oL = P->off[P->L];
#pragma omp parallel for schedule(dynamic, 64) if (nboxes(P->L) >= 256)
    for (int64_t b = 0; b < nboxes(P->L); ++b)
        sort_seg(P->perm.data() + oL[b], oL[b + 1] - oL[b], byy);
}

/* O9: "standard midpoint adaptivity" (Fig. 2) as the uniform baseline of
 * Fig. 4 ("a square and uniformly subdivided multipole mesh").  DESIGN R26:
 * the root is the bounding square [x0, x0 + s) x [y0, y0 + s), s = max(x range, y range)
 * (s = 1 if all points coincide); every box is split at its geometric midpoints, x then y,
 * children 4b + 2 xside + yside as in O2, down to the same depth L.  A point's leaf is
 * (ix, iy) = (floor((x - x0) * S), floor((y - y0) * S)) clamped to 2^L - 1, with
 * S = 2^L / s (one correctly rounded division), interleaved x-high-first.  Inside a leaf
 * the points keep ascending input index (the stable order).  Empty boxes are allowed. */
static void build_tree_midpoint(oracle_plan* P)
{
    const int64_t n = P->n;
    const int L = P->L;
    double x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY;
    for (int64_t i = 0; i < n; ++i) {
        x0 = std::min(x0, P->x[i]); x1 = std::max(x1, P->x[i]);
        y0 = std::min(y0, P->y[i]); y1 = std::max(y1, P->y[i]);
    }
    double side = std::max(x1 - x0, y1 - y0);
    if (!(side > 0.0)) side = 1.0;
    const double S = std::ldexp(1.0, L) / side;
    const int64_t cmax = ((int64_t)1 << L) - 1;
    std::vector<uint64_t> leaf(n);
    for (int64_t i = 0; i < n; ++i) {
        int64_t ix = (int64_t)std::floor((P->x[i] - x0) * S);
        int64_t iy = (int64_t)std::floor((P->y[i] - y0) * S);
        ix = std::min(std::max(ix, (int64_t)0), cmax);
        iy = std::min(std::max(iy, (int64_t)0), cmax);
        uint64_t b = 0;
        for (int j = L - 1; j >= 0; --j) b = 4 * b + 2 * ((ix >> j) & 1) + ((iy >> j) & 1);
        leaf[i] = b;
    }
    P->perm.resize(n);
    for (int64_t i = 0; i < n; ++i) P->perm[i] = (uint32_t)i;
    std::stable_sort(P->perm.begin(), P->perm.end(), [&](uint32_t a, uint32_t b) { return leaf[a] < leaf[b]; });
    P->off.assign(L + 1, std::vector<int64_t>());
    P->off[L].assign(nboxes(L) + 1, 0);
    for (int64_t i = 0; i < n; ++i) P->off[L][leaf[i] + 1] += 1;
    for (int64_t b = 0; b < nboxes(L); ++b) P->off[L][b + 1] += P->off[L][b];
    for (int l = L - 1; l >= 0; --l) {
        P->off[l].assign(nboxes(l) + 1, 0);
        for (int64_t b = 0; b <= nboxes(l); ++b) P->off[l][b] = P->off[L][b << (2 * (L - l))];
    }
}

/* O3: the disc of a box (Criterion 1 asks for spheres containing the sets,
 * P:117-119).  DESIGN R8: centre = midpoint of the tight bounding box, radius
 * = the exact maximum distance from that centre to the box's points. */
static void build_discs(oracle_plan* P)
{
    P->cx.assign(P->L + 1, {});
    P->cy.assign(P->L + 1, {});
    P->rad.assign(P->L + 1, {});
    for (int l = 0; l <= P->L; ++l) {
        int64_t nb = nboxes(l);
        P->cx[l].assign(nb, 0.0);
        P->cy[l].assign(nb, 0.0);
        P->rad[l].assign(nb, 0.0);
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t b = 0; b < nb; ++b) {
            int64_t s = P->off[l][b], e = P->off[l][b + 1];
            if (e == s) {                        /* O9: an empty box has no disc */
                P->cx[l][b] = 0.0; P->cy[l][b] = 0.0; P->rad[l][b] = -1.0;
                continue;
            }
            double xmin = INFINITY, xmax = -INFINITY, ymin = INFINITY, ymax = -INFINITY;
            for (int64_t k = s; k < e; ++k) {
                uint32_t i = P->perm[k];
                xmin = std::min(xmin, P->x[i]); xmax = std::max(xmax, P->x[i]);
                ymin = std::min(ymin, P->y[i]); ymax = std::max(ymax, P->y[i]);
            }
            double cx = 0.5 * (xmin + xmax), cy = 0.5 * (ymin + ymax);
            double r = 0.0;
            for (int64_t k = s; k < e; ++k) {
                uint32_t i = P->perm[k];
                double dx = P->x[i] - cx, dy = P->y[i] - cy;
                r = std::max(r, std::sqrt(dx * dx + dy * dy));
            }
            P->cx[l][b] = cx; P->cy[l][b] = cy; P->rad[l][b] = r;
        }
    }
}

/* O4: connectivity.  "For each box b, the strong connections S(p)
 * of its parent box p are examined; all children of a box in S(p) that satisfy
 * the theta-criterion with respect to b become weakly coupled to b -- the rest
 * remain strongly coupled ... a box is always strongly connected to itself". */
static void build_lists(oracle_plan* P)
{
    P->strong.assign(P->L + 1, {});
    P->weak.assign(P->L + 1, {});
    P->xweak.assign(P->L + 1, {});
    for (int l = 0; l <= P->L; ++l) P->xweak[l].assign(nboxes(l), {});
    P->strong[0].assign(1, std::vector<uint32_t>{0});
    P->weak[0].assign(1, std::vector<uint32_t>{});
    for (int l = 1; l <= P->L; ++l) {
        int64_t nb = nboxes(l);
        P->strong[l].assign(nb, {});
        P->weak[l].assign(nb, {});
        const std::vector<double>& cx = P->cx[l];
        const std::vector<double>& cy = P->cy[l];
        const std::vector<double>& rr = P->rad[l];
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t b = 0; b < nb; ++b) {
            int64_t parent = b / 4;
            if (rr[b] < 0.0) continue;           /* O9: an empty box has no connections */
            for (uint32_t q : P->strong[l - 1][parent]) {
                bool ws[4];
                for (int64_t c = 4 * (int64_t)q; c < 4 * (int64_t)q + 4; ++c)
                    ws[c - 4 * q] = (c != b) && rr[c] >= 0.0 &&
                                    oracle_well_separated(cx[b], cy[b], rr[b], cx[c], cy[c], rr[c], P->theta);
                /* O8: "a box weakly coupled to all children of a parent box can
                 * often interact via the latter instead (whenever the theta-criterion with
                 * respect to that parent is true)".  The parent q is at level l-1. */
                if (P->pm && l >= 2 && ws[0] && ws[1] && ws[2] && ws[3] &&
                    oracle_well_separated(cx[b], cy[b], rr[b], P->cx[l - 1][q], P->cy[l - 1][q],
                                          P->rad[l - 1][q], P->theta)) {
                    P->xweak[l][b].push_back(q);
                    continue;
                }
                for (int64_t c = 4 * (int64_t)q; c < 4 * (int64_t)q + 4; ++c) {
                    if (rr[c] < 0.0) continue;   /* O9: empty candidates take no part */
                    if (ws[c - 4 * q]) P->weak[l][b].push_back((uint32_t)c);
                    else               P->strong[l][b].push_back((uint32_t)c);
                }
            }
        }
    }
}

/* O7: the optional finest-level optimisation of P:370-377.  "A related idea at
 * the finest level is to investigate strongly coupled boxes of very different
 * radii, r << R, say.  If the theta-criterion is true when the roles of r and R
 * are exchanged, then the sources in the larger box can be directly converted
 * into a near field expansion in the smaller box, and the outgoing expansion
 * from the smaller can simply be evaluated at each point in the larger box."
 * For leaf t and each s in its strong list, s != t: if r_t < r_s and the
 * exchanged criterion holds, s's sources go into t's local (p2l_in[t]); if
 * r_s < r_t and it holds, s's multipole is evaluated at t's points (m2p_in[t]);
 * otherwise the pair stays direct (near[t]).  Lists keep the strong order. */
static void build_rr(oracle_plan* P)
{
    const int L = P->L;
    const int64_t nb = nboxes(L);
    P->near.assign(nb, {});
    P->p2l_in.assign(nb, {});
    P->m2p_in.assign(nb, {});
    const std::vector<double>& cx = P->cx[L];
    const std::vector<double>& cy = P->cy[L];
    const std::vector<double>& rr = P->rad[L];
    for (int64_t t = 0; t < nb; ++t) {
        for (uint32_t s : P->strong[L][t]) {
            bool conv = P->rr && (int64_t)s != t &&
                        oracle_rr_exchange(cx[t], cy[t], rr[t], cx[s], cy[s], rr[s], P->theta);
            if (!conv) P->near[t].push_back(s);
            else if (rr[t] < rr[s]) P->p2l_in[t].push_back(s);
            else P->m2p_in[t].push_back(s);
        }
    }
}

int oracle_build_ex(const double* z, int64_t n, double theta, int L, int flags, oracle_plan** out);

int oracle_build(const double* z, int64_t n, double theta, int L, oracle_plan** out)
{
    return oracle_build_ex(z, n, theta, L, 0, out);
}

/* flags bit 0: r/R exchange (O7), bit 1: parent merge (O8), bit 2: midpoint tree (O9) */
int oracle_build_ex(const double* z, int64_t n, double theta, int L, int flags, oracle_plan** out)
{
    if (!out) return -1;
    *out = nullptr;
    if (n < 1 || !(theta > 0.0 && theta < 1.0) || L < 0 || L > 15) return -1;
    if (n < nboxes(L) && !(flags & 4)) return -1;   /* DESIGN R12: no empty boxes (median tree) */
    if (n >= ((int64_t)1 << 31)) return -1;
    for (int64_t i = 0; i < 2 * n; ++i) if (!std::isfinite(z[i])) return -2;
    oracle_plan* P = new (std::nothrow) oracle_plan();
    if (!P) return -3;
    P->n = n; P->L = L; P->theta = theta; P->p = 0;
    P->x.resize(n); P->y.resize(n);
    for (int64_t i = 0; i < n; ++i) {
        /* DESIGN R6: -0 -> +0 (x + 0.0 maps -0 to +0 and leaves others alone) */
        P->x[i] = z[2 * i] + 0.0;
        P->y[i] = z[2 * i + 1] + 0.0;
    }
    P->rr = (flags & 1) ? 1 : 0;
    P->pm = (flags & 2) ? 1 : 0;
    P->midpoint = (flags & 4) ? 1 : 0;
    if (P->midpoint) build_tree_midpoint(P);
    else build_tree(P);
    build_discs(P);
    build_lists(P);
    build_rr(P);
    *out = P;
    return 0;
}

void oracle_free(oracle_plan* P) { delete P; }

int oracle_levels(const oracle_plan* P) { return P ? P->L : -1; }

int oracle_get_perm(const oracle_plan* P, uint32_t* perm)
{
    std::memcpy(perm, P->perm.data(), sizeof(uint32_t) * P->n);
    return 0;
}

int oracle_get_offsets(const oracle_plan* P, int l, int64_t* off)
{
    if (l < 0 || l > P->L) return -1;
    std::memcpy(off, P->off[l].data(), sizeof(int64_t) * (nboxes(l) + 1));
    return 0;
}

int oracle_get_discs(const oracle_plan* P, int l, double* cx, double* cy, double* r)
{
    if (l < 0 || l > P->L) return -1;
    int64_t nb = nboxes(l);
    std::memcpy(cx, P->cx[l].data(), sizeof(double) * nb);
    std::memcpy(cy, P->cy[l].data(), sizeof(double) * nb);
    std::memcpy(r, P->rad[l].data(), sizeof(double) * nb);
    return 0;
}

/* kind 0 = strong, 1 = weak, 5 = cross-level weak (O8, ids of level l-1); leaf level
 * only: 2 = near (P2P), 3 = p2l_in, 4 = m2p_in (O7). */
static const std::vector<std::vector<uint32_t>>& list_of(const oracle_plan* P, int l, int kind)
{
    switch (kind) {
        case 1: return P->weak[l];
        case 5: return P->xweak[l];
        case 2: return P->near;
        case 3: return P->p2l_in;
        case 4: return P->m2p_in;
        default: return P->strong[l];
    }
}

int64_t oracle_list_total(const oracle_plan* P, int l, int kind)
{
    if (l < 0 || l > P->L || kind < 0 || kind > 5 || (kind >= 2 && kind <= 4 && l != P->L)) return -1;
    const auto& LL = list_of(P, l, kind);
    int64_t t = 0;
    for (const auto& v : LL) t += (int64_t)v.size();
    return t;
}

int oracle_get_list(const oracle_plan* P, int l, int kind, int64_t* off, uint32_t* idx)
{
    if (l < 0 || l > P->L || kind < 0 || kind > 5 || (kind >= 2 && kind <= 4 && l != P->L)) return -1;
    const auto& LL = list_of(P, l, kind);
    int64_t t = 0;
    for (size_t b = 0; b < LL.size(); ++b) {
        off[b] = t;
        for (uint32_t c : LL[b]) idx[t++] = c;
    }
    off[LL.size()] = t;
    return 0;
}

/* ------------------------------------------------------------------------- */
/* O5: expansions.  The paper uses "the classical complex polynomial/multipole */
/* representation" and shifts "as usual according to parent/child  */
/* relations"; the forms are written out in DESIGN.md "O5".        */
/* p is the highest retained power (DESIGN R1): p+1 coefficients.              */
/* ------------------------------------------------------------------------- */

/* binomial coefficient C(n,k) by Pascal's rule (the plain definition) */
static std::vector<std::vector<double>> pascal(int nmax)
{
    std::vector<std::vector<double>> C(nmax + 1, std::vector<double>(nmax + 1, 0.0));
    for (int a = 0; a <= nmax; ++a) {
        C[a][0] = 1.0;
        for (int b = 1; b <= a; ++b) C[a][b] = C[a - 1][b - 1] + (b <= a - 1 ? C[a - 1][b] : 0.0);
    }
    return C;
}

/* P2M about c: a_0 = sum m_j, a_k = -sum_j m_j (z_j - c)^k / k, k = 1..p.
 * Far field: a_0 log(z-c) + sum_k a_k (z-c)^-k. */
static void p2m(const cplx* zs, const cplx* ms, int64_t ns, cplx c, int p, cplx* a)
{
    for (int k = 0; k <= p; ++k) a[k] = 0.0;
    for (int64_t j = 0; j < ns; ++j) {
        cplx w = zs[j] - c;
        cplx wk = 1.0;
        a[0] += ms[j];
        for (int k = 1; k <= p; ++k) {
            wk *= w;
            a[k] -= ms[j] * wk / (double)k;
        }
    }
}

/* M2M child centre c -> parent centre c', z0 = c - c':
 *   b_0 = a_0;  b_l = -a_0 z0^l / l + sum_{k=1}^{l} a_k z0^{l-k} C(l-1, k-1). */
static void m2m(const cplx* a, cplx z0, int p, const std::vector<std::vector<double>>& C, cplx* b)
{
    std::vector<cplx> zp(p + 1);
    zp[0] = 1.0;
    for (int l = 1; l <= p; ++l) zp[l] = zp[l - 1] * z0;
    b[0] += a[0];
    for (int l = 1; l <= p; ++l) {
        cplx s = -a[0] * zp[l] / (double)l;
        for (int k = 1; k <= l; ++k) s += a[k] * zp[l - k] * C[l - 1][k - 1];
        b[l] += s;
    }
}

/* M2L multipole at c_s -> local at c_t, z0 = c_s - c_t:
 *   b_0 = a_0 Log(c_t - c_s) + sum_{k=1}^p (-1)^k a_k / z0^k
 *   b_l = -a_0 / (l z0^l) + z0^-l sum_{k=1}^p (-1)^k C(l+k-1, k-1) a_k / z0^k.
 * Log(c_t - c_s) is taken of the componentwise difference (DESIGN R2/O6). */
static void m2l(const cplx* a, double csx, double csy, double ctx, double cty, int p,
                const std::vector<std::vector<double>>& C, cplx* b)
{
    cplx z0(csx - ctx, csy - cty);
    cplx tc(ctx - csx, cty - csy);
    std::vector<cplx> izp(2 * p + 1);               /* z0^-n */
    izp[0] = 1.0;
    cplx iz = 1.0 / z0;
    for (int n = 1; n <= 2 * p; ++n) izp[n] = izp[n - 1] * iz;
    cplx s0 = a[0] * std::log(tc);
    for (int k = 1; k <= p; ++k) s0 += ((k & 1) ? -1.0 : 1.0) * a[k] * izp[k];
    b[0] += s0;
    for (int l = 1; l <= p; ++l) {
        cplx s = -a[0] * izp[l] / (double)l;
        cplx t = 0.0;
        for (int k = 1; k <= p; ++k)
            t += ((k & 1) ? -1.0 : 1.0) * C[l + k - 1][k - 1] * a[k] * izp[k];
        s += izp[l] * t;
        b[l] += s;
    }
}

/* L2L local about c -> c', h = c' - c:  d_k = sum_{l=k}^p b_l C(l,k) h^{l-k}. */
static void l2l(const cplx* b, cplx h, int p, const std::vector<std::vector<double>>& C, cplx* d)
{
    std::vector<cplx> hp(p + 1);
    hp[0] = 1.0;
    for (int l = 1; l <= p; ++l) hp[l] = hp[l - 1] * h;
    for (int k = 0; k <= p; ++k) {
        cplx s = 0.0;
        for (int l = k; l <= p; ++l) s += b[l] * C[l][k] * hp[l - k];
        d[k] += s;
    }
}

/* O7 P2L: the local (near-field) expansion about c of sources z_j, m_j outside
 * the target disc ("the sources in the larger box can be directly
 * converted into a near field expansion in the smaller box"):
 *   log(z - z_j) = Log(c - z_j) + sum_{l>=1} -(z - c)^l / (l (z_j - c)^l),
 * so b_0 += sum_j m_j Log(c - z_j) (componentwise difference, DESIGN R2) and
 * b_l += -sum_j m_j / (l (z_j - c)^l), l = 1..p. */
static void p2l(const cplx* zs, const cplx* ms, int64_t ns, cplx c, int p, cplx* b)
{
    for (int64_t j = 0; j < ns; ++j) {
        cplx u(c.real() - zs[j].real(), c.imag() - zs[j].imag());     /* c - z_j */
        cplx v(zs[j].real() - c.real(), zs[j].imag() - c.imag());     /* z_j - c */
        b[0] += ms[j] * std::log(u);
        cplx iv = 1.0 / v, ivl = 1.0;
        for (int l = 1; l <= p; ++l) {
            ivl *= iv;
            b[l] -= ms[j] * ivl / (double)l;
        }
    }
}

/* O7 M2P: the outgoing expansion of a (smaller) box at c evaluated at z (P:375-376,
 * "the outgoing expansion from the smaller can simply be evaluated at each point
 * in the larger box"): Phi += a_0 Log(z - c) + sum_k a_k (z - c)^-k,
 * dPhi += a_0/(z - c) - sum_k k a_k (z - c)^-(k+1); z - c componentwise. */
static void m2p_eval(const cplx* a, cplx c, int p, cplx z, cplx* phi, cplx* dphi)
{
    cplx w(z.real() - c.real(), z.imag() - c.imag());
    cplx iw = 1.0 / w, iwk = 1.0;
    cplx f = a[0] * std::log(w), df = a[0] * iw;
    for (int k = 1; k <= p; ++k) {
        iwk *= iw;
        f += a[k] * iwk;
        df -= (double)k * a[k] * iwk * iw;
    }
    *phi += f;
    *dphi += df;
}

int oracle_p2l(const double* z, const double* m, int64_t n, double cx, double cy, int p, double* b)
{
    std::vector<cplx> zs(n), ms(n), B(p + 1, 0.0);
    for (int64_t j = 0; j < n; ++j) { zs[j] = cplx(z[2*j], z[2*j+1]); ms[j] = cplx(m[2*j], m[2*j+1]); }
    p2l(zs.data(), ms.data(), n, cplx(cx, cy), p, B.data());
    for (int k = 0; k <= p; ++k) { b[2*k] = B[k].real(); b[2*k+1] = B[k].imag(); }
    return 0;
}

/* exported single-operator entry points (pins; same code as the pipeline) */
int oracle_p2m(const double* z, const double* m, int64_t n, double cx, double cy, int p, double* a)
{
    std::vector<cplx> zs(n), ms(n), A(p + 1);
    for (int64_t j = 0; j < n; ++j) { zs[j] = cplx(z[2*j], z[2*j+1]); ms[j] = cplx(m[2*j], m[2*j+1]); }
    p2m(zs.data(), ms.data(), n, cplx(cx, cy), p, A.data());
    for (int k = 0; k <= p; ++k) { a[2*k] = A[k].real(); a[2*k+1] = A[k].imag(); }
    return 0;
}

int oracle_m2m(const double* a, double cx, double cy, double px, double py, int p, double* b)
{
    auto C = pascal(2 * p + 1);
    std::vector<cplx> A(p + 1), B(p + 1, 0.0);
    for (int k = 0; k <= p; ++k) A[k] = cplx(a[2*k], a[2*k+1]);
    m2m(A.data(), cplx(cx - px, cy - py), p, C, B.data());
    for (int k = 0; k <= p; ++k) { b[2*k] = B[k].real(); b[2*k+1] = B[k].imag(); }
    return 0;
}

int oracle_m2l(const double* a, double csx, double csy, double ctx, double cty, int p, double* b)
{
    auto C = pascal(2 * p + 1);
    std::vector<cplx> A(p + 1), B(p + 1, 0.0);
    for (int k = 0; k <= p; ++k) A[k] = cplx(a[2*k], a[2*k+1]);
    m2l(A.data(), csx, csy, ctx, cty, p, C, B.data());
    for (int k = 0; k <= p; ++k) { b[2*k] = B[k].real(); b[2*k+1] = B[k].imag(); }
    return 0;
}

int oracle_l2l(const double* b, double cx, double cy, double nx, double ny, int p, double* d)
{
    auto C = pascal(2 * p + 1);
    std::vector<cplx> Bv(p + 1), D(p + 1, 0.0);
    for (int k = 0; k <= p; ++k) Bv[k] = cplx(b[2*k], b[2*k+1]);
    l2l(Bv.data(), cplx(nx - cx, ny - cy), p, C, D.data());
    for (int k = 0; k <= p; ++k) { d[2*k] = D[k].real(); d[2*k+1] = D[k].imag(); }
    return 0;
}

/* L2P: Phi += sum_l b_l (z-c)^l ; dPhi += sum_{l>=1} l b_l (z-c)^{l-1}
 * (plain power sums, no Horner). */
static void l2p(const cplx* b, cplx c, int p, cplx z, cplx* phi, cplx* dphi)
{
    cplx w = z - c, wl = 1.0, s = 0.0, ds = 0.0, wlm1 = 1.0;
    for (int l = 0; l <= p; ++l) {
        s += b[l] * wl;
        if (l >= 1) { ds += (double)l * b[l] * wlm1; wlm1 = wl; }
        wl *= w;
    }
    *phi += s;
    *dphi += ds;
}

int oracle_l2p(const double* b, double cx, double cy, int p, const double* z, int64_t n,
               double* phi, double* dphi)
{
    std::vector<cplx> Bv(p + 1);
    for (int k = 0; k <= p; ++k) Bv[k] = cplx(b[2*k], b[2*k+1]);
    for (int64_t i = 0; i < n; ++i) {
        cplx f = 0.0, df = 0.0;
        l2p(Bv.data(), cplx(cx, cy), p, cplx(z[2*i], z[2*i+1]), &f, &df);
        phi[2*i] = f.real(); phi[2*i+1] = f.imag();
        dphi[2*i] = df.real(); dphi[2*i+1] = df.imag();
    }
    return 0;
}

/* Multipole far-field evaluation (O7 M2P; also a pin of P2M) */
int oracle_m2p(const double* a, double cx, double cy, int p, const double* z, int64_t n,
               double* phi, double* dphi)
{
    std::vector<cplx> A(p + 1);
    for (int k = 0; k <= p; ++k) A[k] = cplx(a[2*k], a[2*k+1]);
    for (int64_t i = 0; i < n; ++i) {
        cplx f = 0.0, df = 0.0;
        m2p_eval(A.data(), cplx(cx, cy), p, cplx(z[2*i], z[2*i+1]), &f, &df);
        phi[2*i] = f.real(); phi[2*i+1] = f.imag();
        dphi[2*i] = df.real(); dphi[2*i+1] = df.imag();
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* The evaluation pass: P2M at the leaves -> M2M up -> M2L along   */
/* the weak lists of every level l >= 1 -> L2L down -> L2P + P2P along the     */
/* leaf strong lists -> back to input order.                                   */
/* ------------------------------------------------------------------------- */
int oracle_eval(oracle_plan* P, const double* m, int p, double* phi, double* dphi)
{
    if (!P || p < 1 || p > 64) return -1;
    const int L = P->L;
    const int P1 = p + 1;
    auto C = pascal(2 * p + 1);
    P->p = p;
    std::vector<cplx> zl(P->n), ml(P->n);
    for (int64_t k = 0; k < P->n; ++k) {
        uint32_t i = P->perm[k];
        zl[k] = cplx(P->x[i], P->y[i]);
        ml[k] = cplx(m[2 * i], m[2 * i + 1]);
    }
    P->mpole.assign(L + 1, {});
    P->local.assign(L + 1, {});
    for (int l = 0; l <= L; ++l) {
        P->mpole[l].assign(nboxes(l) * P1, 0.0);
        P->local[l].assign(nboxes(l) * P1, 0.0);
    }
    /* upward: P2M at the leaves */
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t b = 0; b < nboxes(L); ++b) {
        int64_t s = P->off[L][b], e = P->off[L][b + 1];
        p2m(zl.data() + s, ml.data() + s, e - s, cplx(P->cx[L][b], P->cy[L][b]), p,
            P->mpole[L].data() + b * P1);
    }
    /* upward: M2M, children (level l+1) -> parents (level l) */
    for (int l = L - 1; l >= 0; --l) {
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t b = 0; b < nboxes(l); ++b) {
            for (int q = 0; q < 4; ++q) {
                int64_t c = 4 * b + q;
                cplx z0(P->cx[l + 1][c] - P->cx[l][b], P->cy[l + 1][c] - P->cy[l][b]);
                m2m(P->mpole[l + 1].data() + c * P1, z0, p, C, P->mpole[l].data() + b * P1);
            }
        }
    }
    /* M2L along the weak connectivity of every level, then O8's
     * cross-level pairs (multipole of a level l-1 box into a level l local) */
    for (int l = 1; l <= L; ++l) {
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t t = 0; t < nboxes(l); ++t) {
            for (uint32_t s : P->weak[l][t])
                m2l(P->mpole[l].data() + (int64_t)s * P1, P->cx[l][s], P->cy[l][s],
                    P->cx[l][t], P->cy[l][t], p, C, P->local[l].data() + t * P1);
            for (uint32_t q : P->xweak[l][t])
                m2l(P->mpole[l - 1].data() + (int64_t)q * P1, P->cx[l - 1][q], P->cy[l - 1][q],
                    P->cx[l][t], P->cy[l][t], p, C, P->local[l].data() + t * P1);
        }
    }
    /* downward: L2L, parent (level l-1) -> children (level l) */
    for (int l = 1; l <= L; ++l) {
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t c = 0; c < nboxes(l); ++c) {
            int64_t b = c / 4;
            cplx h(P->cx[l][c] - P->cx[l - 1][b], P->cy[l][c] - P->cy[l - 1][b]);
            l2l(P->local[l - 1].data() + b * P1, h, p, C, P->local[l].data() + c * P1);
        }
    }
    /* O7 (rr exchange): sources of larger strongly coupled leaves into the local
     * of the smaller one (after M2L + L2L) */
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t t = 0; t < nboxes(L); ++t) {
        for (uint32_t s : P->p2l_in[t]) {
            int64_t ss = P->off[L][s], se = P->off[L][s + 1];
            p2l(zl.data() + ss, ml.data() + ss, se - ss, cplx(P->cx[L][t], P->cy[L][t]), p,
                P->local[L].data() + t * P1);
        }
    }
    /* leaves: L2P + P2P over the strong leaf connections -- the near
     * list, i.e. the strong list less the O7 conversions -- + O7 M2P */
    std::vector<cplx> f(P->n), df(P->n);
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t t = 0; t < nboxes(L); ++t) {
        int64_t ts = P->off[L][t], te = P->off[L][t + 1];
        for (int64_t i = ts; i < te; ++i) {
            cplx fi = 0.0, dfi = 0.0;
            l2p(P->local[L].data() + t * P1, cplx(P->cx[L][t], P->cy[L][t]), p, zl[i], &fi, &dfi);
            for (uint32_t s : P->near[t]) {
                int64_t ss = P->off[L][s], se = P->off[L][s + 1];
                for (int64_t j = ss; j < se; ++j) {
                    if (j == i) continue;                              /* j != i */
                    cplx dz(zl[i].real() - zl[j].real(), zl[i].imag() - zl[j].imag());
                    fi += ml[j] * std::log(dz);
                    dfi += ml[j] / dz;
                }
            }
            for (uint32_t s : P->m2p_in[t])                            /* O7 */
                m2p_eval(P->mpole[L].data() + (int64_t)s * P1, cplx(P->cx[L][s], P->cy[L][s]), p, zl[i],
                         &fi, &dfi);
            f[i] = fi; df[i] = dfi;
        }
    }
    /* back to input order (FieldResult in original order) */
    for (int64_t k = 0; k < P->n; ++k) {
        uint32_t i = P->perm[k];
        if (phi)  { phi[2 * i] = f[k].real();  phi[2 * i + 1] = f[k].imag(); }
        if (dphi) { dphi[2 * i] = df[k].real(); dphi[2 * i + 1] = df[k].imag(); }
    }
    return 0;
}

/* expansions of the last oracle_eval: kind 0 = multipole, 1 = local */
int oracle_get_expansions(const oracle_plan* P, int l, int kind, double* dst)
{
    if (l < 0 || l > P->L || P->p < 1) return -1;
    const auto& E = kind ? P->local[l] : P->mpole[l];
    std::memcpy(dst, E.data(), sizeof(cplx) * E.size());
    return 0;
}

/* The a-priori relative error law: const * theta^{p+1} / (1-theta)^2,
 * constant normalised to 1 (DESIGN R20). */
double oracle_error_bound(double theta, int p)
{
    return std::pow(theta, p + 1) / ((1.0 - theta) * (1.0 - theta));
}

} /* extern "C" */
