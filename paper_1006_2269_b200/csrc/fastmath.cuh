// fastmath.cuh -- FP64 log|z| / Arg z / reciprocal for the P2P inner loop (k_near).
//
// The pairwise term of Eq. 1 needs, per ordered pair, Log(z_i - z_j) =
// log|dz| + i Arg(dz) (principal branch, DESIGN R2) and 1/dz.  libdevice's log and
// atan2 spend ~60 DFMA plus special-case branches and int<->double conversions on
// these; here they are table-driven and branch-free for the finite, normal, non-zero
// arguments the near field produces (r2 = |dz|^2 > 0):
//   log r2 = e ln2 + L_j + log1p(u),  u = f ic_j - 1, f in [1,2) the mantissa of r2,
//            j = its top 8 bits, ic_j ~ 1/(1 + (j+1/2)/256), L_j = -log(ic_j) exactly
//            rounded for the ROUNDED ic_j (f >= 1.5 is taken as 2 (f/2), L_j absorbing
//            the ln 2, so log r2 ~ 0 does not cancel), |u| < 2^-9, degree-6 series.
//            The mantissa is never extracted: with E' = exponent + [f >= 1.5] (one add
//            and one mask on the high word), u = r2 (ic_j 2^-E') - 1 where the table
//            entry's exponent field is lowered by E' (one integer add; the table holds
//            2 ic_j for f >= 1.5, so the product is f ic_j exactly), and e comes from
//            the double {hi 0x43300000, lo E' << 20} = 2^52 + E' 2^20 by one subtraction;
//   Arg    = octant reduction a = atan(mn/mx), mn <= mx; c = mn/mx rounded to a
//            multiple of 1/256 (22-bit estimate + magic-number rounding, no int<->fp
//            conversion); atan(mn/mx) = atan(c) + atan(t), t = (mn - c mx)/(mx + c mn),
//            |t| < 2^-8, degree-5 series; octant: base + s a as one FMA with {base, s}
//            read from the table by (swap, dx < 0), sign of dy by a sign-bit OR;
//   1/x    = MUFU.RCP64H estimate + one cubic Newton step.
// Polynomial coefficients and constants sit in __constant__ memory (a warp-uniform
// DFMA operand).  Error (tests/test_fastmath.py, host build against long double):
// log|dz| <= 2 ulp, Arg <= 2 ulp.  r2 == 0 (coincident distinct points) yields
// log = -inf; subnormal r2 (|dz| < 1.5e-154) is outside the supported
// range.
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#ifdef __CUDACC__
#define FM_HD __host__ __device__ __forceinline__
#else
#define FM_HD static inline
struct double2 {
    double x, y;
};
struct double4 {
    double x, y, z, w;
};
#endif

#ifdef __CUDA_ARCH__
#define FM_CONST static __constant__
#else
#define FM_CONST static const
#endif

namespace fmm2d {
namespace fm {

constexpr int LOG_BITS = 8;
constexpr int LOG_N = 1 << LOG_BITS;      // 256 intervals of [1,2)
constexpr int ATAN_BITS = 8;
constexpr int ATAN_N = 1 << ATAN_BITS;    // c = j/256, j = 0..256 (257 rows, padded to 264)

// table rows: log {ic_j, L_j}; atan {theta_hi_j, theta_lo_j}
struct Tables {
    double2 lg[LOG_N];
    double2 at[ATAN_N + 8];
};

// The near field's own tables (k_near, k_near_wide): the P2P loop is bound by shared-memory
// wavefronts -- 32 lanes reading random 16-byte rows collide in the 8 bank groups (ncu: 9.4
// wavefronts per LDS.128 against 4 ideal, the shared pipe 73 % busy) -- so
//  - the atan table holds ONE double per row (atan(j/256) rounded; the low part is dropped, an
//    absolute error < 2^-54): 8-byte rows, half the bytes per lookup;
//  - both tables can be REPLICATED: copy k = lane mod R of row j sits at [j R + k], so each copy
//    owns its own banks and only the lanes sharing a copy can collide.
#ifndef FMM2D_NEAR_RL
#define FMM2D_NEAR_RL 1            // copies of the log table (power of two)
#endif
#ifndef FMM2D_NEAR_RA
#define FMM2D_NEAR_RA 1            // copies of the atan table (power of two)
#endif
constexpr int NRL = FMM2D_NEAR_RL, NRA = FMM2D_NEAR_RA;
constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v >> 1); }
constexpr int LRL = ilog2c(NRL), LRA = ilog2c(NRA);
static_assert((1 << LRL) == NRL && (1 << LRA) == NRA, "replication factors are powers of two");
struct TablesN {
    double2 lg[LOG_N * NRL];                       // {ic_j (2 ic_j for f >= 1.5), L_j}
    double th[((ATAN_N + 1) * NRA + 1) & ~1];      // atan(j/256), j = 0..256
    double2 oct[4];                                // {base, s} by 2 swap + (dx < 0)
};
struct AllTables {
    Tables t;
    TablesN n;
};

// [0..3] log1p series -1/6, 1/5, -1/4, 1/3, [4] -1/2, [5] unused, [6..7] atan series 1/5, -1/3,
// [8] ln2 * 2^-20 (exact scaling of the double nearest ln 2), [9] unused, [10] pi/2, [11] unused,
// [12] pi, [13] unused, [14] 2^52 + 1023 * 2^20 (exponent extraction), [15] 1.5 * 2^44
// (rounding to a multiple of 1/256), [16..17] asin series 3/40, 1/6, [18] 1.5 * 2^52 (rounding
// to an integer), [19] 3/8, [20] 1/2
FM_CONST double kC[21] = {
    -1.0 / 6.0, 1.0 / 5.0, -1.0 / 4.0, 1.0 / 3.0, -0.5, 0.0,
    1.0 / 5.0, -1.0 / 3.0,
    6.931471805599453094e-01 / 1048576.0, 0.0,
    1.5707963267948966192e+00, 0.0,
    3.141592653589793116e+00, 0.0,
    4503599627370496.0 + 1023.0 * 1048576.0, 1.5 * 17592186044416.0};

FM_HD int64_t as_bits(double x)
{
#ifdef __CUDA_ARCH__
    return __double_as_longlong(x);
#else
    int64_t b;
    memcpy(&b, &x, 8);
    return b;
#endif
}
FM_HD double from_bits(int64_t b)
{
#ifdef __CUDA_ARCH__
    return __longlong_as_double(b);
#else
    double x;
    memcpy(&x, &b, 8);
    return x;
#endif
}
FM_HD double fma_(double a, double b, double c)
{
#ifdef __CUDA_ARCH__
    return fma(a, b, c);
#else
    return __builtin_fma(a, b, c);
#endif
}

FM_HD int hi_word(double x) { return (int)(as_bits(x) >> 32); }
FM_HD int lo_word(double x) { return (int)as_bits(x); }
FM_HD double make_double(int hi, int lo)
{
#ifdef __CUDA_ARCH__
    return __hiloint2double(hi, lo);
#else
    return from_bits((int64_t)(((uint64_t)(uint32_t)hi << 32) | (uint32_t)lo));
#endif
}

// coarse reciprocal (~2^-22 relative) and the refined one (~1 ulp)
FM_HD double rcp_approx(double x)
{
#ifdef __CUDA_ARCH__
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    return r;
#else
#ifdef FM_HOST_RCP_PERTURB             // worst case of the device estimate (2^-22 relative), for the accuracy test
    return (double)(float)(1.0 / x) * (1.0 + FM_HOST_RCP_PERTURB * 2.384185791015625e-07);
#else
    return (double)(float)(1.0 / x);      // host stand-in with a comparable error
#endif
#endif
}
FM_HD double rcp(double x)
{
    double r = rcp_approx(x);
    double e = fma_(-x, r, 1.0);
    return fma_(r, fma_(e, e, e), r);      // cubic step: err^3
}

// Operand forms matter on B200: an FP64 instruction with three distinct register operands
// occupies the FP64 pipe for 3 cycles instead of 2 (register-file bandwidth; tools/fp64_mix.cu:
// 0.66 against 0.91 of the nominal rate), so the near-field routines keep their constants out of
// the register file -- literal constants (uniform registers / immediates) instead of loads from
// __constant__ arrays, the small high-order coefficients as SHORT immediates (high word only:
// 1/5 enters log1p and atan below 2^-40, so 20 mantissa bits are plenty) -- and are written so
// that no FMA needs three different registers (q = p u, then q u + u).
constexpr double K_FIFTH_SHORT = 0.20000004768371582;        // 0x3FC9999A00000000
constexpr double K_THIRD = 1.0 / 3.0;
constexpr double K_LN2_20 = 6.931471805599453094e-01 / 1048576.0;
constexpr double K_MAGIC_E = 4503599627370496.0 + 1023.0 * 1048576.0;
constexpr double K_MAGIC_Q = 1.5 * 17592186044416.0;

// The reduction shared by log_pos / log_pos5 (header comment): j = the top 8 mantissa bits,
// hw = (exponent + [f >= 1.5]) << 20 = E' << 20, u = r2 (ic_j 2^-E') - 1 = f ic_j - 1 exactly
// as before (power-of-two scalings), e20 = (E' - 1023) 2^20.  Normal r2 < 2^1021.
// LR: log2 of the row stride in rows (the near field's replicated table, TablesN: row j of copy k
// at [j 2^LR + k], tab pointing at copy k's row 0).
template <int LR = 0>
FM_HD void log_reduce(double r2, const double2* __restrict__ tab, double& u, double& e20, double& Lj)
{
    const int hi = hi_word(r2);
    // row j = the top LOG_BITS mantissa bits, as a byte offset (16-byte rows)
    const uint32_t jb = ((uint32_t)hi >> (20 - LOG_BITS - 4 - LR)) & (uint32_t)((LOG_N - 1) << (4 + LR));
    const int hw = (int)(((uint32_t)hi + 0x00080000u) & 0xFFF00000u);
    const double2 T = *reinterpret_cast<const double2*>(reinterpret_cast<const char*>(tab) + jb);
    const double ics = make_double(hi_word(T.x) - hw + 0x3FF00000, lo_word(T.x));
    u = fma_(r2, ics, -1.0);
    e20 = make_double(0x43300000, hw) - K_MAGIC_E;
    Lj = T.y;
}

// log(r2) with a degree-5 series (|u| < 2^-9: truncation < 2^-54 / 6 absolute), used
// by the near-field kernel where only the absolute error of each term matters.  No
// special case for r2 == 0 (coincident distinct points): there arg_t gives NaN, so
// the pair's Phi and Phi' are non-finite anyway.
template <int LR = 0>
FM_HD double log_pos5(double r2, const double2* __restrict__ tab)
{
    double u, e20, Lj;
    log_reduce<LR>(r2, tab, u, e20, Lj);
    // log1p(u) = u - u^2/2 + u^3/3 - u^4/4 + u^5/5 = u + u (u p(u))
    double p = fma_(u, K_FIFTH_SHORT, -0.25);
    p = fma_(p, u, K_THIRD);
    p = fma_(p, u, -0.5);
    const double q = p * u;
    const double lp = fma_(q, u, u);
    const double r = fma_(e20, K_LN2_20, Lj + lp);
    return r;                    // r2 == 0 gives a finite value; Arg(0) is NaN (see k_near)
}

// log(r2) for r2 > 0 normal; -inf for r2 == 0.
FM_HD double log_pos(double r2, const double2* __restrict__ tab)
{
    double u, e20, Lj;
    log_reduce(r2, tab, u, e20, Lj);
    // log1p(u) = u - u^2/2 + u^3/3 - u^4/4 + u^5/5 - u^6/6   (|u| < 2^-9: trunc. 2^-66)
    double p = fma_(kC[0], u, kC[1]);
    p = fma_(p, u, kC[2]);
    p = fma_(p, u, kC[3]);
    p = fma_(p, u, kC[4]);
    const double lp = fma_(p, u * u, u);
    const double r = fma_(e20, kC[8], Lj + lp);       // e ln2 in one rounding (|e| ln2 error < 0.3 ulp)
    return (r2 == 0.0) ? -HUGE_VAL : r;
}

// a = atan(mn/mx) in [0, pi/4] placed in its octant: (swap, neg) -> a, pi/2 - a, pi - a,
// pi/2 + a == base +- a (one rounding), then the sign bit (dy = +0 keeps 0 / pi).
FM_HD double octant_fix(double a, bool swap, bool neg, int64_t signbit)
{
    const double base = swap ? kC[10] : (neg ? kC[12] : 0.0);
    const double sa = from_bits(as_bits(a) ^ ((int64_t)(swap != neg) << 63));
    const double res = base + sa;                           // >= 0
    return from_bits(as_bits(res) | signbit);
}

// principal Arg(dx + i dy) = atan2(dy, dx) in (-pi, pi]; dy = +0 gives 0 or pi.
FM_HD double arg(double dx, double dy, const double2* __restrict__ tab)
{
    const int hx = (int)(as_bits(dx) >> 32), hy = (int)(as_bits(dy) >> 32);   // sign tests on the high words
    const bool swap = fabs(dy) > fabs(dx);    // one DSETP with |.| operand modifiers
    // select the signed values; |.| is applied as an operand modifier by the consumers
    const double mns = swap ? dx : dy;
    const double mxs = swap ? dy : dx;
    const double mn = fabs(mns), mx = fabs(mxs);
    const double q0 = fabs(mns * rcp_approx(mxs));
    // round q0 to a multiple of 2^-8 with the 1.5*2^44 magic number; j = the rounded q0 * 256
    const double y = q0 + kC[15];
    const int jr = (int)as_bits(y) & (2 * ATAN_N - 1);   // 0..256 (any value for mx == 0)
    const int j = jr < ATAN_N ? jr : ATAN_N;
    const double c = y - kC[15];
    const double num = fma_(-c, mx, mn);
    const double den = fma_(c, mn, mx);
    const double t = num * rcp(den);
    // atan(t) = t - t^3/3 + t^5/5   (|t| < 2^-8: truncation 2^-56 relative)
    const double t2 = t * t;
    const double p = fma_(kC[6], t2, kC[7]);
    const double at = fma_(p * t2, t, t);
    const double2 T = tab[j];
    const double a = T.x + (at + T.y);                    // atan(mn/mx) in [0, pi/4]
    return octant_fix(a, swap, hx < 0, (int64_t)(uint32_t)(hy & (int)0x80000000u) << 32);
}

// arg with the octant placement as ONE FMA: rows OCT_ROW + 2 swap + neg of the table hold
// {base, s} = {0, 1}, {pi, -1}, {pi/2, -1}, {pi/2, 1}, and res = s a + base (s a is exact, so
// this is base +- a in one rounding: the same result as arg() bit for bit).  The table index
// is the low word of q0 + 1.5 2^44 itself (no mask: the unsigned clamp covers NaN).
constexpr int OCT_ROW = ATAN_N + 4;
FM_HD double arg_t(double dx, double dy, const double2* __restrict__ tab)
{
    const int hx = hi_word(dx), hy = hi_word(dy);
    const bool swap = fabs(dy) > fabs(dx);
    const double mns = swap ? dx : dy;
    const double mxs = swap ? dy : dx;
    const double mn = fabs(mns), mx = fabs(mxs);
    const double q0 = fabs(mns * rcp_approx(mxs));
    const double y = q0 + kC[15];
    const uint32_t jr = (uint32_t)lo_word(y);
    const int j = (int)(jr < (uint32_t)ATAN_N ? jr : (uint32_t)ATAN_N);
    const double c = y - kC[15];
    const double num = fma_(-c, mx, mn);
    const double den = fma_(c, mn, mx);
    const double t = num * rcp(den);
    const double t2 = t * t;
    const double p = fma_(kC[6], t2, kC[7]);
    const double at = fma_(p * t2, t, t);
    const double2 T = tab[j];
    const double a = T.x + (at + T.y);
    const bool neg = hx < 0;
    const double2 O = (tab + OCT_ROW)[2 * (int)swap + (int)neg];
    const double res = fma_(a, O.y, O.x);
    return from_bits(as_bits(res) | ((int64_t)(uint32_t)(hy & (int)0x80000000u) << 32));
}

// The near field's Arg (k_near): as arg_t, with the quotient t = num/den from the COARSE
// reciprocal and one correction (t0 = num r0, e = 1 - den r0, t = t0 + t0 e: relative error
// e^2 < 2^-44 of |t| < 2^-8, i.e. < 2^-52 ABSOLUTE -- one FP64 operation fewer than the refined
// reciprocal, e and t0 independent, no FMA with three different registers).  Each term m Arg enters Phi with its absolute
// error, like the log term (log_pos5); tests/test_fastmath.py bounds it in units of 2^-52.
// The table is TablesN's single-double atan(j/256) (no low part).
FM_HD double arg_n(double dx, double dy, const double* __restrict__ th, const double2* __restrict__ oct)
{
    const int hx = hi_word(dx), hy = hi_word(dy);
    const bool swap = fabs(dy) > fabs(dx);
    const double mns = swap ? dx : dy;
    const double mxs = swap ? dy : dx;
    const double mn = fabs(mns), mx = fabs(mxs);
    const double q0 = fabs(mns * rcp_approx(mxs));
    const double y = q0 + K_MAGIC_Q;
    const uint32_t jr = (uint32_t)lo_word(y);
    const int j = (int)(jr < (uint32_t)ATAN_N ? jr : (uint32_t)ATAN_N);
    const double c = y - K_MAGIC_Q;
    const double num = fma_(-c, mx, mn);
    const double den = fma_(c, mn, mx);
    // t = num/den = t0 (1 + e + e^2 + ...), t0 = num r0, e = 1 - den r0 (|e| < 2^-22): t0 + t0 e
    const double r0 = rcp_approx(den);
    const double e = fma_(-den, r0, 1.0);
    const double t0 = num * r0;
    const double t = fma_(t0, e, t0);
    const double t2 = t * t;
    const double p = fma_(t2, K_FIFTH_SHORT, -K_THIRD);
    const double at = fma_(p * t2, t, t);
    const double a = th[j * NRA] + at;                        // th: the lane's copy (TablesN)
    const bool neg = hx < 0;
    const double2 O = oct[2 * (int)swap + (int)neg];
    const double res = fma_(a, O.y, O.x);
    return from_bits(as_bits(res) | ((int64_t)(uint32_t)(hy & (int)0x80000000u) << 32));
}

// Arg(dz) and Arg(-dz), the latter of the componentwise difference z_j - z_i (zeros stay
// +0, DESIGN R2): the same reduced angle, mirrored octant (-dx < 0 iff dx > 0) and sign
// (-dy < 0 iff dy > 0).  Used by the symmetric near-field kernel.
FM_HD void arg_pair(double dx, double dy, const double2* __restrict__ tab, double& th, double& thn)
{
    const int64_t bx = as_bits(dx), by = as_bits(dy);
    const bool swap = fabs(dy) > fabs(dx);
    const double mns = swap ? dx : dy;
    const double mxs = swap ? dy : dx;
    const double mn = fabs(mns), mx = fabs(mxs);
    const double q0 = fabs(mns * rcp_approx(mxs));
    const double y = q0 + kC[15];
    const int jr = (int)as_bits(y) & (2 * ATAN_N - 1);
    const int j = jr < ATAN_N ? jr : ATAN_N;
    const double c = y - kC[15];
    const double num = fma_(-c, mx, mn);
    const double den = fma_(c, mn, mx);
    const double t = num * rcp(den);
    const double t2 = t * t;
    const double p = fma_(kC[6], t2, kC[7]);
    const double at = fma_(p * t2, t, t);
    const double2 T = tab[j];
    const double a = T.x + (at + T.y);
    th = octant_fix(a, swap, bx < 0, by & (int64_t)0x8000000000000000ull);
    thn = octant_fix(a, swap, bx > 0, by > 0 ? (int64_t)0x8000000000000000ull : 0);
}

// host: fill the tables (long double evaluation, rounded once to double)
static inline void make_tables(Tables* T)
{
    for (int j = 0; j < LOG_N; ++j) {
        long double c = 1.0L + ((long double)j + 0.5L) / (long double)LOG_N;
        double ic = (double)(1.0L / c);
        T->lg[j].x = (j >= LOG_N / 2 ? 2.0 : 1.0) * ic;        // 2 ic_j for f >= 1.5 (log_reduce)
        // -log(ic) for f in [1, 1.5); -log(2 ic) = log(f/2) offset for f in [1.5, 2)
        T->lg[j].y = (double)(-logl((long double)ic * (j >= LOG_N / 2 ? 2.0L : 1.0L)));
    }
    for (int j = 0; j < ATAN_N + 8; ++j) {
        long double th = atanl((long double)(j <= ATAN_N ? j : ATAN_N) / (long double)ATAN_N);
        double hi = (double)th;
        T->at[j].x = hi;
        T->at[j].y = (double)(th - (long double)hi);
    }
    // octant rows {base, s} for arg_t / arg_n (never reached by the clamped index j <= ATAN_N),
    // indexed by 2 swap + (dx < 0)
    T->at[OCT_ROW + 0].x = 0.0;
    T->at[OCT_ROW + 0].y = 1.0;
    T->at[OCT_ROW + 1].x = kC[12];
    T->at[OCT_ROW + 1].y = -1.0;
    T->at[OCT_ROW + 2].x = kC[10];
    T->at[OCT_ROW + 2].y = -1.0;
    T->at[OCT_ROW + 3].x = kC[10];
    T->at[OCT_ROW + 3].y = 1.0;
}

static inline void make_tables_n(TablesN* N)
{
    static Tables T;
    make_tables(&T);
    for (int j = 0; j < LOG_N; ++j)
        for (int k = 0; k < NRL; ++k) N->lg[j * NRL + k] = T.lg[j];
    for (size_t i = 0; i < sizeof(N->th) / sizeof(double); ++i) N->th[i] = 0.0;
    for (int j = 0; j <= ATAN_N; ++j)
        for (int k = 0; k < NRA; ++k) N->th[j * NRA + k] = (double)atanl((long double)j / (long double)ATAN_N);
    for (int i = 0; i < 4; ++i) N->oct[i] = T.at[OCT_ROW + i];
}

}  // namespace fm
}  // namespace fmm2d
