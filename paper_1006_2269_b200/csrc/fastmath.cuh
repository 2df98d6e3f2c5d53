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
//            the ln 2, so log r2 ~ 0 does not cancel), |u| < 2^-9, degree-6 series;
//   Arg    = octant reduction a = atan(mn/mx), mn <= mx; c = mn/mx rounded to a
//            multiple of 1/256 (22-bit estimate + magic-number rounding, no int<->fp
//            conversion); atan(mn/mx) = atan(c) + atan(t), t = (mn - c mx)/(mx + c mn),
//            |t| < 2^-8, degree-5 series; octant / sign fixes by selects and a sign-bit OR;
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

// [0..3] log1p series -1/6, 1/5, -1/4, 1/3, [4] -1/2, [5] unused, [6..7] atan series 1/5, -1/3,
// [8] ln2 * 2^-32 (exact scaling of the double nearest ln 2), [9] unused, [10] pi/2, [11] unused,
// [12] pi, [13] unused, [14] 2^52 + 1023 * 2^32 (exponent extraction), [15] 1.5 * 2^44
// (rounding to a multiple of 1/256), [16..17] asin series 3/40, 1/6, [18] 1.5 * 2^52 (rounding
// to an integer), [19] 3/8, [20] 1/2
FM_CONST double kC[21] = {
    -1.0 / 6.0, 1.0 / 5.0, -1.0 / 4.0, 1.0 / 3.0, -0.5, 0.0,
    1.0 / 5.0, -1.0 / 3.0,
    6.931471805599453094e-01 / 4294967296.0, 0.0,
    1.5707963267948966192e+00, 0.0,
    3.141592653589793116e+00, 0.0,
    4503599627370496.0 + 1023.0 * 4294967296.0, 1.5 * 17592186044416.0};

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

// coarse reciprocal (~2^-22 relative) and the refined one (~1 ulp)
FM_HD double rcp_approx(double x)
{
#ifdef __CUDA_ARCH__
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    return r;
#else
    return (double)(float)(1.0 / x);      // host stand-in with a comparable error
#endif
}
FM_HD double rcp(double x)
{
    double r = rcp_approx(x);
    double e = fma_(-x, r, 1.0);
    return fma_(r, fma_(e, e, e), r);      // cubic step: err^3
}

// log(r2) with a degree-5 series (|u| < 2^-9: truncation < 2^-54 / 6 absolute), used
// by the near-field kernel where only the absolute error of each term matters.  No
// special case for r2 == 0 (coincident distinct points): there arg_t gives NaN, so
// the pair's Phi and Phi' are non-finite anyway.
FM_HD double log_pos5(double r2, const double2* __restrict__ tab)
{
    const int64_t b = as_bits(r2);
    const int hi = (int)(b >> 32);
    const int j = (hi >> (20 - LOG_BITS)) & (LOG_N - 1);
    const int eb = (hi >> 20) + (j >> (LOG_BITS - 1));
    const double e32 = from_bits((int64_t)(0x43300000 | eb) << 32) - kC[14];
    const double f = from_bits((b & 0x000FFFFFFFFFFFFFll) | 0x3FF0000000000000ll);
    const double2 T = tab[j];
    const double u = fma_(f, T.x, -1.0);
    // log1p(u) = u - u^2/2 + u^3/3 - u^4/4 + u^5/5
    double p = fma_(kC[1], u, kC[2]);
    p = fma_(p, u, kC[3]);
    p = fma_(p, u, kC[4]);
    const double lp = fma_(p, u * u, u);
    const double r = fma_(e32, kC[8], T.y + lp);
    return r;                    // r2 == 0 gives a finite value; Arg(0) is NaN (see k_near)
}

// log(r2) for r2 > 0 normal; -inf for r2 == 0.
FM_HD double log_pos(double r2, const double2* __restrict__ tab)
{
    const int64_t b = as_bits(r2);
    const int hi = (int)(b >> 32);
    const int j = (hi >> (20 - LOG_BITS)) & (LOG_N - 1);
    // exponent (+1 when f >= 1.5) as a double scaled by 2^32, without a conversion:
    // bits 0x43300000:E:00000000 = 2^52 + E 2^32
    const int eb = (hi >> 20) + (j >> (LOG_BITS - 1));
    const double e32 = from_bits((int64_t)(0x43300000 | eb) << 32) - kC[14];
    const double f = from_bits((b & 0x000FFFFFFFFFFFFFll) | 0x3FF0000000000000ll);
    const double2 T = tab[j];
    const double u = fma_(f, T.x, -1.0);
    // log1p(u) = u - u^2/2 + u^3/3 - u^4/4 + u^5/5 - u^6/6   (|u| < 2^-9: trunc. 2^-66)
    double p = fma_(kC[0], u, kC[1]);
    p = fma_(p, u, kC[2]);
    p = fma_(p, u, kC[3]);
    p = fma_(p, u, kC[4]);
    const double lp = fma_(p, u * u, u);
    const double r = fma_(e32, kC[8], T.y + lp);      // e ln2 in one rounding (|e| ln2 error < 0.3 ulp)
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

// arg with the octant base read from the table (rows OCT_ROW, OCT_ROW+1 = {0, pi},
// {pi/2, pi/2} indexed by 2 swap + neg) instead of selects; same result bit for bit.
constexpr int OCT_ROW = ATAN_N + 4;
FM_HD double arg_t(double dx, double dy, const double2* __restrict__ tab)
{
    const int hx = (int)(as_bits(dx) >> 32), hy = (int)(as_bits(dy) >> 32);
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
    const bool neg = hx < 0;
    const double base = reinterpret_cast<const double*>(tab + OCT_ROW)[2 * (int)swap + (int)neg];
    const double sa = from_bits(as_bits(a) ^ ((int64_t)(swap != neg) << 63));
    const double res = base + sa;
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
        T->lg[j].x = ic;
        // -log(ic) for f in [1, 1.5); -log(2 ic) = log(f/2) offset for f in [1.5, 2)
        T->lg[j].y = (double)(-logl((long double)ic * (j >= LOG_N / 2 ? 2.0L : 1.0L)));
    }
    for (int j = 0; j < ATAN_N + 8; ++j) {
        long double th = atanl((long double)(j <= ATAN_N ? j : ATAN_N) / (long double)ATAN_N);
        double hi = (double)th;
        T->at[j].x = hi;
        T->at[j].y = (double)(th - (long double)hi);
    }
    // octant bases for arg_t (rows never reached by the clamped index j <= ATAN_N)
    T->at[OCT_ROW].x = 0.0;
    T->at[OCT_ROW].y = kC[12];
    T->at[OCT_ROW + 1].x = kC[10];
    T->at[OCT_ROW + 1].y = kC[10];
}

}  // namespace fm
}  // namespace fmm2d
