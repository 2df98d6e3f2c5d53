// Host build of paper_1006_2269_b200/csrc/fastmath.cuh against long double references.
// Prints JSON: max error in ulps of log r2 / 2 and of Arg over random and edge inputs.
//   g++ -O2 -ffp-contract=off -o build/test_fastmath tools/test_fastmath.cpp
#include <cmath>
#include <cstdio>
#include <random>
#include "../paper_1006_2269_b200/csrc/fastmath.cuh"
using namespace fmm2d::fm;

static double ulp_err(double got, long double ref)
{
    double r = (double)ref;
    double u = std::nextafter(std::fabs(r), INFINITY) - std::fabs(r);
    if (r == 0.0) u = 4.9e-324;
    return (double)(fabsl((long double)got - ref) / (long double)u);
}

int main()
{
    Tables T;
    make_tables(&T);
    static TablesN N;
    make_tables_n(&N);
    std::mt19937_64 g(12345);
    std::uniform_real_distribution<double> U(-1.0, 1.0);
    std::uniform_real_distribution<double> E(-60.0, 60.0);
    double mlog = 0, marg = 0, mabs_log = 0, margn = 0;
    double mlog5_abs = 0, margn_abs = 0, margn_small_rel = 0;
    long pair_mismatch = 0;
    long n = 0;
    for (long k = 0; k < 4000000; ++k) {
        double s = std::ldexp(1.0, (int)E(g));
        double dx = U(g) * s, dy = U(g) * s;
        if (k % 7 == 0) dy = 0.0;                 // on the real axis
        if (k % 11 == 0) dx = 0.0;                // on the imaginary axis
        if (k % 13 == 0) dy = dx;                 // diagonal
        if (dx == 0.0 && dy == 0.0) continue;
        double r2 = dx * dx + dy * dy;
        double lg = 0.5 * log_pos(r2, T.lg);
        long double rl = 0.5L * logl((long double)r2);
        double a = arg(dx, dy, T.at);
        long double ra = atan2l((long double)dy, (long double)dx);
        // log: ulps of the result (abs error reported too, for |log| ~ 0)
        double el = ulp_err(lg, rl);
        if (fabsl(rl) > 1e-3L) mlog = std::fmax(mlog, el);
        mabs_log = std::fmax(mabs_log, (double)fabsl((long double)lg - rl));
        marg = std::fmax(marg, ulp_err(a, ra));
        // Arg of the componentwise reverse difference (zeros stay +0) from arg_pair
        double th, thn;
        arg_pair(dx, dy, T.at, th, thn);
        double dxn = (dx == 0.0) ? 0.0 : -dx, dyn = (dy == 0.0) ? 0.0 : -dy;
        long double rn = atan2l((long double)dyn, (long double)dxn);
        if (th != a) pair_mismatch++;
        if (arg_t(dx, dy, T.at) != a) pair_mismatch++;       // table-based octant: bit-identical
        margn = std::fmax(margn, ulp_err(thn, rn));
        // near-field log: degree-5 series, absolute error in units of 2^-52 max(1, |log|)
        double lg5 = 0.5 * log_pos5<LRL>(r2, N.lg);
        double sc = std::fmax(1.0, (double)fabsl(rl)) * 2.220446049250313e-16;
        mlog5_abs = std::fmax(mlog5_abs, (double)(fabsl((long double)lg5 - rl) / sc));
        // near-field Arg (arg_n: coarse reciprocal + one residual correction): absolute error in
        // units of 2^-52 max(1, |Arg|), and the relative error where |Arg| is small
        double an = arg_n(dx, dy, N.th, N.oct);
        double sa = std::fmax(1.0, (double)fabsl(ra)) * 2.220446049250313e-16;
        margn_abs = std::fmax(margn_abs, (double)(fabsl((long double)an - ra) / sa));
        if (ra != 0.0L) margn_small_rel = std::fmax(margn_small_rel, (double)(fabsl(((long double)an - ra) / ra)));
        if ((an < 0) != (a < 0) || (an == 0.0) != (a == 0.0)) pair_mismatch++;
        ++n;
    }
    double zero = log_pos(0.0, T.lg);
    printf("{\"log5_max_abs_eps\": %.3f, \"argn_max_abs_eps\": %.3f, \"argn_max_rel\": %.3e, ", mlog5_abs, margn_abs, margn_small_rel);
    printf("\"n\": %ld, \"log_max_ulp\": %.3f, \"log_max_abs\": %.3e, \"arg_max_ulp\": %.3f, \"argneg_max_ulp\": %.3f, "
           "\"pair_mismatch\": %ld, \"log0_is_neg_inf\": %d, \"arg_pi\": %d, \"arg_zero\": %d}\n",
           n, mlog, mabs_log, marg, margn, pair_mismatch, (int)(std::isinf(zero) && zero < 0),
           (int)(arg(-1.0, 0.0, T.at) == M_PI), (int)(arg(2.0, 0.0, T.at) == 0.0));
    return 0;
}
