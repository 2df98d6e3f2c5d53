"""Mutation check of the oracle's pins: apply plausible mistakes (a dropped term,
a wrong sign or index, a transposed operand) to a COPY of oracle_fmm2d.cpp, build
it to a temporary library, and confirm that the CPU test suite fails for each.

    python tools/oracle_mutation_check.py
"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = open(os.path.join(ROOT, "oracle", "oracle_fmm2d.cpp")).read()

MUTATIONS = [
    ("M2L drops (-1)^k", "t += ((k & 1) ? -1.0 : 1.0) * C[l + k - 1][k - 1]", "t += C[l + k - 1][k - 1]"),
    ("M2M binomial index", "C[l - 1][k - 1]", "C[l][k - 1]"),
    ("tree child offset", "oc[4 * b + 1] = s + ceil_half(h0);", "oc[4 * b + 1] = s + h0 / 2;"),
    ("criterion r/R swapped", "return (d > 0.0) && (R + theta * r <= theta * d);",
     "return (d > 0.0) && (r + theta * R <= theta * d);"),
    ("disc radius uses x twice", "double dx = P->x[i] - cx, dy = P->y[i] - cy;",
     "double dx = P->x[i] - cx, dy = P->x[i] - cy;"),
    ("L2L shift sign", "cplx h(P->cx[l][c] - P->cx[l - 1][b], P->cy[l][c] - P->cy[l - 1][b]);",
     "cplx h(P->cx[l - 1][b] - P->cx[l][c], P->cy[l - 1][b] - P->cy[l][c]);"),
    ("M2L log of c_s - c_t", "cplx s0 = a[0] * std::log(tc);", "cplx s0 = a[0] * std::log(-tc);"),
    ("P2M drops 1/k", "a[k] -= ms[j] * wk / (double)k;", "a[k] -= ms[j] * wk;"),
    ("y-split sorts by x", "std::sort(seg + h0, seg + nb, byy);", "std::sort(seg + h0, seg + nb, byx);"),
    ("P2P keeps self pair", "if (j == i) continue;                              /* j != i */", ""),
    ("L2P derivative index", "ds += (double)l * b[l] * wlm1;", "ds += (double)(l - 1) * b[l] * wlm1;"),
    ("M2L from level 2 (R15)", "    for (int l = 1; l <= L; ++l) {\n#pragma omp parallel for schedule(dynamic, 64)\n        for (int64_t t = 0;",
     "    for (int l = 2; l <= L; ++l) {\n#pragma omp parallel for schedule(dynamic, 64)\n        for (int64_t t = 0;"),
    ("lists from level 2", "    for (int l = 1; l <= P->L; ++l) {\n        int64_t nb = nboxes(l);\n        P->strong[l]",
     "    for (int l = 1; l <= P->L; ++l) {\n        if (l == 1) { P->strong[1].assign(4, {}); P->weak[1].assign(4, {});"
     " for (uint32_t b = 0; b < 4; ++b) for (uint32_t c = 0; c < 4; ++c) P->strong[1][b].push_back(c); continue; }\n"
     "        int64_t nb = nboxes(l);\n        P->strong[l]"),
    # O7 r/R exchange
    ("P2L drops the minus sign", "b[l] -= ms[j] * ivl / (double)l;", "b[l] += ms[j] * ivl / (double)l;"),
    ("exchanged criterion unswapped", "return (r < R) && (d > 0.0) && (r + theta * R <= theta * d);",
     "return (r < R) && (d > 0.0) && (R + theta * r <= theta * d);"),
    ("P2L into the larger box", "else if (rr[t] < rr[s]) P->p2l_in[t].push_back(s);",
     "else if (rr[t] > rr[s]) P->p2l_in[t].push_back(s);"),
    # O8 parent merge
    ("merge without the parent criterion", "if (P->pm && l >= 2 && ws[0] && ws[1] && ws[2] && ws[3] &&\n"
     "                    oracle_well_separated(", "if (P->pm && l >= 2 && ws[0] && ws[1] && ws[2] &&\n"
     "                    oracle_well_separated("),
    ("cross M2L from the wrong level", "m2l(P->mpole[l - 1].data() + (int64_t)q * P1, P->cx[l - 1][q], P->cy[l - 1][q],",
     "m2l(P->mpole[l - 1].data() + (int64_t)q * P1, P->cx[l][q], P->cy[l][q],"),
    # O9 midpoint tree
    ("midpoint key y-high", "b = 4 * b + 2 * ((ix >> j) & 1) + ((iy >> j) & 1);",
     "b = 4 * b + 2 * ((iy >> j) & 1) + ((ix >> j) & 1);"),
    ("midpoint cell floor -> round", "int64_t ix = (int64_t)std::floor((P->x[i] - x0) * S);",
     "int64_t ix = (int64_t)std::round((P->x[i] - x0) * S);"),
]


def main():
    missed = 0
    with tempfile.TemporaryDirectory() as td:
        for name, a, b in MUTATIONS:
            assert a in SRC, name
            cpp = os.path.join(td, "m.cpp")
            so = os.path.join(td, "m.so")
            open(cpp, "w").write(SRC.replace(a, b))
            subprocess.check_call(["g++", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-o", so, cpp])
            env = dict(os.environ, FMM2D_ORACLE_LIB=so)
            r = subprocess.run([sys.executable, "-m", "pytest", "tests", "-x", "-q", "-m", "not gpu",
                                "-k", "oracle"], cwd=ROOT, env=env, capture_output=True, text=True)
            ok = r.returncode != 0
            missed += not ok
            print(f"{'CAUGHT' if ok else 'MISSED'}  {name}")
    sys.exit(1 if missed else 0)


if __name__ == "__main__":
    main()
