# k_near variants of the last round-2 session (near.cu / fastmath.cuh defines; C5 near ms by r02_var.sh, base 91.5 at
# 128 threads / 84.6 at 96): -DFMM2D_NEAR_RL=2 -DFMM2D_NEAR_RA=2 (replicated tables) 93.1; RL=2 RA=4 MINB=7 94.2;
# RL=4 RA=4 MINB=6 94.6; -DFMM2D_NEAR_MINB=7 / 6 / 9: 91.8 / 94.4 / 93.6; -DFMM2D_NEAR_UNROLL=2: 91.8;
# FMM2D_NEAR_THREADS=128 / 64 (environment): 91.5 / 93.5 against 84.6 for the picked 96.
# (Removed from the source after measuring: the two targets' chains written stage by stage, the octant sign by
#  XOR + DADD, the swap decision on the high words -- DESIGN.md 6.4.)
bash scripts/build_variants.sh near "-DFMM2D_NEAR_RL=2 -DFMM2D_NEAR_RA=2" "-DFMM2D_NEAR_MINB=7" "-DFMM2D_NEAR_UNROLL=2"
bash scripts/r02_var.sh build/var_near__DFMM2D_NEAR_RL_2__DFMM2D_NEAR_RA_2/libfmm2d.so build/var_near__DFMM2D_NEAR_MINB_7/libfmm2d.so build/var_near__DFMM2D_NEAR_UNROLL_2/libfmm2d.so
FMM2D_NEAR_THREADS=128 bash scripts/r02_var.sh
