# M2L pair-body variants of the last round-2 session (expansions.cu defines; C5 phase times by r02_var.sh):
#   -DFMM2D_M2L_LB=0        contraction one output coefficient at a time          19.26 ms
#   -DFMM2D_M2L_LB=18       k-outermost over all 36 accumulators (default)         17.40 ms
#   -DFMM2D_M2L_PREFETCH=0  without the next-index prefetch (LB=18)                17.42 -> 16.54 ms with it
#   -DFMM2D_M2L_RCP=0       IEEE division for 1/r2                                 16.53 -> 15.84 ms with the Newton step
#   -DFMM2D_M2L_POW2=1|2    powers by doubling, pre- / post-scaling                16.58 / 17.85 ms
bash scripts/build_variants.sh expansions "-DFMM2D_M2L_LB=0" "-DFMM2D_M2L_PREFETCH=0" "-DFMM2D_M2L_RCP=0" "-DFMM2D_M2L_POW2=1" "-DFMM2D_M2L_POW2=2"
bash scripts/r02_var.sh build/var_expansions__DFMM2D_M2L_LB_0/libfmm2d.so build/var_expansions__DFMM2D_M2L_PREFETCH_0/libfmm2d.so build/var_expansions__DFMM2D_M2L_RCP_0/libfmm2d.so build/var_expansions__DFMM2D_M2L_POW2_1/libfmm2d.so build/var_expansions__DFMM2D_M2L_POW2_2/libfmm2d.so
