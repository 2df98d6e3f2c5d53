"""B200-native (sm_100a) evaluation pass of the asymmetric adaptive 2D FMM of
S. Engblom, "On well-separated sets and fast multipole methods" (arXiv 1006.2269).

The compute path is libfmm2d.so (CUDA kernels behind the C ABI in include/fmm2d.h);
this package is its ctypes binding.  See DESIGN.md.
"""
from .fmm2d import (Fmm2d, FmmError, LoopbackShards, lib, LIB_PATH, PMAX, SYMBOLS,  # noqa: F401
                    nccl_unique_id, partition_info, reserve_pool,
                    pool_trim, pool_usage)

__all__ = ["Fmm2d", "FmmError", "LoopbackShards", "lib", "LIB_PATH", "PMAX", "SYMBOLS", "nccl_unique_id",
           "partition_info", "reserve_pool", "pool_trim", "pool_usage"]
