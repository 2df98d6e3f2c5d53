"""Probe: does cudaLimitMaxL2FetchGranularity (32 / 64 / 128 bytes) change the C5 phase times?
The random 8- and 16-byte gathers of k_finish and k_p2m move ~128 bytes of DRAM per element at the
default setting (ncu: 25.6 GB for 4.8 GB algorithmic).  usage: python tools/l2_fetch_probe.py 32 [bench args]"""
import ctypes
import os
import runpy
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rt = ctypes.CDLL("libcudart.so.12")
LIMIT = 0x05                                   # cudaLimitMaxL2FetchGranularity
cur = ctypes.c_size_t(0)
rt.cudaDeviceGetLimit(ctypes.byref(cur), LIMIT)
want = int(sys.argv[1])
rc = rt.cudaDeviceSetLimit(LIMIT, ctypes.c_size_t(want))
now = ctypes.c_size_t(0)
rt.cudaDeviceGetLimit(ctypes.byref(now), LIMIT)
print(f"[l2_fetch_probe] default {cur.value} -> requested {want}: rc {rc}, now {now.value}", file=sys.stderr)
sys.argv = [os.path.join(ROOT, "bench.py")] + sys.argv[2:]
runpy.run_path(sys.argv[0], run_name="__main__")
