#!/usr/bin/env python3
"""Experiment: the context's L2 fetch granularity (cudaLimitMaxL2FetchGranularity) for the bench.
    python scripts/l2_fetch_exp.py BYTES bench-args...   (BYTES 0 = leave the default)
Sets the limit on the primary context of device 0 before torch touches it, prints the value read back, then runs
bench.py in-process with the remaining arguments."""
import ctypes as C
import glob
import os
import runpy
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
want = int(sys.argv[1])
cands = glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "nvidia", "cuda_runtime", "lib",
                               "libcudart.so*")) + glob.glob("/usr/local/cuda/lib64/libcudart.so*")
rt = C.CDLL(cands[0])
assert rt.cudaSetDevice(0) == 0
v = C.c_size_t(0)
rt.cudaDeviceGetLimit(C.byref(v), 5)  # cudaLimitMaxL2FetchGranularity
before = v.value
if want:
    rc = rt.cudaDeviceSetLimit(5, C.c_size_t(want))
    rt.cudaDeviceGetLimit(C.byref(v), 5)
    print(f"[l2_fetch] set {want}: rc {rc}, default {before}, now {v.value}", file=sys.stderr)
else:
    print(f"[l2_fetch] default {before}", file=sys.stderr)
sys.argv = [os.path.join(ROOT, "bench.py")] + sys.argv[2:]
runpy.run_path(sys.argv[0], run_name="__main__")
