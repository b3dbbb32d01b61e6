"""Latency of per-example all-reduce candidates (us per iteration)."""
import ctypes as ct
import sys
sys.path.insert(0, ".")
from paper_2405_04212_b200 import _lib, runtime  # noqa: E402

runtime.require_device()
for n_cta in (1, 16, 74, 148):
    row = []
    for mode in (0, 2, 4, 5, 10, 11, 12):
        v = ct.c_double()
        _lib.call("tmb_microbench_allreduce", n_cta, 512, 20000, mode, ct.byref(v))
        row.append(f"mode{mode}={v.value:.3f}")
    print(f"n_cta={n_cta:4d}  " + "  ".join(row))
