"""Latency of per-example all-reduce candidates (us per iteration).
Modes: see tmb_microbench_allreduce (csrc/tmb_microbench.cu); 20 + G spreads
the trainer's packed arrivals over G L2 lines."""
import ctypes as ct
import sys
sys.path.insert(0, ".")
from paper_2405_04212_b200 import _lib, runtime  # noqa: E402

runtime.require_device()
modes = [int(a) for a in sys.argv[1:]] or [0, 2, 4, 21, 22, 24, 28, 36, 52]
for n_cta in (1, 16, 74, 148):
    row = []
    for mode in modes:
        v = ct.c_double()
        _lib.call("tmb_microbench_allreduce", n_cta, 512, 20000, mode, ct.byref(v))
        row.append(f"mode{mode}={v.value:.3f}")
    print(f"n_cta={n_cta:4d}  " + "  ".join(row), flush=True)
