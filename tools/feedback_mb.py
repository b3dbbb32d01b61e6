"""Trainer feedback microbenchmark (tmb_microbench_feedback): SM cycles per
feedback call on the configs[1] per-CTA slice, by work-list length, for the
k_train_fast body (feedback_quads) and the compact one."""
import ctypes as ct
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_04212_b200 import _lib  # noqa: E402

out = {}
for threads in (512,):
    for variant in [int(v) for v in sys.argv[1:]] or (0, 6, 7, 8, 9, 10, 11):
        for two in (0, 1, 2):
            for nw in (1, 2, 3, 4, 8):
                c = ct.c_double()
                _lib.call("tmb_microbench_feedback", variant, nw, two, threads, 200, ct.byref(c))
                out[f"t{threads}_v{variant}_two{two}_nw{nw}"] = round(c.value, 1)
print(json.dumps(out, indent=1))
