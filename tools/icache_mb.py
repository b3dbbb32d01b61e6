"""Instruction-fetch microbenchmark (tmb_microbench_icache): cycles per
instruction of straight-line blocks of growing size, 1 and 16 warps."""
import ctypes as ct
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_04212_b200 import _lib  # noqa: E402

out = {}
for warps in (1, 4, 16):
    for kb in (8, 16, 32, 64, 96, 128, 192, 256):
        for iters in (1, 20):
            c = ct.c_double()
            _lib.call("tmb_microbench_icache", kb, warps, iters, ct.byref(c))
            out[f"w{warps}_kb{kb}_it{iters}"] = round(c.value, 3)
print(json.dumps(out, indent=1))
