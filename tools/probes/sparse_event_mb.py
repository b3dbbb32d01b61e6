"""Isolated SparseTM event-merge timings (tmb_microbench_sparse_event)."""
import ctypes as ct
import sys
sys.path.insert(0, ".")
from paper_2405_04212_b200 import _lib  # noqa: E402
for which, name in ((0, "Type I out=0"), (1, "Type I out=1"), (2, "Type II")):
    for nw in (1, 4, 8, 16):
        us = ct.c_double()
        _lib.call("tmb_microbench_sparse_event", which, 84, 100, 200, 148, nw, ct.byref(us))
        print(f"{name:14s} n=84 n_act=100 warps/CTA={nw:2d}: {us.value:.3f} us/event")
