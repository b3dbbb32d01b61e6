"""One tmb_microbench_feedback launch (for ncu): variant, n_work, two_events bits, threads."""
import ctypes as ct
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2405_04212_b200 import _lib  # noqa: E402

v, nw, two, thr = (int(a) for a in sys.argv[1:5])
c = ct.c_double()
_lib.call("tmb_microbench_feedback", v, nw, two, thr, 200, ct.byref(c))
print(c.value)
