"""One isolated event-merge microbenchmark launch (for ncu): argv which n n_act warps."""
import ctypes as ct
import sys
sys.path.insert(0, ".")
from paper_2405_04212_b200 import _lib  # noqa: E402
w, n, na, nw = (int(a) for a in (sys.argv[1:5] if len(sys.argv) > 4 else (1, 84, 100, 1)))
us = ct.c_double()
_lib.call("tmb_microbench_sparse_event", w, n, na, 200, 148, nw, ct.byref(us))
print(f"which={w} n={n} n_act={na} warps={nw}: {us.value:.3f} us/event")
