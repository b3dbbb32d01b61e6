"""Per-call latency of the per-example plugin surface (kernels.py -> tmbh_*)
on the paper-listing XOR shapes (8 clauses x 12 positions)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2405_04212_b200 import kernels  # noqa: E402

rng = np.random.default_rng(0)
states = rng.integers(-5, 5, size=(8, 12)).astype(np.int8)
weights = rng.integers(-3, 3, size=(8, 2)).astype(np.int32)
lits = rng.integers(0, 2, size=12).astype(np.uint8)
out = kernels.clause_outputs(states, lits, True, 3)
ut = np.ones(8, bool)
un = np.zeros(8, bool)
for name, fn in (("clause_outputs", lambda: kernels.clause_outputs(states, lits, True, 3)),
                 ("bank_feedback", lambda: kernels.bank_feedback(
                     states, weights, lits, out, 0, 1, ut, un, 1.9, False, -127, 127,
                     np.uint64(5), np.uint64(0)))):
    for _ in range(50):
        fn()
    t = time.perf_counter()
    n = 2000
    for _ in range(n):
        fn()
    print(f"{name}: {(time.perf_counter() - t) / n * 1e6:.1f} us/call", flush=True)
