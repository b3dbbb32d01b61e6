"""Backend parity in the style of the reference's own test_kernels.py
(pkg/tests/test_kernels.py:20-86, numba <-> numpy), here b200 <-> numba:
the INTEGRATION.md stub must return bit-identical outputs, states, weights
and counters.  Runs inside the patched reference copy that
tools/run_reference_suite.py builds (tsetlinkit importable, GPU present)."""

import numpy as np
import pytest

from tsetlinkit.core import derive_stream
from tsetlinkit.kernels import load_backend

numba_k = pytest.importorskip("tsetlinkit.kernels._numba")
b200_k = load_backend("b200")


def bank(rng, C=9, P=14, K=3, lo=-20, hi=20):
    return (rng.integers(lo, hi, size=(C, P)).astype(np.int8),
            rng.integers(-6, 6, size=(C, K)).astype(np.int32))


@pytest.mark.parametrize("training", [True, False])
@pytest.mark.parametrize("budget", [1, 3, 14])
def test_outputs_b200_vs_numba(training, budget):
    rng = np.random.default_rng(10 + budget)
    for _ in range(30):
        states, _ = bank(rng)
        lits = rng.integers(0, 2, size=14).astype(np.uint8)
        assert np.array_equal(b200_k.clause_outputs(states, lits, training, budget),
                              numba_k.clause_outputs(states, lits, training, budget))
    x = rng.integers(0, 2, size=(57, 14)).astype(np.uint8)
    assert np.array_equal(b200_k.clause_outputs_batch(states, x, training, budget),
                          numba_k.clause_outputs_batch(states, x, training, budget))


@pytest.mark.parametrize("boost", [False, True])
@pytest.mark.parametrize("counter", [0, 5, (1 << 32) - 2])
def test_bank_feedback_b200_vs_numba(boost, counter):
    rng = np.random.default_rng(20 + counter % 97 + int(boost))
    seed = np.uint64(derive_stream(7, 3))
    for trial in range(20):
        s1, w1 = bank(rng, C=11, P=40, K=4, lo=-5, hi=5)
        s2, w2 = s1.copy(), w1.copy()
        lits = rng.integers(0, 2, size=40).astype(np.uint8)
        out = rng.integers(0, 2, size=11).astype(np.uint8)
        ut = rng.random(11) < 0.5
        un = rng.random(11) < 0.5
        label, neg = 1, 3
        ca = b200_k.bank_feedback(s1, w1, lits, out, label, neg, ut, un, 2.7, boost, -8, 8,
                                  seed, np.uint64(counter + trial))
        cb = numba_k.bank_feedback(s2, w2, lits, out, label, neg, ut, un, 2.7, boost, -8, 8,
                                   seed, np.uint64(counter + trial))
        assert int(ca) == int(cb)
        assert np.array_equal(s1, s2)
        assert np.array_equal(w1, w2)
