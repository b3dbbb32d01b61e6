"""The reference arm of bench.py (--impl reference) drives the UNMODIFIED
reference (baseline/_ref, numba backend) through executor.train's serial
driver loop from a saved state.  Check that this driver computes exactly
what the oracle computes from the same state (CPU, no GPU)."""

import os
import sys

import numpy as np
import pytest

from conftest import REPO

sys.path.insert(0, REPO)


def _ref():
    import bench
    tk = bench.ref_package()
    if tk is None:
        pytest.skip("baseline/_ref (the pip-installed reference) or numba not available")
    return bench, tk


def test_ref_trainer_equals_oracle_from_checkpoint(oracle):
    bench, tk = _ref()
    from paper_2405_04212_b200 import datasets
    (tx, ty), _ = datasets.mnist_shaped(data_seed=7)
    ep, ck = bench._c2_checkpoint(3)
    assert ep == 3
    kw = datasets.mnist_shaped_config_kwargs(seed=0)
    tr = bench.RefTrainer(tk, kw, tx, ck)
    order = tr.next_order()[:150]
    tr.steps(ty, order)
    cfg = oracle.OracleCfg(**kw)
    st = oracle.OracleTrainState(ck["states"].copy(), ck["weights"].copy(),
                                 ck["block_counters"].copy(), int(ck["fb_counter"]),
                                 int(ck["shuffle_counter"]))
    o_order, _ = oracle.shuffle_permutation(len(ty), oracle.derive_stream(0, 0xD157),
                                            st.shuffle_counter)
    assert np.array_equal(order, o_order[:150])
    oracle.train_steps(cfg, st, oracle.augment_literals(tx), ty, o_order[:150])
    assert np.array_equal(tr.bank.states, st.states)
    assert np.array_equal(tr.bank.weights, st.weights)
    assert tr.blk_rng.counter == int(st.block_counters[0])
    assert tr.fb_rng.counter == st.fb_counter


def test_ref_trainer_fresh_equals_reference_train():
    """From the initial state, the driver loop == the reference's own
    train() (same model after one epoch of a small set)."""
    bench, tk = _ref()
    from paper_2405_04212_b200 import datasets
    (tx, ty), _ = datasets.noisy_xor(n_train=600, n_test=10)
    kw = datasets.noisy_xor_config_kwargs(seed=2)
    tr = bench.RefTrainer(tk, kw, tx)
    for _ in range(2):
        tr.steps(ty, tr.next_order())
    run = tk.train(tk.Config(**kw), (tx, ty), n_epochs=2)
    assert np.array_equal(tr.bank.states, run.model.states)
    assert np.array_equal(tr.bank.weights, run.model.weights)
