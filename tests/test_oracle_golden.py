"""Pin the CPU oracle against fixtures produced by the reference itself
(tests/golden/make_golden.py) and the reference's own known answers."""

import numpy as np
import pytest

from conftest import golden


def test_known_answers(oracle):
    # pkg/tests/test_core.py:104-106
    assert oracle.derive_stream(7, 3) == 0x2C7D03C103AFD766
    assert oracle.stream_u64(oracle.derive_stream(7, 3), 0) == 0xAB6B7B0CE9C8A6AB


def test_rng_golden(oracle):
    g = golden("rng")
    for i, s in enumerate(g["seeds"]):
        for j, idx in enumerate(g["idx"]):
            assert oracle.derive_stream(int(s), int(idx)) == int(g["derived"][i, j])
    for r, st in enumerate(g["starts"]):
        assert np.array_equal(oracle.stream_u64_block(int(g["block_seed"]), int(st), 64),
                              g["blocks"][r])
        assert np.array_equal(oracle.stream_u01_block(int(g["u01_seed"]), int(st), 64),
                              g["u01"][r])


def test_kernels_golden(oracle):
    g = golden("kernels")
    for t in range(int(g["n_cases"])):
        p = lambda k: g[f"c{t}_{k}"]  # noqa: E731
        label, negative, boost, smin, smax, budget = (int(v) for v in p("scalars"))
        states = p("states")
        assert np.array_equal(oracle.clause_outputs(states, p("lits"), True, budget), p("o_tr"))
        assert np.array_equal(oracle.clause_outputs(states, p("lits"), False, budget), p("o_inf"))
        assert np.array_equal(oracle.clause_outputs_batch(states, p("x_lit"), True, budget),
                              p("b_tr"))
        assert np.array_equal(oracle.clause_outputs_batch(states, p("x_lit"), False, budget,
                                                          nthreads=3), p("b_inf"))
        st, w = states.copy(), p("weights").copy()
        c = oracle.bank_feedback(st, w, p("lits"), p("outputs"), label, negative, p("ut"),
                                 p("un"), float(p("s")), boost, smin, smax, int(p("seed")),
                                 int(p("counter")))
        assert c == int(p("new_counter"))
        assert np.array_equal(st, p("st_after")), t
        assert np.array_equal(w, p("w_after")), t


def test_explicit_draws_hook_equals_stream(oracle):
    """The draws hook fed the reference stream's own draws reproduces
    bank_feedback bit for bit (the north star's one-step criterion)."""
    g = golden("kernels")
    for t in range(int(g["n_cases"])):
        p = lambda k: g[f"c{t}_{k}"]  # noqa: E731
        label, negative, boost, smin, smax, budget = (int(v) for v in p("scalars"))
        n_events = int(p("ut").sum() + p("un").sum())
        P = p("states").shape[1]
        c0 = int(p("counter"))
        draws = np.stack([oracle.stream_u01_block(int(p("seed")), ((c0 + e) << 32) & (2**64 - 1), P)
                          for e in range(max(n_events, 1))])
        st, w = p("states").copy(), p("weights").copy()
        c = oracle.bank_feedback_draws(st, w, p("lits"), p("outputs"), label, negative,
                                       p("ut"), p("un"), float(p("s")), boost, smin, smax,
                                       c0, draws)
        assert c == int(p("new_counter"))
        assert np.array_equal(st, p("st_after"))
        assert np.array_equal(w, p("w_after"))


def test_feedback_block_golden(oracle):
    g = golden("feedback")
    for i in range(g["K"].shape[0]):
        K, T, label = int(g["K"][i]), int(g["T"][i]), int(g["label"][i])
        fb_seed = oracle.derive_stream(int(g["seed"][i]), 0xFEED)
        ctr = int(g["ctr"][i])
        u = oracle.stream_u01(fb_seed, ctr)
        neg, pt, pn = oracle.update_probabilities(g["votes"][i, :K], label, T, u)
        assert neg == int(g["negative"][i])
        assert pt == g["p_target"][i] and pn == g["p_negative"][i]
        ut, un = oracle.sample_updates(pt, pn, 37, fb_seed, ctr + 1)
        assert np.array_equal(ut, g["ut"][i]) and np.array_equal(un, g["un"][i])
        assert ctr + 1 + 2 * 37 == int(g["ctr_after"][i])


def test_shuffle_golden(oracle):
    g = golden("shuffle")
    seed = oracle.derive_stream(5, 0xD157)
    for n in (0, 1, 2, 5, 100, 1000):
        a, c = oracle.shuffle_permutation(n, seed, 0)
        b, c = oracle.shuffle_permutation(n, seed, c)
        assert np.array_equal(a, g[f"n{n}_a"]) and np.array_equal(b, g[f"n{n}_b"])
        assert c == int(g[f"n{n}_ctr"])


def _cfg(**kw):
    from oracle.oracle import OracleCfg
    return OracleCfg(**kw)


def test_train_small_golden(oracle):
    g = golden("train_small")
    for i in range(4):
        seed, nb, boost, smin, smax, init = (int(v) for v in g[f"xor{i}_cfg"])
        cfg = _cfg(n_literals=6, n_clauses=8, n_classes=2, s=1.9, threshold=11,
                   n_literal_budget=3, seed=seed, n_blocks=nb, boost_true_positive=bool(boost),
                   state_min=smin, state_max=smax, init_state=init)
        st, accs = oracle.train(cfg, g["xor_x"], g["xor_y"], 3, (g["xor_ex"], g["xor_ey"]))
        assert np.array_equal(st.states, g[f"xor{i}_states"]), i
        assert np.array_equal(st.weights, g[f"xor{i}_weights"]), i
        assert np.array_equal(np.array(accs), g[f"xor{i}_acc"])
    cfg = _cfg(n_literals=20, n_clauses=30, n_classes=3, s=3.0, threshold=15, seed=77,
               n_blocks=2)
    x, y = g["mc_x"], g["mc_y"]
    st, accs = oracle.train(cfg, x[:400], y[:400], 2, (x[400:], y[400:]))
    assert np.array_equal(st.states, g["mc_states"])
    assert np.array_equal(st.weights, g["mc_weights"])
    assert np.array_equal(np.array(accs), g["mc_acc"])
    votes, _ = oracle.batch_votes(st.states, st.weights, oracle.augment_literals(x[400:]))
    assert np.array_equal(votes, g["mc_votes"])


def test_noisy_xor_config1_golden(oracle):
    """BASELINE config 1, 20 epochs, seeds 0-4: bit-exact final models."""
    g = golden("noisy_xor")
    from paper_2405_04212_b200 import datasets
    for seed in range(5):
        cfg = _cfg(**datasets.noisy_xor_config_kwargs(seed))
        st, accs = oracle.train(cfg, g["tx"], g["ty"], 20, (g["ex"], g["ey"]))
        assert np.array_equal(st.states, g[f"s{seed}_states"])
        assert np.array_equal(st.weights, g[f"s{seed}_weights"])
        assert np.array_equal(np.array(accs), g[f"s{seed}_acc"])


def test_mnist_prefix_golden(oracle):
    """BASELINE config 2 shapes (C=2000, P=1568, K=10), 300-example prefix."""
    g = golden("mnist_prefix")
    from paper_2405_04212_b200 import datasets
    cfg = _cfg(**datasets.mnist_shaped_config_kwargs(seed=1))
    st, accs = oracle.train(cfg, g["tx"], g["ty"], 1, (g["ex"], g["ey"]), nthreads=4)
    assert np.array_equal(st.states, g["states"])
    assert np.array_equal(st.weights, g["weights"])
    assert np.array_equal(np.array(accs), g["acc"])


def test_predictor_golden(oracle):
    g = golden("predictor")
    ptr, idx = g["inc_ptr"], g["inc_idx"]
    includes = [idx[ptr[r]:ptr[r + 1]] for r in range(ptr.shape[0] - 1)]
    votes, pred = oracle.ruleset_votes(includes, g["rs_weights"], g["allx"], 9)
    assert np.array_equal(votes, g["votes"])
    assert np.array_equal(pred, np.argmax(g["votes"], axis=1))
    bv, _ = oracle.batch_votes(g["states"], g["weights"], oracle.augment_literals(g["allx"]))
    assert np.array_equal(bv, g["votes"])


def test_sparse_golden(oracle):
    g = golden("sparse")
    ptr, ind = g["indptr"], g["indices"]
    acts = [ind[ptr[i]:ptr[i + 1]] for i in range(ptr.shape[0] - 1)]
    for i in range(3):
        seed, cap, floor, nb = (int(v) for v in g[f"r{i}_cfg"])
        cfg = _cfg(n_literals=60, n_clauses=10, n_classes=2, s=float(g[f"r{i}_s"]),
                   threshold=6, negated_literals_enabled=False, seed=seed,
                   sparse_capacity=None if cap < 0 else cap, sparse_floor=floor, n_blocks=nb)
        banks, _, _ = oracle.sparse_train(cfg, acts, g["labels"], n_epochs=2)
        lits = [l for bk in banks for l in bk.lits]
        sts = [s for bk in banks for s in bk.sts]
        lens = np.array([a.size for a in lits])
        assert np.array_equal(lens, g[f"r{i}_lens"]), i
        if lens.sum():
            assert np.array_equal(np.concatenate(lits), g[f"r{i}_lits"])
            assert np.array_equal(np.concatenate(sts), g[f"r{i}_sts"])
        w = np.concatenate([bk.weights for bk in banks])
        assert np.array_equal(w, g[f"r{i}_weights"])
        assert np.array_equal(oracle.sparse_batch_votes(banks, acts), g[f"r{i}_votes"])


@pytest.mark.parametrize("p", [0.1, 0.5, 1 / 1.9, 0.9 / 1.9, (3.9 - 1) / 3.9, 1 / 3.9, 0.9,
                               1.0 / 10.0, 9.0 / 10.0, 0.0, 1.0])
def test_integer_threshold_identity(p):
    """u < p  <=>  (z >> 11) < ceil(p * 2^53): the device compares integers."""
    import math
    t = math.ceil(p * 2.0 ** 53)
    rs = np.random.default_rng(0)
    m = rs.integers(0, 2 ** 53, size=20000, dtype=np.int64)
    m = np.concatenate([m, np.array([max(t - 2, 0), max(t - 1, 0), min(t, 2**53 - 1),
                                     min(t + 1, 2 ** 53 - 1)], dtype=np.int64)])
    u = m.astype(np.float64) * 2.0 ** -53
    assert np.array_equal(u < p, m < t)
