"""GPU parity: the CUDA path (through the C ABI) against reference-generated
golden fixtures and the CPU oracle.  Bit-exact for everything (integer /
byte / index work; the float64 decision math is IEEE-identical)."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def test_device_rng_matches_reference(gpu):
    import torch
    g = golden("rng")
    from paper_2405_04212_b200 import _lib
    from paper_2405_04212_b200.runtime import ptr, stream_ptr
    for r, st in enumerate(g["starts"]):
        out = torch.empty(64, dtype=torch.int64, device="cuda")
        _lib.call("tmb_stream_u64_block", int(g["block_seed"]), int(st), 64, ptr(out),
                  stream_ptr())
        assert np.array_equal(out.cpu().numpy().view(np.uint64), g["blocks"][r])


def test_plugin_outputs_and_feedback_golden(gpu):
    k = gpu.kernels
    g = golden("kernels")
    for t in range(int(g["n_cases"])):
        p = lambda n: g[f"c{t}_{n}"]  # noqa: E731
        label, negative, boost, smin, smax, budget = (int(v) for v in p("scalars"))
        states = p("states")
        assert np.array_equal(k.clause_outputs(states, p("lits"), True, budget), p("o_tr"))
        assert np.array_equal(k.clause_outputs(states, p("lits"), False, budget), p("o_inf"))
        assert np.array_equal(k.clause_outputs_batch(states, p("x_lit"), True, budget), p("b_tr"))
        assert np.array_equal(k.clause_outputs_batch(states, p("x_lit"), False, budget),
                              p("b_inf"))
        st, w = states.copy(), p("weights").copy()
        c = k.bank_feedback(st, w, p("lits"), p("outputs"), label, negative, p("ut"), p("un"),
                            float(p("s")), boost, smin, smax, p("seed"), p("counter"))
        assert int(c) == int(p("new_counter")), t
        assert np.array_equal(st, p("st_after")), t
        assert np.array_equal(w, p("w_after")), t


def test_explicit_draws_hook(gpu, oracle):
    """One step's state delta is bit-exact when GPU and oracle consume the
    same explicit uniform draws -- both reference-stream draws (checked
    against the reference's own result) and arbitrary draws."""
    k = gpu.kernels
    g = golden("kernels")
    rs = np.random.default_rng(8)
    for t in range(int(g["n_cases"])):
        p = lambda n: g[f"c{t}_{n}"]  # noqa: E731
        label, negative, boost, smin, smax, _ = (int(v) for v in p("scalars"))
        n_ev = int(p("ut").sum() + p("un").sum())
        P = p("states").shape[1]
        c0 = int(p("counter"))
        stream = np.stack([oracle.stream_u01_block(int(p("seed")), ((c0 + e) << 32) % 2**64, P)
                           for e in range(max(n_ev, 1))])
        st, w = p("states").copy(), p("weights").copy()
        c = k.bank_feedback_draws(st, w, p("lits"), p("outputs"), label, negative, p("ut"),
                                  p("un"), float(p("s")), boost, smin, smax, c0, stream)
        assert int(c) == int(p("new_counter"))
        assert np.array_equal(st, p("st_after")) and np.array_equal(w, p("w_after"))
        arbitrary = rs.random((max(n_ev, 1), P))
        arbitrary[rs.random(arbitrary.shape) < 0.05] = 0.0
        st_g, w_g = p("states").copy(), p("weights").copy()
        st_o, w_o = p("states").copy(), p("weights").copy()
        k.bank_feedback_draws(st_g, w_g, p("lits"), p("outputs"), label, negative, p("ut"),
                              p("un"), float(p("s")), boost, smin, smax, c0, arbitrary)
        oracle.bank_feedback_draws(st_o, w_o, p("lits"), p("outputs"), label, negative,
                                   p("ut"), p("un"), float(p("s")), boost, smin, smax, c0,
                                   arbitrary)
        assert np.array_equal(st_g, st_o) and np.array_equal(w_g, w_o)


def _xor_cfg(gpu, i, g):
    seed, nb, boost, smin, smax, init = (int(v) for v in g[f"xor{i}_cfg"])
    return gpu.Config(n_literals=6, n_clauses=8, n_classes=2, s=1.9, threshold=11,
                      n_literal_budget=3, seed=seed, n_blocks=nb,
                      boost_true_positive=bool(boost), state_min=smin, state_max=smax,
                      init_state=init)


def test_train_small_golden(gpu):
    g = golden("train_small")
    for i in range(4):
        cfg = _xor_cfg(gpu, i, g)
        run = gpu.train(cfg, (g["xor_x"], g["xor_y"]), (g["xor_ex"], g["xor_ey"]), n_epochs=3)
        assert np.array_equal(run.model.states, g[f"xor{i}_states"]), i
        assert np.array_equal(run.model.weights, g[f"xor{i}_weights"]), i
        assert np.array_equal(np.array([m.accuracy for m in run.epoch_metrics]),
                              g[f"xor{i}_acc"])
    cfg = gpu.Config(n_literals=20, n_clauses=30, n_classes=3, s=3.0, threshold=15, seed=77,
                     n_blocks=2)
    x, y = g["mc_x"], g["mc_y"]
    run = gpu.train(cfg, (x[:400], y[:400]), (x[400:], y[400:]), n_epochs=2)
    assert np.array_equal(run.model.states, g["mc_states"])
    assert np.array_equal(run.model.weights, g["mc_weights"])
    assert np.array_equal(np.array([m.accuracy for m in run.epoch_metrics]), g["mc_acc"])
    assert np.array_equal(gpu.dataset_votes(run.model, (x[400:], y[400:])), g["mc_votes"])


@pytest.mark.parametrize("n_cta", [1, 3, 8])
@pytest.mark.parametrize("hbm", [False, True])
def test_train_multi_cta_layouts(gpu, n_cta, hbm):
    """Same model for any CTA count and either state residency."""
    g = golden("train_small")
    for i in (0, 1, 3):
        cfg = _xor_cfg(gpu, i, g)
        sess = gpu.DenseTrainSession(cfg, g["xor_x"], g["xor_y"], n_cta=n_cta,
                                     states_in_hbm=hbm)
        for _ in range(3):
            sess.run_epoch()
        m = sess.model()
        assert np.array_equal(m.states, g[f"xor{i}_states"]), (i, n_cta, hbm)
        assert np.array_equal(m.weights, g[f"xor{i}_weights"]), (i, n_cta, hbm)


@pytest.mark.parametrize("n_cta", [1, 7, 16, 20, 37])
@pytest.mark.parametrize("n_blocks", [1, 3, 11])
def test_train_block_layouts_vs_oracle(gpu, oracle, n_cta, n_blocks):
    """Clause blocks that straddle CTA boundaries in both sync domains
    (cluster mode up to 16 CTAs, grid mode above), odd P (not a multiple of
    4: scalar state path), HBM-resident states."""
    rs = np.random.default_rng(n_cta * 100 + n_blocks)
    x = rs.integers(0, 2, size=(250, 27)).astype(np.uint8)
    y = ((x[:, 0] + x[:, 3] * 2 + x[:, 9]) % 4).astype(np.int64)
    cfg = gpu.Config(n_literals=27, n_clauses=45, n_classes=4, s=2.5, threshold=9, seed=n_cta,
                     n_blocks=n_blocks, n_literal_budget=6)
    ost, _ = oracle.train(cfg, x, y, 2)
    for hbm, bal in ((False, True), (True, True), (True, False)):
        sess = gpu.DenseTrainSession(cfg, x, y, n_cta=n_cta, states_in_hbm=hbm,
                                     balanced_feedback=bal)
        sess.run_epoch()
        sess.run_epoch()
        m = sess.model()
        assert np.array_equal(m.states, ost.states), (n_cta, n_blocks, hbm, bal)
        assert np.array_equal(m.weights, ost.weights), (n_cta, n_blocks, hbm, bal)
        assert np.array_equal(sess.block_counters.cpu().numpy().view(np.uint64),
                              ost.block_counters)


def test_noisy_xor_config1_all_seeds(gpu):
    """BASELINE config 1, 20 epochs x seeds 0-4: bit-exact final models and
    per-epoch accuracies, hence identical 5-seed mean accuracy."""
    g = golden("noisy_xor")
    accs_gpu, accs_ref = [], []
    for seed in range(5):
        cfg = gpu.Config(**gpu.datasets.noisy_xor_config_kwargs(seed))
        run = gpu.train(cfg, (g["tx"], g["ty"]), (g["ex"], g["ey"]), n_epochs=20)
        assert np.array_equal(run.model.states, g[f"s{seed}_states"])
        assert np.array_equal(run.model.weights, g[f"s{seed}_weights"])
        accs_gpu.append(run.epoch_metrics[-1].accuracy)
        accs_ref.append(float(g[f"s{seed}_acc"][-1]))
    assert abs(np.mean(accs_gpu) - np.mean(accs_ref)) <= 0.01  # north star: +-1 point
    assert accs_gpu == accs_ref


def test_mnist_shaped_prefix_golden(gpu):
    """BASELINE config 2 shapes (C=2000, P=1568, K=10, T=5000, s=10) over a
    300-example prefix: bit-exact against the reference itself."""
    g = golden("mnist_prefix")
    cfg = gpu.Config(**gpu.datasets.mnist_shaped_config_kwargs(seed=1))
    run = gpu.train(cfg, (g["tx"], g["ty"]), (g["ex"], g["ey"]), n_epochs=1)
    assert np.array_equal(run.model.states, g["states"])
    assert np.array_equal(run.model.weights, g["weights"])
    assert np.array_equal(np.array([m.accuracy for m in run.epoch_metrics]), g["acc"])
    assert np.array_equal(gpu.dataset_votes(run.model, (g["ex"], g["ey"])), g["votes"])


@pytest.mark.parametrize("n_cta,hbm,n_blocks,keys", [
    (0, False, 5, True), (0, True, 5, True), (148, False, 5, True), (148, True, 5, True),
    (5, False, 5, True), (64, True, 5, True),
    (148, False, 1, True), (148, True, 1, True), (148, False, 1, False), (37, False, 1, True),
    (148, True, 1, False), (23, True, 3, True)])
def test_mnist_shaped_longer_vs_oracle(gpu, oracle, n_cta, hbm, n_blocks, keys):
    """2 epochs over 1500 examples of the config-2 shapes against the oracle,
    in cluster mode (<= 16 CTAs, DSMEM exchange) and grid mode (cooperative
    grid, global barrier), with per-block counters via n_blocks=5, and with
    one block through both flag paths (precomputed 16-bit keys: ~180 key
    ties resolved exactly over the run; per-CTA draws); the generic grid
    kernel with HBM states splits the feedback over all CTAs."""
    (tx, ty), (ex, ey) = gpu.datasets.mnist_shaped(n_train=1500, n_test=300, data_seed=3)
    kw = gpu.datasets.mnist_shaped_config_kwargs(seed=9)
    kw["n_blocks"] = n_blocks
    cfg = gpu.Config(**kw)
    sess = gpu.DenseTrainSession(cfg, tx, ty, n_cta=n_cta, states_in_hbm=hbm, flag_keys=keys)
    for _ in range(2):
        sess.run_epoch()
    m = sess.model()
    ost, _ = oracle.train(cfg, tx, ty, 2)
    assert np.array_equal(m.states, ost.states)
    assert np.array_equal(m.weights, ost.weights)
    assert np.array_equal(sess.block_counters.cpu().numpy().view(np.uint64),
                          ost.block_counters)


def test_keyed_trainer_chunked_launches(gpu, oracle):
    """The keyed trainer splits long runs into launches whose keys fit its
    buffer; a tiny forced chunk (and one not dividing the epoch) must give
    the same model."""
    (tx, ty), _ = gpu.datasets.mnist_shaped(n_train=700, n_test=10, data_seed=4)
    cfg = gpu.Config(**gpu.datasets.mnist_shaped_config_kwargs(seed=2))
    ost, _ = oracle.train(cfg, tx, ty, 1)
    try:
        for chunk in (1, 97):
            gpu._lib.call("tmb_set_option", b"train.key_chunk", chunk)
            sess = gpu.DenseTrainSession(cfg, tx, ty, n_cta=148)
            sess.run_epoch()
            m = sess.model()
            assert np.array_equal(m.states, ost.states), chunk
            assert np.array_equal(m.weights, ost.weights), chunk
    finally:
        gpu._lib.call("tmb_set_option", b"train.key_chunk", 0)


def test_predictor_golden(gpu):
    g = golden("predictor")
    bank = gpu.DenseClauseBank(gpu.Config(n_literals=9, n_clauses=16, n_classes=2, s=3.0,
                                          threshold=8, seed=4, n_blocks=2))
    bank.states[:] = g["states"]
    bank.weights[:] = g["weights"]
    rs = gpu.compile_ruleset(bank)
    ptr, idx, w = rs.csr()
    assert np.array_equal(ptr, g["inc_ptr"]) and np.array_equal(idx, g["inc_idx"])
    assert np.array_equal(w, g["rs_weights"])
    votes = gpu.predictor.rule_votes_batch(rs, g["allx"])
    assert np.array_equal(votes, g["votes"])
    assert np.array_equal(gpu.predict_batch(rs, g["allx"]), np.argmax(g["votes"], axis=1))
    for i, row in enumerate(g["allx"][:64]):
        p, e = gpu.predict_and_explain(rs, row, level="literal")
        _, f = gpu.predict_and_explain(rs, row, level="feature")
        assert p == g["preds"][i]
        assert np.array_equal(e.scores, g["lit_scores"][i])
        assert np.array_equal(f.scores, g["feat_scores"][i])
    lit = gpu.augment_literals(g["allx"])
    assert np.array_equal(bank.batch_votes(lit), g["votes"])
    # the batched device path against the reference's own explanations
    p64, s64 = gpu.predict_and_explain_batch(rs, g["allx"][:64], level="literal")
    _, f64 = gpu.predict_and_explain_batch(rs, g["allx"][:64], level="feature")
    assert np.array_equal(p64, g["preds"])
    assert np.array_equal(s64, g["lit_scores"]) and np.array_equal(f64, g["feat_scores"])


def _explain_reference(includes, weights, n_literals, negations, x, for_class):
    # predictor.py:99-124 restated (test oracle)
    lit = np.concatenate([x, 1 - x]) if negations else x
    votes = np.zeros(weights.shape[1], dtype=np.int64)
    fired = []
    for inc, w in zip(includes, weights):
        if np.all(lit[inc] == 1):
            votes += w
            fired.append((inc, w))
    pred = int(np.argmax(votes))
    cls = pred if for_class is None else for_class
    scores = np.zeros(lit.shape[0], dtype=np.int64)
    for inc, w in fired:
        scores[inc] += int(w[cls])
    return pred, scores


@pytest.mark.parametrize("negations", [True, False])
@pytest.mark.parametrize("for_class", [None, 2])
def test_predict_and_explain_batch_random(gpu, negations, for_class):
    """Batched explanations on a larger random rule set with planted firing
    (many rules fire per example), with and without negations, for the
    predicted class and a fixed class."""
    rs_ = np.random.default_rng(17 + int(negations))
    F, R, K, N = 300, 800, 5, 257
    P = 2 * F if negations else F
    includes = []
    for _ in range(R):
        n = int(rs_.integers(1, 6))
        feats = rs_.choice(F, size=n, replace=False)
        pol = rs_.integers(0, 2, size=n) if negations else np.zeros(n, dtype=np.int64)
        includes.append(np.sort(feats + F * pol).astype(np.int64))
    weights = rs_.integers(-9, 10, size=(R, K)).astype(np.int32)
    x = rs_.integers(0, 2, size=(N, F)).astype(np.uint8)
    for e in range(N):
        for j in rs_.integers(0, R, size=6):
            inc = includes[int(j)]
            x[e, inc[inc < F]] = 1
            x[e, inc[inc >= F] - F] = 0
    rset = gpu.RuleSet(F, K, negations, tuple(includes), weights)
    preds, scores = gpu.predict_and_explain_batch(rset, x, level="literal", for_class=for_class)
    for e in range(N):
        p, s = _explain_reference(includes, weights, F, negations, x[e], for_class)
        assert preds[e] == p, e
        assert np.array_equal(scores[e], s), e
    assert (scores != 0).any()


@pytest.mark.parametrize("n_inc,F,K", [(1, 37, 3), (2, 64, 10), (3, 300, 4), (20, 4096, 10)])
def test_inference_random_models_vs_oracle(gpu, oracle, n_inc, F, K):
    """Config-3-style random include models; low include counts make many
    clauses fire (the config-3 model itself fires on ~1% of examples)."""
    rs = np.random.default_rng(n_inc * 1000 + F)
    C = 700
    m = gpu.datasets.inference_model(model_seed=n_inc + F, n_features=F, n_clauses=C,
                                     n_classes=K, n_includes=n_inc)
    N = 3000 if F < 4096 else 800
    x = rs.integers(0, 2, size=(N, F)).astype(np.uint8)
    bank = gpu.DenseClauseBank(gpu.Config(n_literals=F, n_clauses=C, n_classes=K, s=2.0,
                                          threshold=10))
    bank.states[:] = m.states
    bank.weights[:] = m.weights
    votes = gpu.dataset_votes(bank, (x, None))
    ov, op = oracle.batch_votes(m.states, m.weights, oracle.augment_literals(x), nthreads=8)
    assert np.array_equal(votes, ov)
    model = gpu.CompiledModel.from_bank(bank)
    _, pred = model.votes_and_pred(x, want_votes=False, chunk=257)
    assert np.array_equal(pred, op)


@pytest.mark.parametrize("kernel", ["solo", "ws", "ws_plain", "ws_noexit", "cluster", "generic"])
@pytest.mark.parametrize("n_inc,F,K,C,N", [(40, 64, 3, 300, 1000), (17, 784, 10, 2001, 700),
                                           (1, 32, 32, 33, 129), (5, 1000, 2, 5000, 300)])
def test_inference_kernels_tails_and_shapes(gpu, oracle, kernel, n_inc, F, K, C, N):
    """All inference kernels (per-CTA solo, warp-specialised cluster,
    alternating cluster, generic): rules longer than the 16-code heads (tails), feature
    widths that are not multiples of 32, K up to 32, ragged tiles, and
    firing blocks in many tiles (votes pushed across the cluster)."""
    from paper_2405_04212_b200 import _lib
    _lib.call("tmb_set_option", b"infer.force_generic", int(kernel == "generic"))
    _lib.call("tmb_set_option", b"infer.solo", int(kernel == "solo"))
    _lib.call("tmb_set_option", b"infer.warp_specialized", int(kernel.startswith("ws")))
    _lib.call("tmb_set_option", b"infer.eval_mode",
              {"ws_plain": 0, "ws_noexit": 3}.get(kernel, 2))
    try:
        rs = np.random.default_rng(n_inc + F + K)
        # satisfiable clauses: n_inc distinct features, random polarity
        states = np.full((C, 2 * F), -1, dtype=np.int8)
        for j in range(C):
            feats = rs.choice(F, size=n_inc, replace=False)
            pol = rs.integers(0, 2, size=n_inc)
            states[j, feats + F * pol] = 0
        weights = rs.integers(-7, 8, size=(C, K)).astype(np.int32)

        class _M:
            pass
        m = _M()
        m.states, m.weights = states, weights
        # plant firing: make some examples satisfy some clauses
        x = rs.integers(0, 2, size=(N, F)).astype(np.uint8)
        for e in range(0, N, 3):
            j = int(rs.integers(0, C))
            inc = np.flatnonzero(m.states[j] >= 0)
            x[e, inc[inc < F]] = 1
            x[e, inc[inc >= F] - F] = 0
        bank = gpu.DenseClauseBank(gpu.Config(n_literals=F, n_clauses=C, n_classes=K, s=2.0,
                                              threshold=10))
        bank.states[:] = m.states
        bank.weights[:] = m.weights
        model = gpu.CompiledModel.from_bank(bank)
        votes, pred = model.votes_and_pred(x, chunk=200)
        ov, op = oracle.batch_votes(m.states, m.weights, oracle.augment_literals(x), nthreads=8)
        assert np.array_equal(votes, ov)
        assert np.array_equal(pred, op)
        assert (ov != 0).any()
    finally:
        _lib.call("tmb_set_option", b"infer.force_generic", 0)
        _lib.call("tmb_set_option", b"infer.solo", 1)
        _lib.call("tmb_set_option", b"infer.warp_specialized", 1)
        _lib.call("tmb_set_option", b"infer.eval_mode", 2)


def test_inference_ties_and_empty(gpu):
    bank = gpu.DenseClauseBank(gpu.Config(n_literals=2, n_clauses=2, n_classes=3, s=2.0,
                                          threshold=5))
    x = np.array([[1, 0], [0, 1], [1, 1]], dtype=np.uint8)
    assert gpu.evaluate(bank, (x, np.array([0, 2, 1]))) == pytest.approx(1 / 3)
    bank.states[0, 0] = 0
    bank.weights[0] = [0, 3, 3]   # tie between classes 1 and 2 -> 1
    v = gpu.dataset_votes(bank, (x, None))
    assert v.tolist() == [[0, 3, 3], [0, 0, 0], [0, 3, 3]]
    rs = gpu.compile_ruleset(bank)
    assert gpu.predict_batch(rs, x).tolist() == [1, 0, 1]


def test_inference_rejects_non_binary(gpu):
    bank = gpu.DenseClauseBank(gpu.Config(n_literals=4, n_clauses=2, n_classes=2, s=2.0,
                                          threshold=5))
    bank.states[0, 0] = 0
    bank.weights[0] = [1, 0]
    with pytest.raises(gpu.TmbError):
        gpu.dataset_votes(bank, (np.array([[2, 0, 1, 0]], dtype=np.uint8), None))


def test_scalar_spec_functions(gpu):
    """dense.py:29-113 spec helpers (routed through the device kernels)."""
    from paper_2405_04212_b200.core import RngStream, stream_u01_block
    states = np.array([5, -1], dtype=np.int8)
    rng = RngStream.derive(1, 0)
    u0 = stream_u01_block(rng.stream_seed, 0, 1)[0]
    gpu.type_i_feedback(states, np.array([1, 1], np.uint8), 1, 5.0, rng)
    assert states[0] == (6 if u0 < 0.8 else 5) and rng.counter == 1
    st = np.array([-5, 3], dtype=np.int8)
    gpu.type_ii_feedback(st, np.array([0, 0], np.uint8), 1)
    assert st.tolist() == [-4, 3]
    assert gpu.evaluate_clause(np.array([0, -1, -1, 0], np.int8),
                               np.array([1, 0, 0, 1], np.uint8), gpu.EvalMode.INFERENCE, 4) == 1
    bank = gpu.DenseClauseBank(gpu.Config(n_literals=2, n_clauses=2, n_classes=2, s=1.9,
                                          threshold=11, seed=5))
    rng = RngStream.derive(1, 0)
    gpu.clause_update(bank, 0, 0, 1, True, 1, np.array([1, 1, 0, 0], np.uint8), rng)
    assert bank.weights[0, 0] == 1 and rng.counter == 1
    bank.weights[0, 1] = -3
    gpu.clause_update(bank, 0, 1, -1, True, 1, np.array([1, 1, 0, 0], np.uint8), rng)
    assert bank.weights[0, 1] == -4


def test_sample_updates_device_draws(gpu):
    from paper_2405_04212_b200.core import RngStream
    g = golden("feedback")
    for i in range(40):
        K, T, label = int(g["K"][i]), int(g["T"][i]), int(g["label"][i])
        rng = RngStream(gpu.derive_stream(int(g["seed"][i]), 0xFEED), int(g["ctr"][i]))
        d = gpu.update_probabilities(g["votes"][i, :K], label, T, rng)
        assert d.negative_class == int(g["negative"][i])
        assert d.p_target == g["p_target"][i] and d.p_negative == g["p_negative"][i]
        ut, un = gpu.sample_updates(d, 37, rng)
        assert np.array_equal(ut, g["ut"][i]) and np.array_equal(un, g["un"][i])
        assert rng.counter == int(g["ctr_after"][i])


def test_facade_listing(gpu):
    (tx, ty), (ex, ey) = gpu.datasets.noisy_xor(n_train=500, n_test=200)
    tm = gpu.TsetlinMachine(n_literals=12, n_clauses=10, n_classes=2, s=3.9, threshold=15)
    tr = gpu.Trainer(tm, n_epochs=2, seed=1)
    tr.set_train_data(tx, ty)
    tr.set_eval_data(ex, ey)
    res = tr.train()
    assert len(res["eval_acc"]) == 2
    pr = tm.get_predictor()
    assert pr.predict(ex).shape == (200,)
    cls, expl = pr.predict_and_explain(ex[0])
    assert 0 <= cls < 2 and expl.scores.shape == (24,)


# ------------------------------------------------------------------ SparseTM

@pytest.fixture(params=[1, 0], ids=["resident", "global"])
def sparse_mode(request, gpu):
    """Both trainer layouts: clause lists resident in shared memory (default
    when they fit) and lists in global memory with per-event staging."""
    from paper_2405_04212_b200 import _lib
    _lib.call("tmb_set_option", b"sparse.resident", request.param)
    yield request.param
    _lib.call("tmb_set_option", b"sparse.resident", 1)


def _sparse_golden_data(gpu):
    g = golden("sparse")
    ptr, ind = g["indptr"], g["indices"]
    ex = [gpu.SparseExample(ind[ptr[i]:ptr[i + 1]], int(g["labels"][i]))
          for i in range(ptr.shape[0] - 1)]
    return g, gpu.SparseDataset(60, ex)


def test_sparse_train_golden(gpu, sparse_mode):
    """SparseClauseBank training incl. capacity rule, floor/evict, candidate
    domain and 3 clause blocks: bit-exact lists, states, weights, votes."""
    g, ds = _sparse_golden_data(gpu)
    for i in range(3):
        seed, cap, floor, nb = (int(v) for v in g[f"r{i}_cfg"])
        cfg = gpu.Config(n_literals=60, n_clauses=10, n_classes=2, s=float(g[f"r{i}_s"]),
                         threshold=6, negated_literals_enabled=False, seed=seed,
                         sparse_capacity=None if cap < 0 else cap, sparse_floor=floor,
                         n_blocks=nb)
        m = gpu.train(cfg, ds, n_epochs=2).model
        lens = np.array([a.size for a in m.clause_literals])
        assert np.array_equal(lens, g[f"r{i}_lens"]), i
        if lens.sum():
            assert np.array_equal(np.concatenate(m.clause_literals), g[f"r{i}_lits"])
            assert np.array_equal(np.concatenate(m.clause_states), g[f"r{i}_sts"])
        assert np.array_equal(m.weights, g[f"r{i}_weights"])
        assert np.array_equal(m.batch_votes(ds.examples), g[f"r{i}_votes"])


def test_sparse_dense_equivalence(gpu, sparse_mode):
    """test_acceptance.py:66-96 oracle: with the floor at the dense clamp and
    no capacity, the sparse engine replays the dense engine exactly."""
    rs = np.random.default_rng(11)
    ex = []
    for _ in range(100):
        k = int(rs.integers(3, 12))
        ex.append(gpu.SparseExample(np.sort(rs.choice(50, size=k, replace=False)),
                                    int(rs.integers(0, 2))))
    data = gpu.SparseDataset(50, ex)
    floor = -15
    cfg = gpu.Config(n_literals=50, n_clauses=16, n_classes=2, s=2.5, threshold=10, seed=99,
                     n_blocks=4, negated_literals_enabled=False, init_state=floor,
                     state_min=floor, sparse_floor=floor)
    for epochs in (1, 3):
        dense = gpu.train(cfg, data.densify(), n_epochs=epochs).model
        sparse = gpu.train(cfg, data, n_epochs=epochs).model
        assert np.array_equal(dense.weights, sparse.weights)
        for j in range(cfg.n_clauses):
            lits = sparse.clause_literals[j]
            assert np.array_equal(dense.states[j, lits], sparse.clause_states[j])
            assert np.all(dense.states[j, np.setdiff1d(np.arange(50), lits)] == floor)
        xs, _ = data.densify()
        assert np.array_equal(gpu.dataset_votes(dense, (xs, None)), sparse.batch_votes(ex))


def test_sparse_bank_feedback_rules(gpu):
    """test_sparse.py:107-163 semantics through the bank-level device API."""
    from paper_2405_04212_b200.core import RngStream

    def bank(cands=None, **kw):
        p = dict(n_literals=12, n_clauses=2, n_classes=2, s=2.0, threshold=5, seed=1,
                 negated_literals_enabled=False, sparse_floor=-4)
        p.update(kw)
        cfg = gpu.Config(**p)
        return gpu.SparseClauseBank(cfg, candidate_literals=np.arange(12) if cands is None
                                    else cands)

    ex = lambda a: gpu.SparseExample(np.array(a, dtype=np.int64), 0)  # noqa: E731
    b = bank()
    b.weights[0, 1] = 1
    gpu.sparse.sparse_feedback(b, 0, 1, -1, True, 1, ex([0]), RngStream.derive(1, 0))
    assert b.lookup(0, 3) == -3 and b.lookup(0, 0) == -4
    b = bank(cands=np.array([0, 1]))
    b.weights[0, 1] = 1
    gpu.sparse.sparse_feedback(b, 0, 1, -1, True, 1, ex([0]), RngStream.derive(1, 0))
    assert b.clause_literals[0].tolist() == [1]
    b = bank(s=1.0001)
    b.clause_literals[0] = np.array([4], dtype=np.int64)
    b.clause_states[0] = np.array([-3], dtype=np.int8)
    gpu.sparse.sparse_feedback(b, 0, 0, 1, True, 0, ex([]), RngStream.derive(1, 0))
    assert b.clause_literals[0].size == 0
    b = bank(sparse_capacity=2)
    b.weights[0, 1] = 1
    rng = RngStream.derive(1, 0)
    gpu.sparse.sparse_feedback(b, 0, 1, -1, True, 1, ex([11]), rng)
    assert b.clause_literals[0].tolist() == [0, 1] and b.clause_states[0].tolist() == [-3, -3]
    assert rng.counter == 1
    # capacity is not a hard cap: stored pairs always survive
    b = bank(sparse_capacity=2)
    b.clause_literals[0] = np.array([5, 6], dtype=np.int64)
    b.clause_states[0] = np.array([-2, -3], dtype=np.int8)
    b.weights[0, 1] = 1
    gpu.sparse.sparse_feedback(b, 0, 1, -1, True, 1, ex([]), RngStream.derive(1, 0))
    assert b.clause_literals[0].tolist() == [0, 1, 5, 6]


def test_sparse_large_vocab_prefix_vs_oracle(gpu, oracle, sparse_mode):
    """configs[4] shapes on a small slice: 10^6-literal universe, Zipf(1.05)
    documents of 100 tokens, 2000 clauses, capacity 64, floor -15, T=2000,
    s=5 -- 3 training documents against the oracle (its Type II walks all
    ~10^5 candidates), then inference parity on 200 documents."""
    d = gpu.datasets.sparse_zipf(n_docs=2000)
    kw = gpu.datasets.sparse_config_kwargs(seed=3)
    cfg = gpu.Config(**kw)
    acts = [d.row(i) for i in range(len(d))]
    from paper_2405_04212_b200.sparse_train import SparseTrainSession
    sess = SparseTrainSession(cfg, d.indptr, d.indices, d.labels)
    sess.run_epoch(max_steps=3)
    m = sess.model()
    banks, bctr, _ = oracle.sparse_train(cfg, acts, d.labels, n_epochs=1, max_steps=3)
    ob = banks[0]
    assert np.array_equal(m.weights, ob.weights)
    for j in range(cfg.n_clauses):
        assert np.array_equal(m.clause_literals[j], ob.lits[j]), j
        assert np.array_equal(m.clause_states[j], ob.sts[j]), j
    ex = [gpu.SparseExample(a, 0) for a in acts[:200]]
    assert np.array_equal(m.batch_votes(ex), oracle.sparse_batch_votes(banks, acts[:200]))


def test_sparse_resident_equals_global_long_run(gpu):
    """configs[4] shapes, 3000 documents: the shared-memory-resident trainer
    and the global-list trainer end in byte-identical models."""
    from paper_2405_04212_b200 import _lib
    from paper_2405_04212_b200.sparse_train import SparseTrainSession
    d = gpu.datasets.sparse_zipf(n_docs=3000)
    cfg = gpu.Config(**gpu.datasets.sparse_config_kwargs(seed=4))
    models = []
    for mode in (1, 0):
        _lib.call("tmb_set_option", b"sparse.resident", mode)
        try:
            sess = SparseTrainSession(cfg, d.indptr, d.indices, d.labels)
            assert sess.engine.resident == bool(mode)
            sess.run_epoch()
            models.append((sess.model(), sess.stats_dict()))
        finally:
            _lib.call("tmb_set_option", b"sparse.resident", 1)
    (a, sa), (b, sb) = models
    assert sa == sb and sa["events"] > 0
    assert np.array_equal(a.weights, b.weights)
    for j in range(cfg.n_clauses):
        assert np.array_equal(a.clause_literals[j], b.clause_literals[j]), j
        assert np.array_equal(a.clause_states[j], b.clause_states[j]), j


def test_cross_validate_golden(gpu):
    """tuning.cross_validate on the GPU trainer == the reference's report."""
    g = golden("tuning")
    cfg = gpu.Config(n_literals=6, n_clauses=8, n_classes=2, s=1.9, threshold=11,
                     n_literal_budget=3, seed=0)
    from paper_2405_04212_b200 import tuning
    rep = tuning.cross_validate(cfg, (g["cv_x"], g["cv_y"]), 4, 2, seed=9)
    assert np.array_equal(rep.fold_assignments, g["cv_folds"])
    assert np.array_equal(np.array(rep.fold_accuracies), g["cv_acc"])


@pytest.mark.parametrize("tag", ["hold", "cv"])
def test_random_search_golden(gpu, tag):
    """tuning.random_search on the GPU trainer == the reference's ranked
    trials (tuning.py:194-227), holdout and cv_k variants."""
    g = golden("search")
    base = gpu.Config(n_literals=6, n_clauses=8, n_classes=2, s=2.0, threshold=10, seed=0)
    small = gpu.SearchSpace.parse("s uniform 1.5 4.0\nthreshold int 5 20\nn_clauses cat 6,10")
    kw = {"cv_k": 3} if tag == "cv" else {}
    trials = gpu.random_search(small, base, (g["x"], g["y"]), n_trials=5, n_epochs=2, seed=31,
                               **kw)
    assert [t.index for t in trials] == g[tag + "_index"].tolist()
    assert np.array_equal([t.accuracy for t in trials], g[tag + "_acc"])
    assert np.array_equal([t.config.s for t in trials], g[tag + "_s"])


@pytest.fixture(params=[1, 0], ids=["solo", "cluster"])
def infer_kernel(request, gpu):
    from paper_2405_04212_b200 import _lib
    _lib.call("tmb_set_option", b"infer.solo", request.param)
    yield request.param
    _lib.call("tmb_set_option", b"infer.solo", 1)


@pytest.mark.parametrize("F,n_inc,N", [(4096, 20, 3000), (300, 3, 1000), (128, 2, 777)])
def test_inference_bit_packed_input(gpu, oracle, infer_kernel, F, n_inc, N):
    """Bit-packed input (uint64 words, feature f = bit f % 64 of word f // 64)
    through the packed transposer: identical votes / predictions to the uint8
    path and to the oracle, including widths that are not multiples of 128
    (8-byte loads) and ragged tiles."""
    import torch
    m = gpu.datasets.inference_model(model_seed=5, n_features=F, n_clauses=2000,
                                     n_includes=n_inc)
    bank = gpu.DenseClauseBank(gpu.Config(n_literals=F, n_clauses=2000, n_classes=10, s=2.0,
                                          threshold=100))
    bank.states[:] = m.states
    bank.weights[:] = m.weights
    model = gpu.CompiledModel.from_bank(bank)
    xb = gpu.datasets.inference_examples(3, 11, N, n_features=F, packed=True)
    x = gpu.datasets.inference_examples(3, 11, N, n_features=F)
    vb, pb = model.votes_and_pred_packed(xb)
    v8, p8 = model.votes_and_pred(x)
    assert np.array_equal(vb, v8) and np.array_equal(pb, p8)
    ov, op = oracle.batch_votes(m.states, m.weights, oracle.augment_literals(x), nthreads=8)
    assert np.array_equal(vb, ov) and np.array_equal(pb, op)
    # a base 8 bytes off 16-byte alignment forces the 8-byte load path
    flat = torch.zeros(xb.size + 1, dtype=torch.int64, device="cuda")
    xd = flat[1:].view(N, xb.shape[1])
    xd.copy_(torch.from_numpy(xb.view(np.int64)))
    pred = torch.empty(N, dtype=torch.int64, device="cuda")
    model.infer_device_packed(xd, pred_dev=pred)
    assert np.array_equal(pred.cpu().numpy(), op)


def test_configs1_three_full_epochs_vs_oracle(gpu):
    """The bench workload itself: 3 full configs[1] epochs (180 000 examples,
    2000 clauses x 1568 literal positions x 10 classes, T=5000, s=10) through
    the production fused trainer == the oracle's model, RNG counters and
    shuffle position after the same 3 epochs (tests/golden/c2_epoch3.npz,
    written by tests/golden/make_c2_epoch3.py)."""
    g = golden("c2_epoch3")
    (tx, ty), _ = gpu.datasets.mnist_shaped(data_seed=7)
    cfg = gpu.Config(**gpu.datasets.mnist_shaped_config_kwargs(seed=0))
    sess = gpu.DenseTrainSession(cfg, tx, ty)
    for _ in range(3):
        sess.run_epoch()
    states, weights, counters, fb, sh = sess.snapshot()
    assert np.array_equal(states.cpu().numpy(), g["states"])
    assert np.array_equal(weights.cpu().numpy(), g["weights"])
    assert np.array_equal(counters.cpu().numpy().view(np.uint64), g["block_counters"])
    assert fb == int(g["fb_counter"]) and sh == int(g["shuffle_counter"])


@pytest.mark.parametrize("kernel", ["count", "key"])
@pytest.mark.parametrize("K,n_docs,doc_len", [(40, 300, 60), (3, 200, 500), (2, 50, 5000)])
def test_sparse_inference_no_hit_or_class_limits(gpu, oracle, kernel, K, n_docs, doc_len):
    """Both sparse inference kernels (per-warp clause counters; key-literal
    candidates for clause counts too large for the counters) have no
    per-document buffers: thousands of
    clause postings per document (clauses over a small pool of common
    literals), more than 32 classes, documents longer than 4096 ids, empty
    clauses and empty documents -- votes and outputs equal the oracle's
    SparseClauseBank (sparse.py:123-147)."""
    rs = np.random.default_rng(K + doc_len)
    L, C = 20000, 3000
    cfg = gpu.Config(n_literals=L, n_clauses=C, n_classes=K, s=3.0, threshold=10,
                     negated_literals_enabled=False)
    bank = gpu.SparseClauseBank(cfg, candidate_literals=np.arange(L))
    pool = rs.choice(L, size=40, replace=False)
    ob = oracle.SparseOracleBank(cfg, candidates=np.arange(L))
    for j in range(C):
        if j % 97 == 0:
            lits = np.empty(0, np.int64)
        else:
            m = int(rs.integers(1, 4))
            lits = np.unique(np.concatenate([rs.choice(pool, size=m, replace=False),
                                             rs.integers(0, L, size=int(rs.integers(0, 3)))]))
        sts = rs.integers(-5, 3, size=lits.size).astype(np.int8)
        if lits.size:
            sts[0] = 0
        bank.clause_literals[j] = lits.astype(np.int64)
        bank.clause_states[j] = sts
        ob.lits[j], ob.sts[j] = lits.astype(np.int64), sts
    w = rs.integers(-9, 10, size=(C, K)).astype(np.int32)
    bank.weights[:] = w
    ob.weights = w.copy()
    docs = []
    for i in range(n_docs):
        n = 0 if i % 41 == 0 else int(rs.integers(1, doc_len))
        d = np.unique(np.concatenate([rs.choice(pool, size=int(rs.integers(0, 40)), replace=False),
                                      rs.integers(0, L, size=n)]))
        docs.append(d.astype(np.int64))
    ex = [gpu.SparseExample(d, 0) for d in docs]
    gpu._lib.call("tmb_set_option", b"sparse.infer_key", int(kernel == "key"))
    try:
        votes = bank.batch_votes(ex)
        assert np.array_equal(votes, oracle.sparse_batch_votes([ob], docs))
        from paper_2405_04212_b200.sparse_train import sparse_outputs
        outs = sparse_outputs(bank, ex[:40], gpu.EvalMode.INFERENCE)
        for i in range(40):
            assert np.array_equal(outs[i], ob.clause_outputs(docs[i], False)), i
    finally:
        gpu._lib.call("tmb_set_option", b"sparse.infer_key", 0)


def _sparse_docs(rs, n_docs, vocab, lo, hi, planted):
    docs, labels = [], []
    for i in range(n_docs):
        n = int(rs.integers(lo, hi))
        d = np.unique(rs.integers(0, vocab, size=n))
        docs.append(d.astype(np.int64))
        labels.append(int(np.isin(d, planted).sum() % 2))
    return docs, np.array(labels)


def _sparse_vs_oracle(gpu, oracle, cfg, docs, labels, n_epochs, slab=None):
    from paper_2405_04212_b200.sparse_train import SparseTrainSession
    ip = np.zeros(len(docs) + 1, dtype=np.int64)
    np.cumsum([len(d) for d in docs], out=ip[1:])
    sess = SparseTrainSession(cfg, ip, np.concatenate(docs).astype(np.int32), labels, slab=slab)
    for _ in range(n_epochs):
        sess.run_epoch_growing()
    m = sess.model()
    banks, bctr, _ = oracle.sparse_train(cfg, docs, labels, n_epochs=n_epochs)
    ob = banks[0]
    assert np.array_equal(m.weights, ob.weights)
    for j in range(cfg.n_clauses):
        assert np.array_equal(m.clause_literals[j], ob.lits[j]), j
        assert np.array_equal(m.clause_states[j], ob.sts[j]), j
    return sess


def test_sparse_capacity_none_large_candidate_set(gpu, oracle):
    """sparse_capacity=None (the reference default) with 2500+ candidates:
    a Type II event stores every non-active candidate (sparse.py:192-210), so
    lists far exceed the initial 1024-pair slab; the session sizes the slab
    from the candidate set and the model equals the oracle's."""
    rs = np.random.default_rng(5)
    docs, labels = _sparse_docs(rs, 60, 3000, 20, 80, np.arange(0, 3000, 7))
    cfg = gpu.Config(n_literals=3000, n_clauses=12, n_classes=2, s=3.0, threshold=8, seed=2,
                     negated_literals_enabled=False)
    sess = _sparse_vs_oracle(gpu, oracle, cfg, docs, labels, 2)
    assert sess.engine.slab > 1024
    assert max(len(a) for a in sess.model().clause_literals) > 1024


def test_sparse_slab_grows_and_replays(gpu, oracle):
    """A slab too small for the lists the run builds: the epoch is replayed on
    a larger slab and the model equals the oracle's."""
    rs = np.random.default_rng(6)
    docs, labels = _sparse_docs(rs, 80, 400, 10, 40, np.arange(0, 400, 5))
    cfg = gpu.Config(n_literals=400, n_clauses=10, n_classes=2, s=3.0, threshold=8, seed=3,
                     negated_literals_enabled=False, sparse_capacity=12)
    sess = _sparse_vs_oracle(gpu, oracle, cfg, docs, labels, 2, slab=16)
    assert sess.engine.slab > 16


def test_sparse_train_documents_longer_than_stage(gpu, oracle):
    """Training documents with more than 4096 active literals (read in place
    from the CSR row instead of the shared-memory stage)."""
    rs = np.random.default_rng(7)
    docs, labels = _sparse_docs(rs, 12, 30000, 4500, 9000, np.arange(0, 30000, 3))
    assert max(len(d) for d in docs) > 4096
    cfg = gpu.Config(n_literals=30000, n_clauses=8, n_classes=2, s=3.0, threshold=8, seed=4,
                     negated_literals_enabled=False, sparse_capacity=16)
    _sparse_vs_oracle(gpu, oracle, cfg, docs, labels, 2)


def test_train_rejects_non_binary_features(gpu):
    """The device packs literal bits; non-0/1 training bytes raise DataError
    (as the inference and explain paths reject them)."""
    cfg = gpu.Config(n_literals=4, n_clauses=4, n_classes=2, s=3.0, threshold=5)
    x = np.array([[0, 1, 2, 0], [1, 0, 0, 1]], dtype=np.uint8)
    with pytest.raises(gpu.DataError):
        gpu.train(cfg, (x, np.array([0, 1])), n_epochs=1)


@pytest.mark.parametrize("F,C,K,nb,boost,budget", [
    (12, 10, 2, 1, False, None), (6, 8, 2, 2, True, 3), (500, 32, 10, 3, False, 40),
    (31, 17, 4, 5, True, None)])
def test_single_warp_trainer_vs_oracle(gpu, oracle, F, C, K, nb, boost, budget):
    """Tiny banks (C, K <= 32, literal rows <= 32 words) run on
    k_train_tiny (one warp per clause, one block barrier per example) or,
    with train.tiny 0, on the single-warp k_train_warp; both, the generic
    one-CTA cluster kernel (warp_kernel=False) and the oracle give the same
    model, counters and statistics."""
    rs = np.random.default_rng(F + C + K)
    x = rs.integers(0, 2, size=(400, F)).astype(np.uint8)
    y = ((x[:, 0] ^ x[:, 1]) + 2 * x[:, 2] * (K > 2)).astype(np.int64) % K
    cfg = gpu.Config(n_literals=F, n_clauses=C, n_classes=K, s=2.7, threshold=9, seed=C,
                     n_blocks=nb, boost_true_positive=boost, n_literal_budget=budget)
    ost, _ = oracle.train(cfg, x, y, 3)
    stats = []
    try:
        for kernel in ("k_train_tiny", "k_train_warp", None):
            gpu._lib.call("tmb_set_option", b"train.tiny", int(kernel == "k_train_tiny"))
            sess = gpu.DenseTrainSession(cfg, x, y, warp_kernel=kernel is not None)
            if kernel:
                assert sess.launch["kernel"] == kernel
                assert sess.launch["threads"] == (32 * C if kernel == "k_train_tiny" else 32)
            for _ in range(3):
                sess.run_epoch()
            m = sess.model()
            assert np.array_equal(m.states, ost.states), kernel
            assert np.array_equal(m.weights, ost.weights), kernel
            assert np.array_equal(sess.block_counters.cpu().numpy().view(np.uint64),
                                  ost.block_counters), kernel
            stats.append(sess.stats_dict())
    finally:
        gpu._lib.call("tmb_set_option", b"train.tiny", 1)
    assert stats[0] == stats[1] == stats[2]


@pytest.mark.parametrize("window,n_cta,n_train", [(1, 148, 700), (5, 148, 703), (16, 37, 1500),
                                                  (16, 20, 333), (7, 148, 5)])
def test_speculative_windows_vs_oracle(gpu, oracle, window, n_cta, n_train):
    """k_train_spec (one exchange per window of up to `window` steps, kept
    per-step sums corrected by the work list) against the oracle and against
    k_train_fast (train.spec_window=0): models, block counters and the
    per-step trace (negative class, both class sums, events) are identical --
    window sizes that do not divide the run, runs shorter than one window,
    more than 32 clauses per CTA (multi-word output bitsets)."""
    import torch
    (tx, ty), _ = gpu.datasets.mnist_shaped(n_train=n_train, n_test=10, data_seed=6)
    cfg = gpu.Config(**gpu.datasets.mnist_shaped_config_kwargs(seed=4))
    ost, _ = oracle.train(cfg, tx, ty, 2)
    got = {}
    try:
        for w in (window, 0):
            gpu._lib.call("tmb_set_option", b"train.spec_window", w)
            sess = gpu.DenseTrainSession(cfg, tx, ty, n_cta=n_cta)
            trace = torch.zeros((2, n_train, 4), dtype=torch.int64, device="cuda")
            for e in range(2):
                gpu._lib.call("tmb_trainer_set_trace", sess._h, trace[e].data_ptr())
                sess.run_epoch()
            m = sess.model()
            assert np.array_equal(m.states, ost.states), w
            assert np.array_equal(m.weights, ost.weights), w
            assert np.array_equal(sess.block_counters.cpu().numpy().view(np.uint64),
                                  ost.block_counters), w
            got[w] = trace.cpu().numpy()
    finally:
        gpu._lib.call("tmb_set_option", b"train.spec_window", 16)
    assert np.array_equal(got[window], got[0])
    assert got[0][:, :, 3].sum() > 0  # the run has events


@pytest.mark.parametrize("n_blocks,keys", [(5, True), (1, False), (3, False)])
def test_hbm_state_trainer_1024_threads_vs_oracle(gpu, oracle, n_blocks, keys):
    """The HBM-state generic grid trainer built for 1024-thread CTAs
    (train.hbm_threads=1024: twice the warps, two state words in flight per
    thread, grid-balanced SIMD feedback) against the oracle (one block with
    16-bit flag keys takes the fast trainers instead)."""
    (tx, ty), _ = gpu.datasets.mnist_shaped(n_train=800, n_test=10, data_seed=8)
    kw = gpu.datasets.mnist_shaped_config_kwargs(seed=12)
    kw["n_blocks"] = n_blocks
    cfg = gpu.Config(**kw)
    try:
        gpu._lib.call("tmb_set_option", b"train.hbm_threads", 1024)
        sess = gpu.DenseTrainSession(cfg, tx, ty, states_in_hbm=True, flag_keys=keys)
        assert sess.launch["threads"] == 1024 and not sess.launch["states_in_smem"]
        for _ in range(2):
            sess.run_epoch()
        m = sess.model()
    finally:
        gpu._lib.call("tmb_set_option", b"train.hbm_threads", 1024)
    ost, _ = oracle.train(cfg, tx, ty, 2)
    assert np.array_equal(m.states, ost.states)
    assert np.array_equal(m.weights, ost.weights)
    assert np.array_equal(sess.block_counters.cpu().numpy().view(np.uint64), ost.block_counters)


@pytest.mark.parametrize("weights", [0, 1 | (50 << 8) | (50 << 16), 255 | (1 << 8) | (255 << 16)])
def test_balanced_feedback_weighted_split_vs_oracle(gpu, oracle, weights):
    """HBM-state grid trainer, balanced feedback: the union of the CTAs' work
    lists is cut at cost-weighted positions (train.gbal_weights).  Whatever
    the weights -- unweighted, Type II nearly free, silent Type I rows 255
    times cheaper than firing ones (a share of cheap rows then holds more work
    items than the cmax + 4 staging buffer: the chunked path) -- every quad is
    applied exactly once, so the model equals the oracle's.  First epoch of the MNIST-shaped config: every step is
    non-empty with ~2 000 events."""
    (tx, ty), _ = gpu.datasets.mnist_shaped(n_train=240, n_test=10, data_seed=11)
    cfg = gpu.Config(**gpu.datasets.mnist_shaped_config_kwargs(seed=15))
    try:
        gpu._lib.call("tmb_set_option", b"train.gbal_weights", weights)
        sess = gpu.DenseTrainSession(cfg, tx, ty, states_in_hbm=True, flag_keys=False)
        assert sess.launch["kernel"] == "k_train (grid)" and not sess.launch["states_in_smem"]
        sess.run_epoch()
        m = sess.model()
        stats = sess.stats_dict()
    finally:
        gpu._lib.call("tmb_set_option", b"train.gbal_weights", 2 | (5 << 8) | (6 << 16))
    ost, _ = oracle.train(cfg, tx, ty, 1)
    assert np.array_equal(m.states, ost.states)
    assert np.array_equal(m.weights, ost.weights)
    assert np.array_equal(sess.block_counters.cpu().numpy().view(np.uint64), ost.block_counters)
    assert stats["events"] > 100 * len(ty)


def test_speculative_trainer_large_threshold_vs_oracle(gpu, oracle):
    """k_train_spec with T > 8192 (no threshold table in shared memory: the
    window decision computes the exact thresholds in f64) against the
    oracle."""
    (tx, ty), _ = gpu.datasets.mnist_shaped(n_train=600, n_test=10, data_seed=9)
    kw = gpu.datasets.mnist_shaped_config_kwargs(seed=13)
    kw["threshold"] = 9000
    cfg = gpu.Config(**kw)
    sess = gpu.DenseTrainSession(cfg, tx, ty)
    assert sess.launch["kernel"] == "k_train_spec"
    for _ in range(2):
        sess.run_epoch()
    m = sess.model()
    ost, _ = oracle.train(cfg, tx, ty, 2)
    assert np.array_equal(m.states, ost.states)
    assert np.array_equal(m.weights, ost.weights)
