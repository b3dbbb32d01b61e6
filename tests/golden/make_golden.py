"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba python tests/golden/make_golden.py

It imports the unmodified reference package ``tsetlinkit`` from
/root/reference/pkg/src (numba backend, its default) and writes small
``.npz`` fixtures next to this script.  The fixtures travel with the repo; the
GPU box never reads /root/reference.  Each fixture records which reference
function produced it.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")

import tsetlinkit as tk  # noqa: E402
from tsetlinkit import kernels  # noqa: E402
from tsetlinkit.core import (RngStream, derive_stream, stream_u01_block,  # noqa: E402
                             stream_u64, stream_u64_block)
from tsetlinkit.executor import shuffle_permutation  # noqa: E402
from tsetlinkit.feedback import sample_updates, update_probabilities  # noqa: E402
from tsetlinkit.predictor import compile_ruleset, predict_and_explain, rule_votes  # noqa: E402
from tsetlinkit.sparse import SparseDataset, SparseExample  # noqa: E402

from paper_2405_04212_b200 import datasets  # noqa: E402

assert kernels.BACKEND_NAME == "numba", kernels.BACKEND_NAME


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def rng_fixture():
    rs = np.random.default_rng(0)
    seeds = rs.integers(0, 2**63, size=24, dtype=np.uint64)
    seeds = np.concatenate([seeds, np.array([0, 7, 2**64 - 1], dtype=np.uint64)])
    idx = np.array([0, 1, 3, 5, 0xFEED, 0xD157, 2**32, 2**40 + 3], dtype=np.uint64)
    derived = np.array([[derive_stream(int(s), int(i)) for i in idx] for s in seeds],
                       dtype=np.uint64)
    starts = np.array([0, 17, 2**32, 2**33 + 5, 2**64 - 3], dtype=np.uint64)
    blocks = np.stack([stream_u64_block(int(derived[0, 0]), int(st), 64) for st in starts])
    u01 = np.stack([stream_u01_block(int(derived[1, 1]), int(st), 64) for st in starts])
    save("rng", seeds=seeds, idx=idx, derived=derived, starts=starts,
         block_seed=np.uint64(derived[0, 0]), blocks=blocks,
         u01_seed=np.uint64(derived[1, 1]), u01=u01,
         known=np.array([derive_stream(7, 3), stream_u64(derive_stream(7, 3), 0)],
                        dtype=np.uint64))


def kernel_fixture():
    """kernels.clause_outputs / clause_outputs_batch / bank_feedback on
    random banks (mirrors pkg/tests/test_kernels.py shapes, larger)."""
    rs = np.random.default_rng(1)
    out = {}
    cases = []
    for t in range(40):
        C = int(rs.integers(1, 40))
        P = int(rs.integers(1, 130))
        K = int(rs.integers(2, 6))
        lo, hi = sorted(rs.integers(-30, 30, size=2))
        states = rs.integers(-20, 20, size=(C, P)).astype(np.int8)
        if t % 3 == 0:  # sparse includes, more firing
            states = np.where(rs.random((C, P)) < 0.05, 0, -1).astype(np.int8)
        weights = rs.integers(-6, 6, size=(C, K)).astype(np.int32)
        lits = rs.integers(0, 2, size=P).astype(np.uint8)
        budget = int(rs.integers(1, P + 1))
        outputs = rs.integers(0, 2, size=C).astype(np.uint8)
        ut = rs.random(C) < 0.6
        un = rs.random(C) < 0.6
        label = int(rs.integers(0, K))
        negative = int((label + 1 + rs.integers(0, K - 1)) % K)
        s = float(rs.uniform(1.01, 12.0))
        boost = bool(t % 4 == 1)
        smin, smax = int(min(lo, -1)), int(max(hi, 0))
        smin, smax = max(smin, -127), min(smax, 127)
        states = np.clip(states, smin, smax).astype(np.int8)
        seed = derive_stream(int(rs.integers(0, 2**62)), int(rs.integers(0, 8)))
        counter = int(rs.integers(0, 2**33)) if t % 5 == 0 else int(rs.integers(0, 1000))
        if t == 7:
            counter = 2**32 - 2  # window base wraps mod 2^64 after 2^32 events
        o_tr = kernels.clause_outputs(states, lits, True, budget)
        o_inf = kernels.clause_outputs(states, lits, False, budget)
        x_lit = rs.integers(0, 2, size=(16, P)).astype(np.uint8)
        b_tr = kernels.clause_outputs_batch(states, x_lit, True, budget)
        b_inf = kernels.clause_outputs_batch(states, x_lit, False, budget)
        st2, w2 = states.copy(), weights.copy()
        new_counter = kernels.bank_feedback(st2, w2, lits, outputs, label, negative, ut, un,
                                            s, boost, smin, smax, np.uint64(seed),
                                            np.uint64(counter))
        pre = f"c{t}_"
        out.update({pre + "states": states, pre + "weights": weights, pre + "lits": lits,
                    pre + "x_lit": x_lit, pre + "outputs": outputs, pre + "ut": ut,
                    pre + "un": un, pre + "o_tr": o_tr, pre + "o_inf": o_inf,
                    pre + "b_tr": b_tr, pre + "b_inf": b_inf, pre + "st_after": st2,
                    pre + "w_after": w2,
                    pre + "scalars": np.array([label, negative, int(boost), smin, smax,
                                               budget], dtype=np.int64),
                    pre + "s": np.float64(s), pre + "seed": np.uint64(seed),
                    pre + "counter": np.uint64(counter),
                    pre + "new_counter": np.uint64(int(new_counter))})
        cases.append(t)
    out["n_cases"] = np.int64(len(cases))
    save("kernels", **out)


def feedback_fixture():
    rs = np.random.default_rng(2)
    rows = []
    for t in range(200):
        K = int(rs.integers(2, 12))
        T = int(rs.integers(1, 20000))
        votes = rs.integers(-3 * T, 3 * T, size=K).astype(np.int64)
        label = int(rs.integers(0, K))
        seed = int(rs.integers(0, 2**62))
        ctr = int(rs.integers(0, 10**6))
        rng = RngStream(derive_stream(seed, 0xFEED), ctr)
        d = update_probabilities(votes, label, T, rng)
        C = 37
        ut, un = sample_updates(d, C, rng)
        rows.append((K, T, label, seed, ctr, votes, d.negative_class, d.p_target,
                     d.p_negative, ut, un, rng.counter))
    save("feedback",
         K=np.array([r[0] for r in rows]), T=np.array([r[1] for r in rows]),
         label=np.array([r[2] for r in rows]),
         seed=np.array([r[3] for r in rows], dtype=np.uint64),
         ctr=np.array([r[4] for r in rows], dtype=np.uint64),
         votes=np.stack([np.pad(r[5], (0, 12 - r[0])) for r in rows]),
         negative=np.array([r[6] for r in rows]),
         p_target=np.array([r[7] for r in rows]), p_negative=np.array([r[8] for r in rows]),
         ut=np.stack([r[9] for r in rows]), un=np.stack([r[10] for r in rows]),
         ctr_after=np.array([r[11] for r in rows], dtype=np.uint64))
    perms = {}
    for n in (0, 1, 2, 5, 100, 1000):
        rng = RngStream.derive(5, 0xD157)
        p1 = shuffle_permutation(n, rng)
        p2 = shuffle_permutation(n, rng)
        perms[f"n{n}_a"] = p1
        perms[f"n{n}_b"] = p2
        perms[f"n{n}_ctr"] = np.uint64(rng.counter)
    save("shuffle", **perms)


def train_fixture():
    """Full executor.train runs: final states / weights / accuracies."""
    out = {}
    # paper-listing XOR config (pkg/tests/conftest.py:14-27 shapes, our data)
    rs = np.random.default_rng(1234)
    x = rs.integers(0, 2, size=(400, 6)).astype(np.uint8)
    y = (x[:, 0] ^ x[:, 1]).astype(np.int64)
    ex, ey = x[300:], y[300:]
    x, y = x[:300], y[:300]
    out["xor_x"], out["xor_y"], out["xor_ex"], out["xor_ey"] = x, y, ex, ey
    runs = [dict(seed=42, n_blocks=1), dict(seed=3, n_blocks=3),
            dict(seed=9, n_blocks=1, boost_true_positive=True),
            dict(seed=11, n_blocks=2, state_min=-10, state_max=9, init_state=-3)]
    for i, kw in enumerate(runs):
        cfg = tk.Config(n_literals=6, n_clauses=8, n_classes=2, s=1.9, threshold=11,
                        n_literal_budget=3, **kw)
        run = tk.train(cfg, (x, y), (ex, ey), n_epochs=3)
        out[f"xor{i}_states"] = run.model.states
        out[f"xor{i}_weights"] = run.model.weights
        out[f"xor{i}_acc"] = np.array([m.accuracy for m in run.epoch_metrics])
        out[f"xor{i}_cfg"] = np.array([kw.get("seed"), kw.get("n_blocks"),
                                       int(kw.get("boost_true_positive", False)),
                                       kw.get("state_min", -127), kw.get("state_max", 127),
                                       kw.get("init_state", -1)], dtype=np.int64)
    # multi-class, wider: 3 classes, 20 features, 30 clauses, 2 blocks
    rs = np.random.default_rng(99)
    x = rs.integers(0, 2, size=(500, 20)).astype(np.uint8)
    y = ((x[:, 0] + 2 * x[:, 3] + x[:, 7]) % 3).astype(np.int64)
    cfg = tk.Config(n_literals=20, n_clauses=30, n_classes=3, s=3.0, threshold=15,
                    seed=77, n_blocks=2)
    run = tk.train(cfg, (x[:400], y[:400]), (x[400:], y[400:]), n_epochs=2)
    out["mc_x"], out["mc_y"] = x, y
    out["mc_states"], out["mc_weights"] = run.model.states, run.model.weights
    out["mc_acc"] = np.array([m.accuracy for m in run.epoch_metrics])
    votes = tk.executor.dataset_votes(run.model, (x[400:], y[400:]))
    out["mc_votes"] = votes
    save("train_small", **out)


def noisy_xor_fixture():
    """BASELINE config 1 (Noisy-XOR), 20 epochs, model seeds 0-4."""
    (tx, ty), (ex, ey) = datasets.noisy_xor()
    out = {"tx": tx, "ty": ty, "ex": ex, "ey": ey}
    for seed in range(5):
        cfg = tk.Config(**datasets.noisy_xor_config_kwargs(seed))
        run = tk.train(cfg, (tx, ty), (ex, ey), n_epochs=20)
        out[f"s{seed}_states"] = run.model.states
        out[f"s{seed}_weights"] = run.model.weights
        out[f"s{seed}_acc"] = np.array([m.accuracy for m in run.epoch_metrics])
        print("noisy-xor seed", seed, "final acc", run.epoch_metrics[-1].accuracy)
    save("noisy_xor", **out)


def mnist_prefix_fixture():
    """BASELINE config 2 shape (2000 clauses, 1568 positions, K=10, T=5000,
    s=10) on a 300-example prefix of the synthetic MNIST-shaped set."""
    (tx, ty), (ex, ey) = datasets.mnist_shaped(n_train=600, n_test=200)
    cfg = tk.Config(**datasets.mnist_shaped_config_kwargs(seed=1))
    run = tk.train(cfg, (tx[:300], ty[:300]), (ex, ey), n_epochs=1)
    votes = tk.executor.dataset_votes(run.model, (ex, ey))
    save("mnist_prefix", tx=tx[:300], ty=ty[:300], ex=ex, ey=ey,
         states=run.model.states, weights=run.model.weights,
         acc=np.array([m.accuracy for m in run.epoch_metrics]), votes=votes)


def predictor_fixture():
    rs = np.random.default_rng(5)
    x = rs.integers(0, 2, size=(200, 9)).astype(np.uint8)
    y = (x[:, 0] & x[:, 1] | x[:, 4]).astype(np.int64)
    cfg = tk.Config(n_literals=9, n_clauses=16, n_classes=2, s=3.0, threshold=8, seed=4,
                    n_blocks=2)
    model = tk.train(cfg, (x, y), n_epochs=3).model
    rs_ = compile_ruleset(model)
    allx = np.array(np.meshgrid(*[[0, 1]] * 9, indexing="ij")).reshape(9, -1).T.astype(np.uint8)
    votes = np.stack([rule_votes(rs_, r) for r in allx])
    lit_scores, feat_scores, preds = [], [], []
    for r in allx[:64]:
        p, e = predict_and_explain(rs_, r, level="literal")
        _, f = predict_and_explain(rs_, r, level="feature")
        lit_scores.append(e.scores)
        feat_scores.append(f.scores)
        preds.append(p)
    inc_ptr = np.cumsum([0] + [len(i) for i in rs_.includes]).astype(np.int64)
    inc_idx = (np.concatenate(rs_.includes).astype(np.int64) if rs_.n_rules
               else np.zeros(0, np.int64))
    save("predictor", states=model.states, weights=model.weights, allx=allx, votes=votes,
         rs_weights=rs_.weights, inc_ptr=inc_ptr, inc_idx=inc_idx,
         lit_scores=np.stack(lit_scores), feat_scores=np.stack(feat_scores),
         preds=np.array(preds))


def sparse_fixture():
    """SparseClauseBank training incl. capacity rule and candidates domain."""
    rs = np.random.default_rng(11)
    n_lit = 60
    support = np.sort(rs.choice(n_lit, size=40, replace=False))
    examples = []
    for _ in range(120):
        k = int(rs.integers(3, 12))
        active = np.sort(rs.choice(support, size=k, replace=False)).astype(np.int64)
        examples.append(SparseExample(active, int(active[0] % 2)))
    ds = SparseDataset(n_lit, examples)
    out = {}
    ptr = np.cumsum([0] + [len(e.active) for e in examples]).astype(np.int64)
    out["indptr"] = ptr
    out["indices"] = np.concatenate([e.active for e in examples]).astype(np.int64)
    out["labels"] = ds.labels
    runs = [dict(seed=1, sparse_capacity=None, sparse_floor=-15, n_blocks=1),
            dict(seed=2, sparse_capacity=4, sparse_floor=-6, n_blocks=1),
            dict(seed=3, sparse_capacity=2, sparse_floor=-4, n_blocks=3, s=1.5)]
    for i, kw in enumerate(runs):
        kw = dict(kw)
        s = kw.pop("s", 2.5)
        cfg = tk.Config(n_literals=n_lit, n_clauses=10, n_classes=2, s=s, threshold=6,
                        negated_literals_enabled=False, **kw)
        model = tk.train(cfg, ds, n_epochs=2).model
        lens = np.array([a.size for a in model.clause_literals], dtype=np.int64)
        out[f"r{i}_lens"] = lens
        out[f"r{i}_lits"] = (np.concatenate(model.clause_literals)
                             if lens.sum() else np.zeros(0, np.int64))
        out[f"r{i}_sts"] = (np.concatenate(model.clause_states)
                            if lens.sum() else np.zeros(0, np.int8))
        out[f"r{i}_weights"] = model.weights
        out[f"r{i}_votes"] = model.batch_votes(examples)
        out[f"r{i}_cfg"] = np.array([kw["seed"], -1 if kw["sparse_capacity"] is None
                                     else kw["sparse_capacity"], kw["sparse_floor"],
                                     kw["n_blocks"]], dtype=np.int64)
        out[f"r{i}_s"] = np.float64(s)
    save("sparse", **out)


def tuning_fixture():
    """tuning.stratified_kfold assignments and a cross_validate report."""
    from tsetlinkit.tuning import cross_validate, stratified_kfold
    rs = np.random.default_rng(17)
    out = {}
    for t in range(12):
        k = int(rs.integers(2, 6))
        labels = rs.integers(0, 3, size=int(rs.integers(3 * k + 3, 90)))
        while np.bincount(labels, minlength=3).min() < k:
            labels = rs.integers(0, 3, size=labels.size)
        out[f"t{t}_labels"] = labels
        out[f"t{t}_k"] = np.int64(k)
        out[f"t{t}_folds"] = stratified_kfold(labels, k, seed=t)
    x = rs.integers(0, 2, size=(240, 6)).astype(np.uint8)
    y = (x[:, 0] ^ x[:, 1]).astype(np.int64)
    cfg = tk.Config(n_literals=6, n_clauses=8, n_classes=2, s=1.9, threshold=11,
                    n_literal_budget=3, seed=0)
    rep = cross_validate(cfg, (x, y), 4, 2, seed=9)
    out["cv_x"], out["cv_y"] = x, y
    out["cv_acc"] = np.array(rep.fold_accuracies)
    out["cv_folds"] = rep.fold_assignments
    save("tuning", **out)


def search_fixture():
    """tuning.SearchSpace parse / sample draws and a random_search ranking
    (holdout split and cv_k variants) on a small XOR-shaped problem."""
    from tsetlinkit.tuning import SearchSpace, random_search
    from tsetlinkit.core import RngStream as RS
    text = ("# comment line\n"
            "s loguniform 1.5 6.0\n"
            "threshold int 5 25\n"
            "n_clauses cat 6,8,10\n"
            "boost_true_positive cat true,false\n"
            "state_max uniform 50 127\n")
    space = SearchSpace.parse(text)
    rng = RS.derive(123, 0x5EA7)
    draws = [space.sample(rng) for _ in range(40)]
    out = {"space_text": np.frombuffer(text.encode(), dtype=np.uint8)}
    for name in ("s", "threshold", "n_clauses", "boost_true_positive", "state_max"):
        out["draw_" + name] = np.array([d[name] for d in draws], dtype=np.float64)
    rs = np.random.default_rng(23)
    x = rs.integers(0, 2, size=(200, 6)).astype(np.uint8)
    y = (x[:, 0] ^ x[:, 1]).astype(np.int64)
    base = tk.Config(n_literals=6, n_clauses=8, n_classes=2, s=2.0, threshold=10, seed=0)
    small = SearchSpace.parse("s uniform 1.5 4.0\nthreshold int 5 20\nn_clauses cat 6,10")
    for tag, kw in (("hold", dict()), ("cv", dict(cv_k=3))):
        trials = random_search(small, base, (x, y), n_trials=5, n_epochs=2, seed=31, **kw)
        out[tag + "_index"] = np.array([t.index for t in trials], dtype=np.int64)
        out[tag + "_acc"] = np.array([t.accuracy for t in trials], dtype=np.float64)
        out[tag + "_s"] = np.array([t.config.s for t in trials], dtype=np.float64)
        out[tag + "_T"] = np.array([t.config.threshold for t in trials], dtype=np.int64)
        out[tag + "_C"] = np.array([t.config.n_clauses for t in trials], dtype=np.int64)
    out["x"], out["y"] = x, y
    save("search", **out)


def modelio_fixture():
    """GTM1 model files written by the reference (dataio.save_model) for a
    dense bank, a sparse bank and a rule set, with the models' contents."""
    import io
    import tempfile

    from tsetlinkit.dataio import save_model
    out = {}
    rs = np.random.default_rng(23)
    x = rs.integers(0, 2, size=(150, 7)).astype(np.uint8)
    y = (x[:, 1] | x[:, 3]).astype(np.int64)
    cfg = tk.Config(n_literals=7, n_clauses=6, n_classes=2, s=2.5, threshold=5,
                    n_literal_budget=4, seed=8, boost_true_positive=True)
    dense = tk.train(cfg, (x, y), n_epochs=2).model
    ex = [SparseExample(np.sort(rs.choice(40, size=int(rs.integers(2, 9)), replace=False))
                        .astype(np.int64), int(rs.integers(0, 2))) for _ in range(80)]
    scfg = tk.Config(n_literals=40, n_clauses=5, n_classes=2, s=2.0, threshold=4, seed=2,
                     negated_literals_enabled=False, sparse_capacity=3, sparse_floor=-5)
    sparse = tk.train(scfg, SparseDataset(40, ex), n_epochs=2).model
    rset = compile_ruleset(dense)
    with tempfile.TemporaryDirectory() as td:
        for name, m in (("dense", dense), ("sparse", sparse), ("ruleset", rset)):
            path = os.path.join(td, name + ".gtm")
            save_model(m, path)
            out[name + "_bytes"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
    out["dense_states"], out["dense_weights"] = dense.states, dense.weights
    lens = np.array([a.size for a in sparse.clause_literals], dtype=np.int64)
    out["sparse_lens"] = lens
    out["sparse_lits"] = np.concatenate(sparse.clause_literals) if lens.sum() else np.zeros(0, np.int64)
    out["sparse_sts"] = np.concatenate(sparse.clause_states) if lens.sum() else np.zeros(0, np.int8)
    out["sparse_weights"] = sparse.weights
    save("modelio", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["rng", "kernels", "feedback", "train", "noisy_xor", "mnist",
                             "predictor", "sparse", "tuning", "modelio", "search"]
    table = {"rng": rng_fixture, "kernels": kernel_fixture, "feedback": feedback_fixture,
             "train": train_fixture, "noisy_xor": noisy_xor_fixture,
             "mnist": mnist_prefix_fixture, "predictor": predictor_fixture,
             "sparse": sparse_fixture, "tuning": tuning_fixture, "modelio": modelio_fixture,
             "search": search_fixture}
    for name in which:
        table[name]()
