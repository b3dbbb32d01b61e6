"""CPU-only tests: host logic mirrored from the reference, the C ABI library
loads and exports every declared symbol, and compute fails loudly without a
GPU (no silent CPU fallback)."""

import os
import re

import numpy as np
import pytest

from conftest import REPO, golden

import paper_2405_04212_b200 as tmb
from paper_2405_04212_b200 import _lib
from paper_2405_04212_b200.core import RngStream, derive_stream, stream_u64


def header_functions():
    src = open(os.path.join(REPO, "include", "tsetlin_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tmbh?_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n
        assert n in _lib.SIGNATURES, f"{n} missing from the ctypes signature table"
    assert lib.tmb_abi_version() == 1


def test_host_rng_known_answers():
    assert derive_stream(7, 3) == 0x2C7D03C103AFD766
    assert stream_u64(derive_stream(7, 3), 0) == 0xAB6B7B0CE9C8A6AB
    assert _lib.load().tmb_derive_stream(7, 3) == 0x2C7D03C103AFD766
    g = golden("rng")
    for i, s in enumerate(g["seeds"]):
        for j, idx in enumerate(g["idx"]):
            assert derive_stream(int(s), int(idx)) == int(g["derived"][i, j])
    for r, st in enumerate(g["starts"]):
        assert np.array_equal(tmb.stream_u64_block(int(g["block_seed"]), int(st), 64),
                              g["blocks"][r])


def test_rng_cursor():
    rng = RngStream.derive(3, 2)
    a, b = rng.next_u01(), rng.next_u01()
    assert rng.counter == 2 and a == tmb.stream_u01(rng.stream_seed, 0)
    rng = RngStream.derive(3, 2)
    assert rng.take_window() == 0 and rng.take_window() == 2 ** 32


def test_shuffle_matches_reference():
    g = golden("shuffle")
    for n in (0, 1, 2, 5, 100, 1000):
        rng = RngStream.derive(5, 0xD157)
        a = tmb.shuffle_permutation(n, rng)
        b = tmb.shuffle_permutation(n, rng)
        assert np.array_equal(a, g[f"n{n}_a"]) and np.array_equal(b, g[f"n{n}_b"])
        assert rng.counter == int(g[f"n{n}_ctr"])


def test_partition_clauses():
    assert tmb.partition_clauses(8, 4) == [range(0, 2), range(2, 4), range(4, 6), range(6, 8)]
    assert sorted(len(r) for r in tmb.partition_clauses(5, 2)) == [2, 3]
    with pytest.raises(ValueError):
        tmb.partition_clauses(3, 4)


@pytest.mark.parametrize("kw", [dict(n_literals=0), dict(n_classes=1), dict(s=1.0),
                                dict(threshold=0), dict(n_literal_budget=0),
                                dict(init_state=0), dict(state_max=128), dict(n_blocks=9),
                                dict(sparse_floor=0), dict(sparse_capacity=0), dict(seed=-1)])
def test_config_invariants(kw):
    base = dict(n_literals=4, n_clauses=8, n_classes=2, s=2.0, threshold=5)
    base.update(kw)
    with pytest.raises(tmb.ConfigError):
        tmb.Config(**base)


def test_config_derived():
    c = tmb.Config(n_literals=4, n_clauses=8, n_classes=2, s=2.0, threshold=5,
                   n_literal_budget=100)
    assert c.n_literal_positions == 8 and c.effective_budget == 8
    assert c.with_overrides(negated_literals_enabled=False).n_literal_positions == 4
    cfg = tmb.Config(n_literals=5_000_000, n_clauses=2000, n_classes=10, s=10.0, threshold=100)
    assert tmb.dense_state_bytes(cfg) == 2 * 10 ** 10  # PAPER.md:124-125 (18.6 GiB)


def test_update_probabilities_host_matches_reference():
    g = golden("feedback")
    for i in range(g["K"].shape[0]):
        K, T, label = int(g["K"][i]), int(g["T"][i]), int(g["label"][i])
        rng = RngStream(derive_stream(int(g["seed"][i]), 0xFEED), int(g["ctr"][i]))
        d = tmb.update_probabilities(g["votes"][i, :K], label, T, rng)
        assert d.negative_class == int(g["negative"][i])
        assert d.p_target == g["p_target"][i] and d.p_negative == g["p_negative"][i]
    assert tmb.clip_votes(30, 11) == 11 and tmb.clip_votes(-30, 11) == -11


def test_data_validation_before_device():
    cfg = tmb.Config(n_literals=6, n_clauses=8, n_classes=2, s=1.9, threshold=11)
    with pytest.raises(tmb.DataError):
        tmb.train(cfg, (np.zeros((4, 5), np.uint8), np.zeros(4, np.int64)))
    with pytest.raises(tmb.DataError):
        tmb.train(cfg, (np.zeros((4, 6), np.uint8), np.array([0, 1, 2, 0])))
    with pytest.raises(tmb.DataError):
        tmb.train(cfg, (np.zeros((0, 6), np.uint8), np.zeros(0, np.int64)))
    with pytest.raises(ValueError):
        tmb.train(cfg, (np.zeros((4, 6), np.uint8), np.zeros(4, np.int64)), n_jobs=0)


def test_sparse_example_validation():
    with pytest.raises(tmb.ContractViolation):
        tmb.SparseExample(np.array([5, 2]), 0)
    with pytest.raises(tmb.ContractViolation):
        tmb.SparseExample(np.array([2, 2, 5]), 0)
    with pytest.raises(tmb.ContractViolation):
        tmb.SparseExample(np.array([2, 50]), 0).check_range(12)


def test_compute_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(_lib.TmbError):
        tmb.kernels.clause_outputs(np.zeros((2, 4), np.int8), np.zeros(4, np.uint8), True, 4)
    cfg = tmb.Config(n_literals=6, n_clauses=8, n_classes=2, s=1.9, threshold=11)
    with pytest.raises(_lib.TmbError):
        tmb.train(cfg, (np.zeros((4, 6), np.uint8), np.zeros(4, np.int64)))


def test_datasets_shapes():
    (tx, ty), (ex, ey) = tmb.datasets.noisy_xor()
    assert tx.shape == (5000, 12) and ex.shape == (5000, 12)
    assert int((ty != (tx[:, 0] ^ tx[:, 1])).sum()) == 2000
    (mx, my), _ = tmb.datasets.mnist_shaped(n_train=200, n_test=10)
    assert mx.shape == (200, 784) and set(np.unique(mx)) <= {0, 1}
    m = tmb.datasets.inference_model(n_clauses=50)
    assert m.states.shape == (50, 8192) and np.all((m.states >= 0).sum(axis=1) == 20)
    a = tmb.datasets.inference_examples(3, 10, 5)
    b = tmb.datasets.inference_examples(3, 12, 2)
    assert np.array_equal(a[2:4], b)


def test_gtm1_model_files_byte_identical_to_reference(tmp_path):
    """GTM1 save/load: the reference's own files for a
    dense bank, a sparse bank and a rule set are reproduced byte for byte
    from the same model contents, and load back to the same contents."""
    import numpy as np

    from conftest import golden
    from paper_2405_04212_b200 import DenseClauseBank, SparseClauseBank, compile_ruleset
    from paper_2405_04212_b200.core import Config
    from paper_2405_04212_b200.modelio import (ModelFormatError, load_model, model_bytes,
                                               model_from_bytes, save_model)
    g = golden("modelio")
    cfg = Config(n_literals=7, n_clauses=6, n_classes=2, s=2.5, threshold=5, n_literal_budget=4,
                 seed=8, boost_true_positive=True)
    dense = DenseClauseBank(cfg)
    dense.states[:] = g["dense_states"]
    dense.weights[:] = g["dense_weights"]
    assert model_bytes(dense) == g["dense_bytes"].tobytes()
    scfg = Config(n_literals=40, n_clauses=5, n_classes=2, s=2.0, threshold=4, seed=2,
                  negated_literals_enabled=False, sparse_capacity=3, sparse_floor=-5)
    sparse = SparseClauseBank(scfg)
    ends = np.cumsum(g["sparse_lens"])
    starts = ends - g["sparse_lens"]
    sparse.clause_literals = [g["sparse_lits"][a:b].astype(np.int64) for a, b in zip(starts, ends)]
    sparse.clause_states = [g["sparse_sts"][a:b].astype(np.int8) for a, b in zip(starts, ends)]
    sparse.weights = g["sparse_weights"].astype(np.int32)
    assert model_bytes(sparse) == g["sparse_bytes"].tobytes()
    rset = compile_ruleset(dense)
    assert model_bytes(rset) == g["ruleset_bytes"].tobytes()
    # load the reference's files and re-save them (round trip)
    for name in ("dense", "sparse", "ruleset"):
        raw = g[name + "_bytes"].tobytes()
        m = model_from_bytes(raw)
        assert model_bytes(m) == raw, name
        path = tmp_path / f"{name}.gtm"
        save_model(m, path)
        assert path.read_bytes() == raw
        assert model_bytes(load_model(path)) == raw
    m = model_from_bytes(g["dense_bytes"].tobytes())
    assert np.array_equal(m.states, g["dense_states"]) and m.cfg == cfg
    for bad in (b"XXXX" + raw[4:], raw + b"\0", raw[:-1]):
        try:
            model_from_bytes(bad)
        except ModelFormatError:
            pass
        else:
            raise AssertionError("malformed file accepted")


# ---------------------------------------------------------------- search --
def _oracle_train(cfg, data, n_epochs):
    from oracle import oracle
    x, y = data
    st, _ = oracle.train(cfg, x, y, n_epochs)
    return st


def _oracle_eval(st, data):
    from oracle import oracle
    x, y = data
    _, pred = oracle.batch_votes(st.states, st.weights, oracle.augment_literals(x))
    return float(np.mean(pred == np.asarray(y)))


def test_search_space_parse_and_sample_match_reference():
    """SearchSpace.parse / sample draws == the reference's (tuning.py:34-101)."""
    from paper_2405_04212_b200 import RngStream, SearchSpace
    g = np.load(os.path.join(REPO, "tests", "golden", "search.npz"))
    space = SearchSpace.parse(bytes(g["space_text"]).decode())
    rng = RngStream.derive(123, 0x5EA7)
    draws = [space.sample(rng) for _ in range(40)]
    for name in ("s", "threshold", "n_clauses", "boost_true_positive", "state_max"):
        assert np.array_equal(np.array([d[name] for d in draws], dtype=np.float64),
                              g["draw_" + name]), name
    with pytest.raises(ValueError):
        SearchSpace.parse("s uniform 3 1")
    with pytest.raises(ValueError):
        SearchSpace.parse("s loguniform 0 1")
    with pytest.raises(ValueError):
        SearchSpace.parse("s gaussian 0 1")


@pytest.mark.parametrize("tag", ["hold", "cv"])
def test_random_search_ranking_matches_reference(tag):
    """random_search host logic (trial draws, coercion, holdout split, CV,
    ranking with ties by index) with the oracle as trainer == the
    reference's trials (tuning.py:194-227)."""
    from paper_2405_04212_b200 import Config, SearchSpace, random_search
    g = np.load(os.path.join(REPO, "tests", "golden", "search.npz"))
    base = Config(n_literals=6, n_clauses=8, n_classes=2, s=2.0, threshold=10, seed=0)
    small = SearchSpace.parse("s uniform 1.5 4.0\nthreshold int 5 20\nn_clauses cat 6,10")
    kw = {"cv_k": 3} if tag == "cv" else {}
    trials = random_search(small, base, (g["x"], g["y"]), n_trials=5, n_epochs=2, seed=31,
                           train_fn=_oracle_train, evaluate_fn=_oracle_eval, **kw)
    assert [t.index for t in trials] == g[tag + "_index"].tolist()
    assert np.array_equal([t.accuracy for t in trials], g[tag + "_acc"])
    assert np.array_equal([t.config.s for t in trials], g[tag + "_s"])
    assert [t.config.threshold for t in trials] == g[tag + "_T"].tolist()
    assert [t.config.n_clauses for t in trials] == g[tag + "_C"].tolist()
    assert all(isinstance(t.config.threshold, int) for t in trials)
