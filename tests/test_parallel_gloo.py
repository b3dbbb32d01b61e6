"""Multi-process host logic on CPU (gloo, world_size 2): sharding, sweep /
CV job distribution and gathering.  The per-job compute is the CPU oracle
(test infrastructure), so results must equal the single-process run."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import REPO


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


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


def _sparse_case():
    """A trained oracle sparse bank and ragged documents (some empty)."""
    from oracle import oracle

    from paper_2405_04212_b200.core import Config
    rng = np.random.default_rng(3)
    docs = []
    for i in range(90):
        n = 0 if i % 17 == 0 else int(rng.integers(1, 40))
        docs.append(np.sort(rng.choice(300, size=n, replace=False)).astype(np.int64))
    labels = np.array([int(np.isin(d, np.arange(20)).sum() > 1) for d in docs])
    cfg = Config(n_literals=300, n_clauses=12, n_classes=2, s=3.0, threshold=10, seed=4,
                 negated_literals_enabled=False, sparse_capacity=8)
    banks, _, _ = oracle.sparse_train(cfg, docs, labels, n_epochs=2)
    return banks[0], docs


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, REPO)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch.distributed as dist

    from paper_2405_04212_b200 import datasets, parallel, tuning
    from paper_2405_04212_b200.core import Config
    parallel.init_from_env("gloo")
    (tx, ty), (ex, ey) = datasets.noisy_xor(n_train=300, n_test=100)
    # sweep: 4 configs over 2 ranks
    cfgs = [Config(**{**datasets.noisy_xor_config_kwargs(seed), "s": s})
            for seed, s in ((0, 3.9), (1, 2.0), (2, 5.0), (3, 3.0))]
    accs = parallel.run_sweep(cfgs, (tx, ty), (ex, ey), 2, train_fn=_oracle_train,
                              evaluate_fn=_oracle_eval)
    # CV over the ranks
    rep = tuning.cross_validate(cfgs[0], (tx, ty), 3, 1, seed=5, train_fn=_oracle_train,
                                evaluate_fn=_oracle_eval)
    # random search: 5 trials over the ranks
    space = tuning.SearchSpace.parse("s uniform 1.5 5.0\nthreshold int 5 20")
    trials = tuning.random_search(space, cfgs[0], (tx, ty), n_trials=5, n_epochs=1, seed=8,
                                  train_fn=_oracle_train, evaluate_fn=_oracle_eval)
    # sharded rows
    lo, hi = parallel.shard_range(101, world, rank)
    rows = parallel.gather_rows(np.arange(lo, hi), 101)
    # sharded sparse inference (configs[4] path): nnz-balanced CSR row shards,
    # each rank votes its rows (oracle bank standing in for the device engine),
    # predictions gathered once
    bank, docs = _sparse_case()
    ip = np.zeros(len(docs) + 1, dtype=np.int64)
    np.cumsum([len(a) for a in docs], out=ip[1:])
    slo, shi = parallel.csr_shard(ip, world, rank)
    from oracle import oracle
    v = oracle.sparse_batch_votes([bank], docs[slo:shi])
    spred = parallel.gather_rows(np.argmax(v, axis=1), len(docs))
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), accs=np.array(accs),
             cv=np.array(rep.fold_accuracies), folds=rep.fold_assignments, rows=rows,
             search=np.array([[t.index, t.accuracy] for t in trials]), spred=spred,
             sshard=np.array([slo, shi]))
    dist.barrier()
    dist.destroy_process_group()


def test_sweep_cv_and_sharding_over_two_gloo_ranks(tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0 = np.load(tmp_path / "r0.npz")
    r1 = np.load(tmp_path / "r1.npz")
    for key in ("accs", "cv", "folds", "rows", "search", "spred"):
        assert np.array_equal(r0[key], r1[key]), key
    assert np.array_equal(r0["rows"], np.arange(101))
    # the two shards tile the documents; gathered predictions == unsharded
    assert r0["sshard"][0] == 0 and r0["sshard"][1] == r1["sshard"][0]
    bank, docs = _sparse_case()
    assert r1["sshard"][1] == len(docs)
    from oracle import oracle
    assert np.array_equal(r0["spred"], np.argmax(oracle.sparse_batch_votes([bank], docs), axis=1))
    # single-process reference for the same jobs
    import sys
    sys.path.insert(0, REPO)
    from paper_2405_04212_b200 import datasets, tuning
    from paper_2405_04212_b200.core import Config
    (tx, ty), (ex, ey) = datasets.noisy_xor(n_train=300, n_test=100)
    cfgs = [Config(**{**datasets.noisy_xor_config_kwargs(seed), "s": s})
            for seed, s in ((0, 3.9), (1, 2.0), (2, 5.0), (3, 3.0))]
    single = [_oracle_eval(_oracle_train(c, (tx, ty), 2), (ex, ey)) for c in cfgs]
    assert np.array_equal(r0["accs"], np.array(single))
    rep = tuning.cross_validate(cfgs[0], (tx, ty), 3, 1, seed=5, train_fn=_oracle_train,
                                evaluate_fn=_oracle_eval)
    assert np.array_equal(r0["cv"], np.array(rep.fold_accuracies))
    space = tuning.SearchSpace.parse("s uniform 1.5 5.0\nthreshold int 5 20")
    trials = tuning.random_search(space, cfgs[0], (tx, ty), n_trials=5, n_epochs=1, seed=8,
                                  train_fn=_oracle_train, evaluate_fn=_oracle_eval)
    assert np.array_equal(r0["search"], np.array([[t.index, t.accuracy] for t in trials]))


def test_shard_and_job_assignment():
    from paper_2405_04212_b200 import parallel
    for n in (0, 1, 7, 4194304):
        for world in (1, 2, 3, 8):
            ranges = [parallel.shard_range(n, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
    # nnz-balanced CSR shards: contiguous, covering, within one row of balance
    rng = np.random.default_rng(1)
    for n in (0, 1, 5, 1000):
        lens = rng.integers(0, 200, size=n)
        ip = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(lens, out=ip[1:])
        for world in (1, 2, 3, 8):
            rs = [parallel.csr_shard(ip, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            if n:
                loads = [ip[b] - ip[a] for a, b in rs]
                assert max(loads) - ip[-1] / world <= lens.max(initial=0) + 1
    jobs = [parallel.jobs_of(8, 3, r) for r in range(3)]
    assert sorted(j for js in jobs for j in js) == list(range(8))


def test_stratified_kfold_matches_reference_semantics():
    from paper_2405_04212_b200 import tuning
    rng = np.random.default_rng(0)
    for trial in range(30):
        k = int(rng.integers(2, 6))
        labels = rng.integers(0, 3, size=int(rng.integers(3 * k, 80)))
        if np.bincount(labels, minlength=3).min() < k:
            continue
        folds = tuning.stratified_kfold(labels, k, seed=trial)
        for cls in range(3):
            per = [int(np.sum((labels == cls) & (folds == f))) for f in range(k)]
            assert max(per) - min(per) <= 1


def test_stratified_kfold_golden():
    from conftest import golden

    from paper_2405_04212_b200 import tuning
    g = golden("tuning")
    for t in range(12):
        assert np.array_equal(tuning.stratified_kfold(g[f"t{t}_labels"], int(g[f"t{t}_k"]), t),
                              g[f"t{t}_folds"])
