"""Longer GPU-vs-oracle parity runs at the benchmarked shapes than the test
suite can afford (the oracle is the slow side), one part per invocation; run
on the GPU box, results to gpurun_out/ (copied to profiles/ by hand):

    python tools/long_parity.py c2 --epochs 8      # configs[1], full epochs
    python tools/long_parity.py c4 --steps 400     # configs[3], full shape
    python tools/long_parity.py c5 --docs 1500     # configs[4], full shape

Each prints one JSON line: what ran, whether every compared array is equal,
and SHA-1 digests of the GPU model.  Verification evidence, not a test: the
suite's own cases (tests/test_gpu_fullsize.py) stay small enough for CI.
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def sha(a):
    return hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("part", choices=["c2", "c4", "c5"])
    ap.add_argument("--epochs", type=int, default=8)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--docs", type=int, default=1500)
    args = ap.parse_args()
    import torch

    import paper_2405_04212_b200 as tmb
    from oracle import oracle
    from paper_2405_04212_b200 import datasets
    t0 = time.time()
    out = {"part": args.part}
    if args.part == "c2":
        (tx, ty), _ = datasets.mnist_shaped(data_seed=7)
        cfg = tmb.Config(**datasets.mnist_shaped_config_kwargs(seed=0))
        sess = tmb.DenseTrainSession(cfg, tx, ty)
        for _ in range(args.epochs):
            sess.run_epoch()
        m = sess.model()
        t1 = time.time()
        ost, _ = oracle.train(cfg, tx, ty, args.epochs)
        eq = {"states": bool(np.array_equal(m.states, ost.states)),
              "weights": bool(np.array_equal(m.weights, ost.weights)),
              "block_counters": bool(np.array_equal(
                  sess.block_counters.cpu().numpy().view(np.uint64), ost.block_counters)),
              "fb_counter": bool(sess.fb_counter == ost.fb_counter)}
        out.update(workload=f"configs[1]: {args.epochs} full epochs ({args.epochs * len(ty)} "
                            f"examples), bench data and model seeds", kernel=sess.launch["kernel"],
                   events=int(ost.block_counters[0]), gpu_states=sha(m.states),
                   gpu_weights=sha(m.weights))
    elif args.part == "c4":
        (tx, ty), _ = datasets.bag_of_words(data_seed=4)
        cfg = tmb.Config(**datasets.bag_of_words_config_kwargs(seed=0))
        sess = tmb.DenseTrainSession(cfg, tx, ty)
        order = sess.next_order()[:args.steps]
        sess.run_steps(torch.from_numpy(order.astype(np.int32)).cuda())
        m = sess.model()
        t1 = time.time()
        st = oracle.new_train_state(cfg)
        oracle.train_steps(cfg, st, oracle.augment_literals(tx), ty, order.astype(np.int64))
        eq = {"states": bool(np.array_equal(m.states, st.states)),
              "weights": bool(np.array_equal(m.weights, st.weights)),
              "block_counters": bool(np.array_equal(
                  sess.block_counters.cpu().numpy().view(np.uint64), st.block_counters)),
              "fb_counter": bool(sess.fb_counter == st.fb_counter)}
        out.update(workload=f"configs[3]: first {args.steps} steps of epoch 1 at full shape "
                            f"(bench data and model seeds)", kernel=sess.launch["kernel"],
                   events=int(st.block_counters[0]), gpu_states=sha(m.states),
                   gpu_weights=sha(m.weights))
    else:
        from paper_2405_04212_b200.sparse_train import SparseTrainSession
        d = datasets.sparse_zipf(data_seed=5)
        cfg = tmb.Config(**datasets.sparse_config_kwargs(seed=0))
        ocfg = oracle.OracleCfg(**datasets.sparse_config_kwargs(seed=0))
        cands = np.unique(d.indices).astype(np.int64)
        sh_seed = oracle.derive_stream(ocfg.seed, oracle.SHUFFLE_STREAM)
        order, _ = oracle.shuffle_permutation(len(d), sh_seed, 0)
        n = args.docs
        docs = [d.row(int(i)) for i in order[:n]]
        labels = d.labels[order[:n]].astype(np.int64)
        ptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum([len(r) for r in docs], out=ptr[1:])
        idx = np.concatenate(docs).astype(np.int32)
        sess = SparseTrainSession(cfg, ptr, idx, labels, candidates=cands)
        sess.run_steps(torch.arange(n, dtype=torch.int32, device="cuda"))
        m = sess.model()
        _, _, _, bc = sess.engine.get_lists()
        t1 = time.time()
        banks, bctr, fb = oracle.sparse_train(ocfg, docs, labels, candidates=cands,
                                              order=np.arange(n))
        bk = banks[0]
        lists_eq = all(np.array_equal(m.clause_literals[j], bk.lits[j]) and
                       np.array_equal(m.clause_states[j], bk.sts[j])
                       for j in range(cfg.n_clauses))
        eq = {"clause_lists_and_states": bool(lists_eq),
              "weights": bool(np.array_equal(m.weights, bk.weights)),
              "block_counters": bool(np.array_equal(bc, np.asarray(bctr, dtype=np.uint64)))}
        out.update(workload=f"configs[4]: first {n} documents of epoch 1 at full shape "
                            f"({cands.size} candidate literals; bench data and model seeds)",
                   events=int(bctr[0]), gpu_weights=sha(m.weights),
                   stored_pairs=int(sum(len(x) for x in m.clause_literals)))
    out.update(equal=eq, all_equal=all(eq.values()), gpu_s=round(t1 - t0, 1),
               oracle_s=round(time.time() - t1, 1))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
