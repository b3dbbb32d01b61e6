"""Writes tests/golden/c5_prefix.npz: the CPU oracle's SparseTM model after
the first documents of epoch 1 of the benchmarked configs[4] workload
(bench.py rank 0: datasets.sparse_zipf(data_seed=5), 10^6 documents x 100
Zipf(1.05) ids over a 10^6 vocabulary; sparse_config_kwargs(seed=0): 2000
clauses, capacity 64, floor -15, T=2000, s=5, negations off).

Test infrastructure only.  The oracle restates SparseClauseBank feedback
(sparse.py:162-249) and executor.train's sparse branch (executor.py:287-289:
candidates = union of the WHOLE training set's actives), so every Type II
event walks the full ~10^6-literal candidate set, as the reference does.

Stored: the consumed documents (CSR, in epoch order) with labels, the
candidate set as a bitmap, the trained model (clause lists / states as CSR,
weights, block counter), and the oracle's votes on the next 2000 documents
of the epoch (held out from this prefix).

    python tests/golden/make_c5_prefix.py [--n 300]
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from oracle import oracle  # noqa: E402
from paper_2405_04212_b200 import datasets  # noqa: E402


def csr(rows):
    ptr = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum([len(r) for r in rows], out=ptr[1:])
    idx = np.concatenate(rows).astype(np.int32) if len(rows) else np.zeros(0, np.int32)
    return ptr, idx


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=300)
    ap.add_argument("--n-test", type=int, default=2000)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default=os.path.join(HERE, "c5_prefix.npz"))
    args = ap.parse_args()
    t0 = time.time()
    d = datasets.sparse_zipf(data_seed=5)
    print(f"dataset {time.time() - t0:.0f}s", flush=True)
    cfg = oracle.OracleCfg(**datasets.sparse_config_kwargs(seed=args.seed))
    cands = np.unique(d.indices).astype(np.int64)
    sh_seed = oracle.derive_stream(cfg.seed, oracle.SHUFFLE_STREAM)
    order, _ = oracle.shuffle_permutation(len(d), sh_seed, 0)
    n, nt = args.n, args.n_test
    docs = [d.row(int(i)) for i in order[:n]]
    labels = d.labels[order[:n]].astype(np.int64)

    def progress(step):
        if step % 25 == 0:
            print(f"step {step}/{n} {time.time() - t0:.0f}s", flush=True)

    banks, bctr, fb = oracle.sparse_train(cfg, docs, labels, candidates=cands,
                                          order=np.arange(n), progress=progress)
    bk = banks[0]
    m_ptr, m_lits = csr(bk.lits)
    m_sts = np.concatenate(bk.sts).astype(np.int8) if m_lits.size else np.zeros(0, np.int8)
    tdocs = [d.row(int(i)) for i in order[n:n + nt]]
    tlab = d.labels[order[n:n + nt]].astype(np.int64)
    tvotes = oracle.sparse_batch_votes(banks, tdocs)
    acc = float(np.mean(np.argmax(tvotes, axis=1) == tlab))
    ip, ix = csr(docs)
    tip, tix = csr(tdocs)
    bits = np.zeros(cfg.n_literals, dtype=np.uint8)
    bits[cands] = 1
    np.savez_compressed(args.out, seed=np.int64(cfg.seed), indptr=ip, indices=ix, labels=labels,
                        cand_bits=np.packbits(bits, bitorder="little"), m_ptr=m_ptr,
                        m_lits=m_lits, m_sts=m_sts, weights=bk.weights,
                        bctr=np.asarray(bctr, dtype=np.uint64), fb=np.uint64(fb),
                        t_indptr=tip, t_indices=tix, t_labels=tlab, t_votes=tvotes,
                        accuracy=np.float64(acc))
    print(f"wrote {args.out}: {n} documents, {int(bctr[0])} events, held-out accuracy {acc:.4f},"
          f" pairs {m_lits.size}, {time.time() - t0:.0f}s")


if __name__ == "__main__":
    main()
