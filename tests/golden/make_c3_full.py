"""Writes tests/golden/c3_full.npz: the CPU oracle's votes for ALL 2^22
examples of the benchmarked configs[2] workload (bench.py: data_seed 3,
model_seed 11, 4096 features, 10000 clauses x 20 includes, 10 classes).

Test infrastructure only.  The votes come from the oracle's restatement of
the reference's dense path, DenseClauseBank.batch_votes (dense.py:171-174 ->
kernels/_numba.py:61-68 one-output loop with early exit), run over the
augmented literals (core.py:232-242).  Predictions follow as argmax with ties
to the lowest class (executor.py:382).

Only examples whose vote row is non-zero are stored (with their index); every
other example has all-zero votes and therefore prediction 0 by the argmax
rule, so the fixture determines all 2^22 vote rows and predictions.  A
per-chunk checksum of the predictions is stored as well.

Run once (about 45 min on 8 host threads):
    python tests/golden/make_c3_full.py [--threads 8]
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

N_TOTAL = 1 << 22
DATA_SEED, MODEL_SEED = 3, 11
F, C, K = 4096, 10000, 10


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--chunk", type=int, default=1 << 15)
    ap.add_argument("--n", type=int, default=N_TOTAL)
    ap.add_argument("--out", default=os.path.join(HERE, "c3_full.npz"))
    args = ap.parse_args()
    m = datasets.inference_model(model_seed=MODEL_SEED, n_features=F, n_clauses=C, n_classes=K)
    idx_parts, vote_parts, pred_sums = [], [], []
    t0 = time.time()
    for lo in range(0, args.n, args.chunk):
        cnt = min(args.chunk, args.n - lo)
        xs = datasets.inference_examples(DATA_SEED, lo, cnt, n_features=F)
        votes, pred = oracle.batch_votes(m.states, m.weights, oracle.augment_literals(xs),
                                         nthreads=args.threads)
        nz = np.flatnonzero(np.any(votes != 0, axis=1))
        idx_parts.append((lo + nz).astype(np.int32))
        vote_parts.append(votes[nz].astype(np.int32))
        pred_sums.append(int(pred.sum()))
        done = lo + cnt
        el = time.time() - t0
        print(f"{done}/{args.n} examples, {sum(p.size for p in idx_parts)} firing, "
              f"{el:.0f}s elapsed, eta {el / done * (args.n - done):.0f}s", flush=True)
    np.savez_compressed(args.out, n=np.int64(args.n), chunk=np.int64(args.chunk),
                        data_seed=np.int64(DATA_SEED), model_seed=np.int64(MODEL_SEED),
                        index=np.concatenate(idx_parts), votes=np.concatenate(vote_parts),
                        pred_chunk_sums=np.asarray(pred_sums, dtype=np.int64))
    print("wrote", args.out)


if __name__ == "__main__":
    main()
