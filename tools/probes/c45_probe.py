"""Throughput probe for configs[3] (BoW dense training) and configs[4]
(SparseTM training + inverted-index inference)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2405_04212_b200 as tmb  # noqa: E402
from paper_2405_04212_b200 import datasets, sparse_train  # noqa: E402

def ev():
    return torch.cuda.Event(enable_timing=True)

if "c5" in sys.argv:
    t0 = time.time()
    d = datasets.sparse_zipf()
    print("c5 data", round(time.time() - t0, 1), "s", d.indptr.shape, d.indices.shape)
    cfg = tmb.Config(**datasets.sparse_config_kwargs(seed=0))
    sess = sparse_train.SparseTrainSession(cfg, d.indptr, d.indices, d.labels)
    order = sess.run_epoch(max_steps=20000)   # warm-up slice
    torch.cuda.synchronize()
    for n in (100000, 300000):
        a, b = ev(), ev()
        s0 = sess.stats_dict()
        a.record()
        sess.run_epoch(max_steps=n)
        b.record()
        torch.cuda.synchronize()
        s1 = sess.stats_dict()
        ms = a.elapsed_time(b)
        print(f"c5 train {n} docs: {ms:.1f} ms -> {n / ms * 1e3:.0f} docs/s; events/doc "
              f"{(s1['events'] - s0['events']) / n:.1f} draws/doc {(s1['draws'] - s0['draws']) / n:.0f}")
    eng = sess.engine
    for _ in range(2):
        v, p = eng.votes_and_pred(sess.indptr, sess.indices, sess.N)
    a, b = ev(), ev()
    a.record()
    v, p = eng.votes_and_pred(sess.indptr, sess.indices, sess.N)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print(f"c5 infer {sess.N} docs: {ms:.2f} ms -> {sess.N / ms * 1e3 / 1e6:.1f} M docs/s; "
          f"acc {(p.cpu().numpy() == d.labels).mean():.3f}")
if "c4" in sys.argv:
    t0 = time.time()
    (tx, ty), (ex, ey) = datasets.bag_of_words()
    print("c4 data", round(time.time() - t0, 1), "s", tx.shape)
    cfg = tmb.Config(**datasets.bag_of_words_config_kwargs(seed=0))
    sess = tmb.DenseTrainSession(cfg, tx, ty)
    print("launch", sess.launch)
    order = torch.from_numpy(sess.next_order().astype(np.int32)).cuda()
    sess.run_steps(order[:1000])
    torch.cuda.synchronize()
    for lo, hi in ((1000, 6000), (6000, 25000)):
        a, b = ev(), ev()
        s0 = sess.stats_dict()
        a.record()
        sess.run_steps(order[lo:hi])
        b.record()
        torch.cuda.synchronize()
        s1 = sess.stats_dict()
        ms = a.elapsed_time(b)
        n = hi - lo
        print(f"c4 train {n} ex: {ms:.1f} ms -> {n / ms * 1e3:.0f} ex/s; events/ex "
              f"{(s1['events'] - s0['events']) / n:.1f} draws/ex {(s1['draws'] - s0['draws']) / n:.0f}")
