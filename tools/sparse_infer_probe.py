"""configs[4] sparse inference on one trained model (600 000 documents of
epoch 1): postings / candidate statistics and the time per 10^6 documents
of each inference kernel (TMB_LIB selects a library build)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2405_04212_b200 as tmb  # noqa: E402
from paper_2405_04212_b200 import _lib, datasets, sparse_train  # noqa: E402

tmb.runtime.require_device()
d = datasets.sparse_zipf(data_seed=5)
cfg = tmb.Config(**datasets.sparse_config_kwargs(seed=0))
sess = sparse_train.SparseTrainSession(cfg, d.indptr, d.indices, d.labels)
from paper_2405_04212_b200.executor import shuffle_permutation  # noqa: E402
order = shuffle_permutation(sess.N, sess.shuffle_rng).astype(np.int32)
sess.run_steps(torch.from_numpy(order[:600000]).cuda())
lits, sts, w, _ = sess.engine.get_lists()
inc = [l[s >= 0] for l, s in zip(lits, sts)]
n_inc = np.array([len(a) for a in inc])
cnt = np.zeros(cfg.n_literals, np.int64)
for a in inc:
    cnt[a] += 1
sample = [d.row(i) for i in range(2000)]
nh = np.array([cnt[r].sum() for r in sample])
print(f"clauses with includes {int((n_inc > 0).sum())}, includes per clause mean {n_inc.mean():.1f} "
      f"max {n_inc.max()}, postings per document mean {nh.mean():.1f} max {nh.max()}", flush=True)
for opt, name in ((0, "count (or this build's default)"), (1, "key")):
    try:
        _lib.call("tmb_set_option", b"sparse.infer_key", opt)
    except Exception:
        if opt:
            break
    for _ in range(2):
        v, p = sess.engine.votes_and_pred(sess.indptr, sess.indices, sess.N)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        v, p = sess.engine.votes_and_pred(sess.indptr, sess.indices, sess.N)
    b.record()
    torch.cuda.synchronize()
    print(f"{name}: {a.elapsed_time(b) / 3:.2f} ms per 10^6 documents (incl. index build), "
          f"checksum {int(p.sum())} {int(v.abs().sum())}", flush=True)
