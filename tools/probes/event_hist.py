"""Distribution of update events per training step (configs[1] shapes)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2405_04212_b200 as tmb  # noqa: E402
from paper_2405_04212_b200 import _lib, datasets  # noqa: E402
from paper_2405_04212_b200.runtime import ptr  # noqa: E402

(tx, ty), _ = datasets.mnist_shaped(n_train=60000, n_test=10)
cfg = tmb.Config(**datasets.mnist_shaped_config_kwargs(seed=0))
sess = tmb.DenseTrainSession(cfg, tx, ty, n_cta=148)
for ep in range(4):
    tr = torch.zeros(len(ty) * 4, dtype=torch.int64, device="cuda")
    _lib.call("tmb_trainer_set_trace", sess._h, ptr(tr))
    sess.run_epoch()
    torch.cuda.synchronize()
    ev = tr.cpu().numpy().reshape(-1, 4)[:, 3]
    q = np.percentile(ev, [10, 50, 75, 90, 95, 99, 99.9])
    share = [ev[ev > t].sum() / ev.sum() for t in (100, 300, 1000)]
    print(f"epoch {ep + 1}: mean {ev.mean():.1f} pct10/50/75/90/95/99/99.9 {q.astype(int)} "
          f"share of events in steps >100/>300/>1000: {np.round(share, 3)} "
          f"frac steps >100: {(ev > 100).mean():.3f}")
