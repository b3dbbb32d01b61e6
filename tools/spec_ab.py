"""A/B of the configs[1] fast grid trainers: k_train_fast (train.spec_window=0)
against k_train_spec at several window sizes, from the committed oracle
checkpoint after epoch 3 (tests/golden/c2_epoch3.npz), timing epochs 4..4+E-1
with CUDA events and checking every variant ends bit-identical to the first.

    python tools/spec_ab.py --windows 0 16 8 --epochs 3
"""

import argparse
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--windows", type=int, nargs="+", default=[0, 16])
    ap.add_argument("--epochs", type=int, default=3)
    ap.add_argument("--threads", type=int, default=0)
    args = ap.parse_args()
    import torch

    import paper_2405_04212_b200 as tmb
    from paper_2405_04212_b200 import _lib, datasets

    (tx, ty), _ = datasets.mnist_shaped(data_seed=7)
    cfg = tmb.Config(**datasets.mnist_shaped_config_kwargs(seed=0))
    g = np.load(os.path.join(REPO, "tests", "golden", "c2_epoch3.npz"))
    ref = None
    out = []
    for wsz in args.windows:
        _lib.call("tmb_set_option", b"train.spec_window", wsz)
        sess = tmb.DenseTrainSession(cfg, tx, ty, threads=args.threads,
                                     states=g["states"], weights=g["weights"])
        sess.block_counters.copy_(torch.from_numpy(g["block_counters"].view(np.int64)))
        sess.fb_counter = int(g["fb_counter"])
        sess.shuffle_rng.counter = int(g["shuffle_counter"])
        ms = []
        for _ in range(args.epochs):
            order = sess.next_order().astype(np.int32)
            od = torch.from_numpy(order).cuda()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            sess.run_steps(od)
            b.record()
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        st = sess.states.cpu().numpy()
        w = sess.weights.cpu().numpy()
        bc = sess.block_counters.cpu().numpy()
        same = None
        if ref is None:
            ref = (st, w, bc)
        else:
            same = bool(np.array_equal(st, ref[0]) and np.array_equal(w, ref[1])
                        and np.array_equal(bc, ref[2]))
        rec = dict(window=wsz, launch=sess.launch, ms_per_epoch=ms,
                   us_per_example=[m * 1e3 / len(ty) for m in ms], identical_to_first=same,
                   stats=sess.stats_dict())
        out.append(rec)
        print(json.dumps(rec), flush=True)
        del sess
    _lib.call("tmb_set_option", b"train.spec_window", 16)


if __name__ == "__main__":
    main()
