"""Per-phase clock64 profile of the fused trainer on the configs[1] shapes.

    python tools/phase_profile.py [--cta N ...] [--threads T] [--epochs E]

Prints, per launch configuration, microseconds per example spent by thread 0
of each CTA in each kernel phase (mean and max over CTAs) for the last epoch.
"""
import argparse
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2405_04212_b200 as tmb  # noqa: E402
from paper_2405_04212_b200 import _lib, datasets  # noqa: E402
from paper_2405_04212_b200.runtime import ptr  # noqa: E402

NAMES = ["eval(+votes)", "arrive", "precompute", "wait+decide", "flag count/bitmaps",
         "scan+events", "feedback", "-"]

ap = argparse.ArgumentParser()
ap.add_argument("--cta", type=int, nargs="*", default=[16, 148])
ap.add_argument("--threads", type=int, default=0)
ap.add_argument("--epochs", type=int, default=4)
ap.add_argument("--n-train", type=int, default=60000)
ap.add_argument("--no-keys", action="store_true", help="per-CTA flag draws instead of keys")
args = ap.parse_args()

(tx, ty), _ = datasets.mnist_shaped(n_train=args.n_train, n_test=10)
clk_hz = torch.cuda.get_device_properties(0).clock_rate * 1e3
for n_cta in args.cta:
    cfg = tmb.Config(**datasets.mnist_shaped_config_kwargs(seed=0))
    sess = tmb.DenseTrainSession(cfg, tx, ty, n_cta=n_cta, threads=args.threads,
                                 flag_keys=not args.no_keys)
    for _ in range(args.epochs - 1):
        sess.run_epoch()
    ph = torch.zeros(sess.launch["n_cta"] * 8, dtype=torch.int64, device="cuda")
    _lib.call("tmb_trainer_set_profile", sess._h, ptr(ph))
    st = torch.cuda.Event(enable_timing=True)
    en = torch.cuda.Event(enable_timing=True)
    st.record()
    sess.run_epoch()
    en.record()
    torch.cuda.synchronize()
    ms = st.elapsed_time(en)
    p = ph.cpu().numpy().reshape(-1, 8).astype(np.float64) / clk_hz * 1e6 / len(ty)
    print(f"n_cta={sess.launch['n_cta']} threads={sess.launch['threads']} "
          f"smem_states={sess.launch['states_in_smem']}: {ms * 1e3 / len(ty):.2f} us/example "
          f"(clock {clk_hz / 1e6:.0f} MHz)")
    for q in range(7):
        print(f"   {NAMES[q]:22s} mean {p[:, q].mean():6.3f}  max {p[:, q].max():6.3f}  "
              f"cta0 {p[0, q]:6.3f} us/ex")
