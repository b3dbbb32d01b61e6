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

NAMES = ["eval(+votes)", "arrive", "precompute", "wait+decide", "flag bitmaps",
         "scan+events", "feedback", "-"]
NAMES_FAST = ["arrive", "all-reduce wait", "decide", "sync (B1)", "events (count+apply)",
              "feedback", "re-eval", "sums"]

ap = argparse.ArgumentParser()
ap.add_argument("--cta", type=int, nargs="*", default=[16, 148])
ap.add_argument("--threads", type=int, default=0)
ap.add_argument("--epochs", type=int, default=4)
ap.add_argument("--n-train", type=int, default=60000)
ap.add_argument("--skip", type=int, default=0, help="train.debug_skip ablation bits")
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
    nc = sess.launch["n_cta"]
    ph = torch.zeros(nc * (8 + 3072 + 9), dtype=torch.int64, device="cuda")
    _lib.call("tmb_trainer_set_profile", sess._h, ptr(ph))
    _lib.call("tmb_set_option", b"train.debug_skip", args.skip)
    trace = torch.zeros(len(ty) * 4, dtype=torch.int64, device="cuda")
    _lib.call("tmb_trainer_set_trace", sess._h, ptr(trace))
    st = torch.cuda.Event(enable_timing=True)
    en = torch.cuda.Event(enable_timing=True)
    st.record()
    sess.run_epoch()
    en.record()
    torch.cuda.synchronize()
    _lib.call("tmb_set_option", b"train.debug_skip", 0)
    ms = st.elapsed_time(en)
    tl = ph.cpu().numpy()[nc * 8:nc * (8 + 3072)].reshape(1024, nc, 3).astype(np.float64)
    p = ph.cpu().numpy()[:nc * 8].reshape(-1, 8).astype(np.float64) / clk_hz * 1e6 / len(ty)
    print(f"n_cta={sess.launch['n_cta']} threads={sess.launch['threads']} "
          f"smem_states={sess.launch['states_in_smem']}: {ms * 1e3 / len(ty):.2f} us/example "
          f"(clock {clk_hz / 1e6:.0f} MHz)")
    for q in range(8):
        name = (NAMES if args.no_keys else NAMES_FAST)[q]
        print(f"   {name:22s} mean {p[:, q].mean():6.3f}  max {p[:, q].max():6.3f}  "
              f"cta0 {p[0, q]:6.3f} us/ex")
    if not args.no_keys:
        raw = ph.cpu().numpy().astype(np.float64)
        hp = raw[nc * (8 + 3072):nc * (8 + 3072 + 8)].reshape(nc, 8)
        nh = raw[nc * (8 + 3072 + 8):nc * (8 + 3072 + 9)]
        nl = len(ty) - nh
        lp = raw[:nc * 8].reshape(nc, 8)
        print(f"   per step, warp 0 of each CTA (light / empty steps n={nl.mean():.0f}, "
              f"heavy steps (> 64 flag entries) n={nh.mean():.0f}):")
        for q in range(8):
            lt = lp[:, q] / np.maximum(nl, 1) / clk_hz * 1e9
            hv = hp[:, q] / np.maximum(nh, 1) / clk_hz * 1e9
            print(f"     {NAMES_FAST[q]:22s} light mean {lt.mean():7.0f} ns   heavy mean {hv.mean():7.0f} "
                  f"max {hv.max():7.0f} ns")
    if tl[:, :, 0].min() > 0:
        last = tl[:, :, 0].max(axis=1, keepdims=True)
        det = tl[:, :, 1] - last            # detection after the last arrival
        skew = last - tl[:, :, 0]           # own arrival before the last one
        step = np.diff(tl[:, :, 2].max(axis=1))
        who = np.argmax(tl[:, :, 0], axis=1)
        print(f"   timeline (ns, steps 64..1087): step {np.median(step):.0f} median; "
              f"detect-after-last-arrival mean {det.mean():.0f} min {det.min():.0f} "
              f"max {det.max():.0f}; arrival skew mean {skew.mean():.0f} "
              f"max {skew.max():.0f}; last arriver CTAs {np.bincount(who, minlength=nc).argsort()[-5:]}")
        end_to_arr = tl[1:, :, 0] - tl[:-1, :, 2].max(axis=1, keepdims=True)
        print(f"   from the previous step's last end to arrival: mean {end_to_arr.mean():.0f} "
              f"min {end_to_arr.min():.0f} max {end_to_arr.max():.0f}")
        med = np.median(tl, axis=1, keepdims=True)
        off = (tl - med).mean(axis=0)  # per CTA mean offset of arrival / detect / end
        worst = np.argsort(off[:, 0])[-6:]
        for r in worst:
            print(f"   cta {r:3d}: arrival {off[r, 0]:7.0f}  detect {off[r, 1]:7.0f}  "
                  f"end {off[r, 2]:7.0f} ns vs median")
        print(f"   median CTA spread of detection {np.median(tl[:, :, 1].max(1) - tl[:, :, 1].min(1)):.0f} ns")
        A = np.median(tl[:, :, 0], axis=1); L = tl[:, :, 0].max(axis=1)
        D = np.median(tl[:, :, 1], axis=1); E = np.median(tl[:, :, 2], axis=1)
        EM = tl[:, :, 2].max(axis=1)
        q = lambda v: f"p50 {np.median(v):6.0f} mean {v.mean():6.0f} p90 {np.percentile(v, 90):6.0f}"
        print("   per step: last-arrival minus median arrival  ", q(L - A))
        print("             median detect minus last arrival   ", q(D - L))
        print("             median end minus median detect     ", q(E - D))
        print("             max end minus median end           ", q(EM - E))
        print("             next median arrival minus med. end ", q(A[1:] - E[:-1]))
    evs = trace.cpu().numpy().reshape(-1, 4)[64:1088, 3]
    dur = np.diff(np.median(tl[:, :, 1], axis=1))  # detect-to-detect per step
    ev_next = evs[:-1]
    for name, m in (("empty", ev_next == 0), ("1-100 events", (ev_next > 0) & (ev_next <= 100)),
                    (">100 events", ev_next > 100)):
        if m.any():
            print(f"   steps with {name:13s}: n={m.sum():3d} median detect-to-detect "
                  f"{np.median(dur[m]):6.0f} ns mean {dur[m].mean():6.0f}")
    if tl[:, :, 0].min() > 0:
        send, det = tl[:, :, 0], tl[:, :, 1]
        sh = send[2:] - det[:-2]            # send of A(e) after detection of e-2 (per CTA)
        q2 = lambda v: f"p10 {np.percentile(v, 10):6.0f} p50 {np.median(v):6.0f} p90 {np.percentile(v, 90):6.0f}"
        e_empty = (evs[:-2] == 0) & (evs[1:-1] == 0)
        print("   [empty pairs] send(A e) - det(e-2) per CTA:", q2(sh[e_empty].ravel()))
        spread = send.max(axis=1) - np.median(send, axis=1)
        lat = np.median(det, axis=1) - send.max(axis=1)
        print("   [empty] send spread (max - median):", q2(spread[2:][e_empty]),
              " det(med) - last send:", q2(lat[2:][e_empty]))
