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
    ap.add_argument("--n-cta", type=int, default=0, help="CTAs (0 = one per SM)")
    ap.add_argument("--dbg", type=int, default=0, help="train.debug_skip bits (timing ablations)")
    ap.add_argument("--ents", type=int, default=64, help="train.spec_entries (0 = auto)")
    ap.add_argument("--prof", action="store_true",
                    help="k_train_spec phase counters (clock64 per CTA, see tmb_train.cu)")
    args = ap.parse_args()
    import torch

    import paper_2405_04212_b200 as tmb
    from paper_2405_04212_b200 import _lib, datasets

    (tx, ty), _ = datasets.mnist_shaped(data_seed=7)
    cfg = tmb.Config(**datasets.mnist_shaped_config_kwargs(seed=0))
    g = np.load(os.path.join(REPO, "tests", "golden", "c2_epoch3.npz"))
    ref = None
    out = []
    _lib.call("tmb_set_option", b"train.debug_skip", args.dbg)
    _lib.call("tmb_set_option", b"train.spec_entries", args.ents)
    for wsz in args.windows:
        _lib.call("tmb_set_option", b"train.spec_window", wsz)
        sess = tmb.DenseTrainSession(cfg, tx, ty, threads=args.threads, n_cta=args.n_cta,
                                     states=g["states"], weights=g["weights"])
        sess.block_counters.copy_(torch.from_numpy(g["block_counters"].view(np.int64)))
        sess.fb_counter = int(g["fb_counter"])
        sess.shuffle_rng.counter = int(g["shuffle_counter"])
        ms = []
        prof = None
        if args.prof and wsz > 0:
            ncta = sess.launch["n_cta"]
            prof = torch.zeros(ncta * 16 + ncta * 2048 * 14, dtype=torch.int64, device="cuda")
            _lib.call("tmb_trainer_set_profile", sess._h, prof.data_ptr())

        def reset():
            if prof is not None:
                prof.zero_()
        phases = []
        for _ in range(args.epochs):
            order = sess.next_order().astype(np.int32)
            od = torch.from_numpy(order).cuda()
            reset()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            sess.run_steps(od)
            b.record()
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
            if prof is not None:
                allp = prof.cpu().numpy()
                p = allp[:ncta * 16].reshape(-1, 16).astype(np.float64)
                tl = allp[ncta * 16:].reshape(ncta, 2048, 14).astype(np.float64)
                heavy = (tl[:, :, 0] > 0).all(axis=0) & (tl[:, :, 1] > 0).all(axis=0)
                polled = (tl[:, :, 1] > 0).all(axis=0)
                h = tl[:, heavy, :]
                cyc = 1.9  # cycles per ns (approx.)
                ev = (h[:, :, 3] - h[:, :, 2]) / cyc
                fb = (h[:, :, 4] - h[:, :, 3]) / cyc
                pb = (h[:, :, 5] - h[:, :, 4]) / cyc
                chain = (h[:, :, 5] - h[:, :, 2]) / cyc
                # latency: next polled window's earliest completion - latest publication
                idx = np.nonzero(heavy)[0]
                lat = []
                for w in idx:
                    nxt = w + 2
                    if nxt < 2048 and polled[nxt]:
                        lat.append(tl[:, nxt, 1].min() - tl[:, w, 0].max())
                med = lambda a: float(np.median(a))
                nw = h[:, :, 6]
                fb_by_nwork = {int(v): round(float(np.median(fb[nw == v])), 1)
                               for v in range(0, 12) if (nw == v).sum() > 20}
                nw_max = nw.max(axis=0)
                ent = h[0, :, 7]
                timeline = dict(
                    heavy_windows=int(heavy.sum()),
                    chain_ns=dict(median_cta=med(np.median(chain, axis=0)), max_cta=med(chain.max(axis=0))),
                    events_ns=dict(median_cta=med(np.median(ev, axis=0)), max_cta=med(ev.max(axis=0))),
                    feedback_ns=dict(median_cta=med(np.median(fb, axis=0)), max_cta=med(fb.max(axis=0))),
                    correct_push_ns=dict(median_cta=med(np.median(pb, axis=0)), max_cta=med(pb.max(axis=0))),
                    done_spread_ns=med(h[:, :, 1].max(axis=0) - h[:, :, 1].min(axis=0)),
                    pub_skew_ns=med(h[:, :, 0].max(axis=0) - np.median(h[:, :, 0], axis=0)),
                    decide_ns=med(np.median((h[:, :, 8] - h[:, :, 2]) / cyc, axis=0)),
                    prep_ns=med(np.median((h[:, :, 9] - h[:, :, 8]) / cyc, axis=0)),
                    prep_warm_ns=med(np.median((h[:, :, 10] - h[:, :, 9]) / cyc, axis=0)),
                    count_own_ns=med(np.median((h[:, :, 3] - h[:, :, 10]) / cyc, axis=0)),
                    count_ns=med(np.median((h[:, :, 11] - h[:, :, 10]) / cyc, axis=0)),
                    own_events_ns=med(np.median((h[:, :, 12] - h[:, :, 11]) / cyc, axis=0)),
                    own_events_max_ns=med(((h[:, :, 12] - h[:, :, 11]) / cyc).max(axis=0)),
                    count_max_ns=med(((h[:, :, 11] - h[:, :, 10]) / cyc).max(axis=0)),
                    events_barrier_ns=med(np.median((h[:, :, 3] - h[:, :, 12]) / cyc, axis=0)),
                    fb_ns_by_nwork=fb_by_nwork,
                    nwork_max_cta=np.percentile(nw_max, [10, 50, 90]).tolist(),
                    nwork_mean_cta=float(nw.mean()),
                    entries=np.percentile(ent, [10, 50, 90]).tolist(),
                    events_ns_by_entries={b: round(float(np.median(ev[:, (ent >= lo) & (ent < hi)])), 1)
                                          for b, (lo, hi) in {"<=64": (0, 65), "65-512": (65, 513),
                                                              "513-2048": (513, 2049), ">2048": (2049, 1e9)}.items()
                                          if ((ent >= lo) & (ent < hi)).sum() > 5},
                    next_latency_ns=np.percentile(lat, [10, 50, 90]).round().tolist() if lat else None)
                names = {0: "poll", 1: "decide", 2: "ev_prep", 15: "ev_count_own", 3: "feedback",
                         13: "nw_wait", 14: "nw_eval", 4: "nw_push"}
                nne = max(1.0, p[0, 9])
                tot = p[:, 12].mean()
                phases.append(dict(
                    share={n: round(p[:, q].mean() / tot, 4) for q, n in names.items()},
                    ns_per_nonempty={n: round(p[:, q].mean() / nne / 1.9, 1) for q, n in names.items()},
                    windows=int(p[0, 8]), nonempty=int(p[0, 9]), heavy=int(p[0, 10]),
                    staged=int(p[0, 11]), loop_cycles=int(tot), timeline=timeline))
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
                   stats=sess.stats_dict(), phases=phases)
        out.append(rec)
        print(json.dumps(rec), flush=True)
        del sess
    _lib.call("tmb_set_option", b"train.spec_window", 16)
    _lib.call("tmb_set_option", b"train.spec_entries", 64)


if __name__ == "__main__":
    main()
