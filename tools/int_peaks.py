"""Measure the integer-pipe issue rates and the cross-SM signal latency on the
box (roofline denominators for the integer / latency bound kernels).

    python tools/int_peaks.py [--out profiles/r02_int_peaks.json]

Per op: lane-ops per SM per clock (one CTA of 1024 threads per SM, 8
dependent chains per thread), the SM clock the CTAs ran at, and the implied
whole-GPU peak at that clock.  Ping-pong: one write observed by a peer SM
through L2 (ld.relaxed.gpu poll), in ns and SM cycles.
"""

from __future__ import annotations

import argparse
import ctypes as ct
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

OPS = ["LOP3", "IADD3", "SHF", "IMAD", "IMAD.WIDE (+IADD3 pair as ptxas emits mad.wide)",
       "POPC", "PRMT", "LOP3+IMAD interleaved", "SplitMix64 draw + threshold compare"]


def measure(iters: int = 512, threads: int = 1024):
    from paper_2405_04212_b200 import _lib
    sm = ct.c_int()
    maj, mnr, smem = ct.c_int(), ct.c_int(), ct.c_int()
    l2 = ct.c_int64()
    _lib.call("tmb_device_info", 0, ct.byref(sm), ct.byref(maj), ct.byref(mnr), ct.byref(l2),
              ct.byref(smem))
    out = {"sm_count": sm.value, "threads_per_cta": threads, "ops": {}}
    for op, name in enumerate(OPS):
        r, mhz = ct.c_double(), ct.c_double()
        _lib.call("tmb_microbench_pipe", op, sm.value, threads, iters, ct.byref(r), ct.byref(mhz))
        out["ops"][name] = {"per_clk_per_sm": r.value, "sm_mhz": mhz.value,
                            "gpu_peak_G_per_s": r.value * sm.value * mhz.value / 1e3}
    pp = {}
    for mode, name in ((0, "st.relaxed"), (1, "red.relaxed.add")):
        ns, cyc = ct.c_double(), ct.c_double()
        _lib.call("tmb_microbench_pingpong", mode, 20000, ct.byref(ns), ct.byref(cyc))
        pp[name] = {"ns_per_hop": ns.value, "sm_cycles_per_hop": cyc.value}
    out["pingpong_l2"] = pp
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    res = measure()
    txt = json.dumps(res, indent=1)
    print(txt)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(txt + "\n")


if __name__ == "__main__":
    main()
