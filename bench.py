"""Benchmark: BASELINE.json metric "train examples/sec; inference examples/sec
at 1/2/4/8 B200 vs roofline".

Default workload (the ONE JSON line's headline): configs[1], MNIST-shaped
Coalesced-TM training (784 features / 1568 literals, 2000 clauses, 10
classes, T=5000, s=10, 60000 examples).  A step is one training epoch over
the 60000 examples (one launch of the fused persistent kernel).  The line
also carries a "secondary" object for configs[2] (batched inference over
2^22 examples, 10000 clauses x 20 includes, 4096 features).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--workload c2-train|c3-infer|c4-train|c5-sparse]

N > 1 (torchrun, NCCL): training is sequential per example, so
each rank trains an independent replica (different model seed) -- "replicas
only", weak scaling; inference shards examples across ranks.  Times are CUDA
events on the launching stream, max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

PEAKS = {}
try:
    with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
        PEAKS = json.load(fh)
except OSError:
    pass
HBM_PEAK = float(PEAKS.get("hbm_gbs", 6650.0))
HBM_PEAK_SRC = "measured" if "hbm_gbs" in PEAKS else "fallback"


# config.workload of every workload: the b200 arm and the reference arm print
# the same string (the reference arm times a bounded sample of it)
WORKLOADS = {
    "c2-train": "configs[1]: MNIST-shaped CoTM training, step = 1 epoch",
    "c1-train": ("configs[0]: Noisy-XOR, 10 clauses, T=15, s=3.9; step = the 5-seed study: five "
                 "20-epoch trainings of 5000 examples (model seeds 0..4), concurrent on five "
                 "streams / SMs"),
    "c3-infer": ("configs[2]: 2^22 examples x 4096 features, 10000 clauses x 20 includes, 10 "
                 "classes; step = one pass over all examples"),
    "c4-train": ("configs[3]: bag-of-words training, 10000 clauses x 20000 literal positions, "
                 "step = 5000 consecutive examples of the epoch"),
    "c5-sparse": ("configs[4]: SparseTM, 10^6-literal vocabulary, 2000 clauses, capacity 64; "
                  "step = 100000 consecutive training documents"),
}


def sweep_workload(world: int, step_n: int) -> str:
    return (f"configs[3] sweep: 8 independent bag-of-words trainings (10000 clauses x 20000 "
            f"positions), job j on rank j mod {world}; step = {step_n} examples of every job")


def ncu_traffic(kernel: str):
    """DRAM bytes (read + write) per launch of `kernel` from the newest
    committed `ncu --set full` summary under profiles/ (captured on the same
    workload by tools/profile_round.sh), with its source; (None, None) if
    absent."""
    import glob
    units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    for f in sorted(glob.glob(os.path.join(REPO, "profiles", "*_ncu_full_summary.json")),
                    reverse=True):
        try:
            data = json.load(open(f))
        except (OSError, ValueError):
            continue
        for rec in data.values():
            if kernel in rec.get("Kernel Name", ""):
                tot = 0.0
                for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    val, unit = rec[key].split()
                    tot += float(val) * units[unit]
                return tot, os.path.basename(f)
    return None, None


def ncu_pipes(kernel: str):
    """Pipe utilisation of `kernel` from the same committed ncu summary as
    ncu_traffic: ALU / FMA pipe activity, issue-slot use and shared-memory
    wavefronts, each as % of its peak (the integer-pipe roofline of a
    kernel that is neither HBM- nor tensor-bound), or None."""
    import glob
    keys = {"alu_pipe_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "issue_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed"}
    for f in sorted(glob.glob(os.path.join(REPO, "profiles", "*_ncu_full_summary.json")),
                    reverse=True):
        try:
            data = json.load(open(f))
        except (OSError, ValueError):
            continue
        for rec in data.values():
            if kernel in rec.get("Kernel Name", ""):
                out = {"source": os.path.basename(f), "kernel": rec["Kernel Name"]}
                for name, key in keys.items():
                    if key in rec:
                        out[name] = float(rec[key].split()[0])
                return out
    return None


# ---------------------------------------------------------------- infra --

def dist_init():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    import torch
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100", "-f", self.path],
                stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *exc):
        time.sleep(0.15)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx = max(mx, float(parts[2]))
                except ValueError:
                    continue
                for n, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
            os.unlink(self.path)
        except OSError:
            pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def flush_l2(buf):
    buf.zero_()


def host_desc():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return model, os.cpu_count() or 1


# --------------------------------------------------------- c2 training --

_LIVE = {}


def live_peaks():
    """Integer-pipe and cross-SM latency peaks measured on THIS box right now
    (tmb_microbench_pipe / tmb_microbench_pingpong; tools/int_peaks.py
    writes the full table, profiles/r02_int_peaks.json): LOP3 and full
    SplitMix64 draw+compare rates per SM per clock, the SM clock they ran
    at, and one L2 hop (a red.relaxed.gpu observed by a peer SM's poll)."""
    if _LIVE:
        return _LIVE
    import ctypes as ct

    import torch

    from paper_2405_04212_b200 import _lib
    sm = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    out = {"sm_count": sm, "source": "measured live (tmb_microbench_pipe, tmb_microbench_pingpong)"}
    for op, name in ((0, "lop3"), (8, "draw")):
        r, mhz = ct.c_double(), ct.c_double()
        _lib.call("tmb_microbench_pipe", op, sm, 1024, 256, ct.byref(r), ct.byref(mhz))
        out[f"{name}_per_clk_per_sm"] = r.value
        out[f"{name}_sm_mhz"] = mhz.value
        out[f"{name}_peak_per_s"] = r.value * sm * mhz.value * 1e6
    ns, cyc = ct.c_double(), ct.c_double()
    _lib.call("tmb_microbench_pingpong", 1, 20000, ct.byref(ns), ct.byref(cyc))
    out["l2_hop_ns"] = ns.value
    out["l2_hop_cycles"] = cyc.value
    _LIVE.update(out)
    return _LIVE


def c2_data(rank: int):
    from paper_2405_04212_b200 import datasets
    return datasets.mnist_shaped(data_seed=7)


def oracle_train_rate(cfg, states, weights, counters, fb_counter, x_lit, labels, order,
                      budget_s: float):
    """Time the CPU oracle (C restatement of the reference train loop) from a
    given model state on a prefix of `order`; returns (ex/s, examples)."""
    from oracle import oracle
    st = oracle.OracleTrainState(states.copy(), weights.copy(), counters.copy().view(np.uint64),
                                 fb_counter, 0)
    done, t0 = 0, time.perf_counter()
    chunk = 100
    while time.perf_counter() - t0 < budget_s and done < len(order):
        oracle.train_steps(cfg, st, x_lit, labels, order[done:done + chunk])
        done += min(chunk, len(order) - done)
    dt = time.perf_counter() - t0
    return done / dt, done, dt


def bench_c2_train(args, rank, world, local):
    import torch

    import paper_2405_04212_b200 as tmb
    from paper_2405_04212_b200 import _lib, datasets
    (tx, ty), (ex, ey) = c2_data(rank)
    cfg = tmb.Config(**datasets.mnist_shaped_config_kwargs(seed=rank))
    sess = tmb.DenseTrainSession(cfg, tx, ty, n_cta=args.train_cta, threads=args.train_threads)
    N = len(ty)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(args.warmup):
        sess.run_epoch()
    torch.cuda.synchronize()
    # model state at the start of the timed region (for the CPU baseline)
    st0 = sess.states.cpu().numpy().copy()
    w0 = sess.weights.cpu().numpy().copy()
    c0 = sess.block_counters.cpu().numpy().copy()
    fb0 = sess.fb_counter
    stats0 = sess.stats_dict()
    snap = sess.snapshot()  # e2e replays the same epochs from this state
    launches0 = _lib.launch_count()
    orders = [sess.next_order().astype(np.int32) for _ in range(args.steps)]
    orders_dev = [torch.from_numpy(o).cuda() for o in orders]
    k_ms = []
    barrier(world)
    with ClockSampler(local) as clk:
        barrier(world)
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for i in range(args.steps):
            flush_l2(flush)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            sess.run_steps(orders_dev[i])
            b.record(stream)
            k_ms.append((a, b))
        t_end.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    elapsed_ms = t_start.elapsed_time(t_end)
    launches = _lib.launch_count() - launches0
    kern_ms = [a.elapsed_time(b) for a, b in k_ms]
    stats1 = sess.stats_dict()
    dstats = {k: stats1[k] - stats0[k] for k in stats1}
    elapsed_ms = max_over_ranks(elapsed_ms, world)
    total_examples = args.steps * N * world
    value = total_examples / (elapsed_ms / 1e3)

    # ---- end to end through the public API with host buffers (per step:
    # H2D of the epoch's features+labels from pinned memory, device packing,
    # host shuffle, the fused kernel, D2H of the trained model).  Replays the
    # timed epochs from the same model state, so the work is identical.
    sess.restore(snap)
    xp = torch.from_numpy(np.ascontiguousarray(tx)).pin_memory()
    yp = torch.from_numpy(np.ascontiguousarray(ty.astype(np.int32))).pin_memory()
    st_host = torch.empty(sess.states.shape, dtype=torch.int8).pin_memory()
    w_host = torch.empty(sess.weights.shape, dtype=torch.int32).pin_memory()
    barrier(world)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        xd = xp.to("cuda", non_blocking=True)
        sess.labels = yp.to("cuda", non_blocking=True)
        from paper_2405_04212_b200.runtime import ptr, stream_ptr
        _lib.call("tmb_pack_literals", ptr(xd), N, cfg.n_literals, 1, ptr(sess.lit_words),
                  stream_ptr())
        order = sess.next_order().astype(np.int32)
        od = torch.from_numpy(order).pin_memory().to("cuda", non_blocking=True)
        sess.run_steps(od)
        st_host.copy_(sess.states, non_blocking=True)
        w_host.copy_(sess.weights, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1), world)
    e2e_value = total_examples / (e2e_ms / 1e3)
    h2d = tx.nbytes + N * 4 + N * 4
    d2h = sess.states.numel() + 4 * sess.weights.numel()

    # ---- untimed replay of the same epochs with the per-step trace: which
    # steps were non-empty (update probability of the label or the negative
    # class > 0, feedback.py:33-44) -- each of those needs one grid exchange
    # before the next step can be decided; empty steps need none
    sess.restore(snap)
    trace = torch.zeros((N, 4), dtype=torch.int64, device="cuda")
    _lib.call("tmb_trainer_set_trace", sess._h, trace.data_ptr())
    n_nonempty = 0
    for i in range(args.steps):
        sess.next_order()
        sess.run_steps(orders_dev[i])
        t = trace.cpu().numpy()
        n_nonempty += int(((t[:, 1] < cfg.threshold) | (t[:, 2] > -cfg.threshold)).sum())
    _lib.call("tmb_trainer_set_trace", sess._h, None)
    nonempty_frac = n_nonempty / (args.steps * N)

    # ---- roofline of the dominant kernel (k_train_spec)
    kname = sess.launch.get("kernel", "k_train_fast")
    per_launch_ms = float(np.mean(kern_ms))
    ex_per_launch = N
    P, C, W = cfg.n_literal_positions, cfg.n_clauses, (cfg.n_literal_positions + 31) // 32
    # algorithmic HBM bytes per example: literal row (W words) + label +
    # order entry; the model is on-chip for the whole launch.
    hbm_bytes_ex = 4 * W + 4 + 4
    achieved_gbs = hbm_bytes_ex * ex_per_launch / (per_launch_ms / 1e3) / 1e9
    ev_per_ex = dstats["events"] / max(dstats["examples"], 1)
    draws_per_ex = dstats["draws"] / max(dstats["examples"], 1)
    sm_count = torch.cuda.get_device_properties(local).multi_processor_count
    clocks = clk.summary()
    f_sm = (clocks["sm_mhz"] or 1965.0) * 1e6
    # integer work per example at the measured peaks: every reference draw
    # (one SplitMix64 + threshold compare each; the kernel evaluates all of
    # them branch-free) plus the bit-packed clause evaluation (C*W LOP3)
    lp = live_peaks()
    int_s_ex = draws_per_ex / lp["draw_peak_per_s"] + C * W / lp["lop3_peak_per_s"]
    tr_train, tr_train_src = ncu_traffic(kname)
    # latency floors of sequential online training: (hardware) one L2 hop
    # between SMs per example -- every example's decision needs every CTA's
    # partial class sums; (protocol) the trainer's own exchange with no work
    import ctypes as ct
    floor = ct.c_double()
    _lib.call("tmb_microbench_allreduce", sess.launch["n_cta"], 512, 20000, 4, ct.byref(floor))
    us_ex = per_launch_ms * 1e3 / ex_per_launch
    hop_us = lp["l2_hop_ns"] / 1e3

    line = {
        "metric": "train examples/sec (configs[1] MNIST-shaped CoTM training)",
        "value": value, "unit": "examples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "int8 TA states / int32 weights / u64 SplitMix64",
        "data": "synthetic (seeded MNIST-shaped generator, datasets.mnist_shaped)",
        "config": {"workload": WORKLOADS["c2-train"],
                   "n_features": 784, "n_literals": P, "n_clauses": C, "n_classes": 10,
                   "threshold": cfg.threshold, "s": cfg.s, "examples_per_epoch": N,
                   "epochs_timed": f"{args.warmup + 1}..{args.warmup + args.steps}",
                   "parallelism": f"replicas x{world} (online training is sequential)",
                   "l2": "256 MiB buffer written before every timed epoch",
                   "launch": sess.launch},
        "gpu_launches": int(launches),
        "work": {"events_per_example": ev_per_ex, "draws_per_example": draws_per_ex,
                 "type_i_per_example": dstats["type_i"] / max(dstats["examples"], 1),
                 "state_updates_per_example": dstats["state_updates"] / max(dstats["examples"], 1)},
        "roofline": {"kernel": f"{kname} (fused persistent trainer"
                               + (f", speculative windows of {sess.launch['spec_window']} steps)"
                                  if sess.launch.get("spec_window") else ")"),
                     "bound": "latency",
                     "achieved": 1e6 / us_ex, "peak": 1e6 / (hop_us * nonempty_frac),
                     "unit": "examples/s",
                     "frac": hop_us * nonempty_frac / us_ex, "traffic": tr_train,
                     "traffic_source": tr_train_src,
                     "achieved_us_per_example": us_ex,
                     "floor_us_per_example": hop_us * nonempty_frac,
                     "nonempty_fraction": nonempty_frac,
                     "achieved_us_per_nonempty_step": us_ex / max(nonempty_frac, 1e-9),
                     "floor": "one cross-SM L2 hop (red.relaxed.gpu observed by a peer SM's "
                              "ld.relaxed.gpu poll, measured live by tmb_microbench_pingpong) "
                              "per NON-EMPTY step: such a step's feedback changes the clauses "
                              "the next step is evaluated with, and its decision needs every "
                              "CTA's partial class sums (SPEC.md:360); runs of empty steps "
                              "(both update probabilities 0) are decided together, one "
                              "exchange per window",
                     "peak_source": lp["source"], "avg_launch_ms": per_launch_ms},
        "roofline_int": {"bound": "int (SplitMix64 draws + LOP3 evaluation at measured "
                                  "per-SM rates)",
                         "frac": int_s_ex * 1e6 / us_ex,
                         "int_us_per_example": int_s_ex * 1e6, "achieved_us_per_example": us_ex,
                         "draw_peak_per_s": lp["draw_peak_per_s"],
                         "lop3_peak_per_s": lp["lop3_peak_per_s"],
                         "ops_per_example": {"draws": draws_per_ex, "lop3": C * W}},
        "roofline_hbm": {"achieved": achieved_gbs, "peak": HBM_PEAK, "unit": "GB/s",
                         "frac": achieved_gbs / HBM_PEAK, "peak_source": HBM_PEAK_SRC,
                         "algorithmic_bytes_per_example": hbm_bytes_ex,
                         "traffic": tr_train,
                         "traffic_note": "ncu DRAM bytes of one launch (one epoch): the per-step "
                                         "records (literal row + bucketed 16-bit flag keys, "
                                         "~17 KB/step) read once from HBM (the other 147 CTAs "
                                         "hit L2) -- a deliberate trade, ~10 GB/s, not binding"},
        "pipes_ncu": ncu_pipes(kname),
        "roofline_latency": {"bound": "the trainer's own exchange protocol, no work, once per "
                                      "non-empty step",
                             "floor_us_per_example": floor.value * nonempty_frac,
                             "achieved_us_per_example": us_ex,
                             "frac": floor.value * nonempty_frac / us_ex,
                             "floor_source": "tmb_microbench_allreduce mode 4 (two-word relaxed "
                                             "red + warp spin), same CTA count, x the "
                                             "non-empty fraction"},
        "clocks": clocks,
        "e2e": {"value": e2e_value, "unit": "examples/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h),
                "path": "pinned host features/labels -> H2D -> tmb_pack_literals -> host "
                        "Fisher-Yates -> tmb_trainer_run -> D2H model"},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # N=1 only (contract)
        from oracle import oracle
        x_lit = oracle.augment_literals(tx)
        rate, n_done, dt = oracle_train_rate(cfg, st0, w0, c0, fb0, x_lit, ty,
                                             orders[0].astype(np.int64), args.cpu_seconds)
        model_name, ncpu = host_desc()
        line["cpu_baseline"] = {"value": rate, "unit": "examples/s", "cores": 1, "kind": "port",
                                "sample": f"oracle C port of executor.train, {n_done} examples "
                                          f"of timed epoch {args.warmup + 1} from the same "
                                          f"model state ({dt:.1f}s, 1 thread; training is "
                                          f"sequential with n_blocks=1)",
                                "host": model_name, "host_cores": ncpu}
    if not args.no_secondary:
        line["secondary"] = bench_c3_infer(args, rank, world, local, embedded=True)
    return line


# ------------------------------------------------------- c1 training --

def bench_c1_train(args, rank, world, local):
    """configs[0]: Noisy-XOR CoTM (12 features, 10 clauses, 2 classes, T=15,
    s=3.9), 5000 training examples, 20 epochs, evaluated over model seeds
    0..4 (the north star's 5-seed criterion).  Step = the whole 5-seed study:
    five complete 20-epoch trainings, run concurrently -- each session's
    tiny-bank trainer (k_train_tiny) on its own CUDA stream, so the five land on five SMs
    (500 000 examples per step); epoch orders from the host shuffle are
    precomputed.  The per-training latency (one seed's 20 epochs alone on its
    stream) is reported beside it.  e2e = the public train(cfg, train, eval,
    n_epochs=20) call for each of the five seeds in turn (H2D of the data,
    per-epoch test accuracy, D2H of the model).  N > 1: replicas."""
    import torch

    import paper_2405_04212_b200 as tmb
    from paper_2405_04212_b200 import _lib, datasets
    (tx, ty), (ex, ey) = datasets.noisy_xor()
    n_epochs, N, n_seeds = 20, len(ty), 5
    stream = torch.cuda.current_stream()
    streams = [torch.cuda.Stream() for _ in range(n_seeds)]

    def seed_of(i):
        return i % 5 if world == 1 else 5 * rank + i % 5

    def prepare(i):
        cfg = tmb.Config(**datasets.noisy_xor_config_kwargs(seed=seed_of(i)))
        sess = tmb.DenseTrainSession(cfg, tx, ty)
        orders = [torch.from_numpy(sess.next_order().astype(np.int32)).cuda()
                  for _ in range(n_epochs)]
        return sess, orders

    def study(preps, per_stream_events=None):
        """The five trainings, one per stream, all epochs issued."""
        for si, (sess, orders) in enumerate(preps):
            with torch.cuda.stream(streams[si]):
                if per_stream_events is not None:
                    per_stream_events[si][0].record(streams[si])
                for o in orders:
                    sess.run_steps(o)
                if per_stream_events is not None:
                    per_stream_events[si][1].record(streams[si])

    for i in range(args.warmup):
        study([prepare(n_seeds * i + s_) for s_ in range(n_seeds)])
    torch.cuda.synchronize()
    launches0 = _lib.launch_count()
    steps_preps = [[prepare(n_seeds * (args.warmup + i) + s_) for s_ in range(n_seeds)]
                   for i in range(args.steps)]
    torch.cuda.synchronize()
    ev = []
    lat = []
    barrier(world)
    with ClockSampler(local) as clk:
        for preps in steps_preps:
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            pse = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(n_seeds)]
            a.record(stream)
            for st in streams:
                st.wait_event(a)
            study(preps, pse)
            for st in streams:
                stream.wait_stream(st)
            b.record(stream)
            ev.append((a, b))
            lat.append(pse)
        torch.cuda.synchronize()
        barrier(world)
    launches = _lib.launch_count() - launches0
    ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in ev), world)
    n_ex = args.steps * n_seeds * n_epochs * N
    value = n_ex * world / (ms / 1e3)
    us_step = ms * 1e3 / n_ex
    seed_ms = [x.elapsed_time(y) for pse in lat for x, y in pse]
    us_training_example = float(np.mean(seed_ms)) * 1e3 / (n_epochs * N)
    preps = [p_ for preps_ in steps_preps for p_ in preps_]
    accs = []
    draws = sum(sess.stats_dict()["draws"] for sess, _ in preps)
    for sess, _ in preps:
        accs.append(tmb.evaluate(sess.model(), (ex, ey)))
    draws_ex = draws / n_ex
    lp = live_peaks()
    sm_count = torch.cuda.get_device_properties(local).multi_processor_count
    # one warp issues on one of the SM's four schedulers: its share of the
    # measured per-SM SplitMix64 draw rate is the integer peak it can reach
    warp_draw_peak = lp["draw_peak_per_s"] / sm_count / 4
    # e2e through the public train() (per-epoch evaluation included, as the
    # reference's train(eval_data=...) does), the five seeds in turn
    barrier(world)
    t0 = time.perf_counter()
    e2e_acc = []
    for i in range(args.steps * n_seeds):
        cfg = tmb.Config(**datasets.noisy_xor_config_kwargs(seed=seed_of(i)))
        run = tmb.train(cfg, (tx, ty), (ex, ey), n_epochs=n_epochs)
        e2e_acc.append(run.epoch_metrics[-1].accuracy)
    e2e_s = max_over_ranks(time.perf_counter() - t0, world)
    line = {
        "metric": "train examples/sec (configs[0] Noisy-XOR CoTM training)",
        "value": value, "unit": "examples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "us_per_example": us_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "int8 TA states / int32 weights / u64 SplitMix64",
        "data": "synthetic (datasets.noisy_xor: 12 Bernoulli(0.5) features, 40% train "
                "label noise)",
        "config": {"workload": WORKLOADS["c1-train"],
                   "latency_us_per_example_one_training": us_training_example,
                   "launch": preps[0][0].launch,
                   "parallelism": f"replicas x{world} (online training is sequential)",
                   "l2": "model and data (60 KB) are L2/SMEM-resident by design; nothing to "
                         "flush that the workload re-reads"},
        "gpu_launches": int(launches),
        "accuracy": {"test_accuracy_per_step": accs, "mean": float(np.mean(accs))},
        "roofline": {"kernel": preps[0][0].launch.get("kernel", "k_train_warp"),
                     "bound": "latency (one CTA per training, one warp per clause: the "
                              "per-example chain eval -> block barrier -> class sums -> "
                              "decision -> feedback; no parallelism across examples)",
                     "achieved": 1e6 / us_step, "unit": "examples/s",
                     "peak": n_seeds * warp_draw_peak / max(draws_ex, 1e-9),
                     "frac": (1e6 / us_step) * draws_ex / (n_seeds * warp_draw_peak),
                     "draws_per_example": draws_ex,
                     "peak_note": "the reference draws of an example at one scheduler's share "
                                  "per training of the measured per-SM SplitMix64 draw rate "
                                  "(k_train_warp's footprint; k_train_tiny spreads a training "
                                  "over its SM's four schedulers, so the fraction is of a "
                                  "quarter of the five SMs it occupies)",
                     "peak_source": lp["source"]},
        "clocks": clk.summary(),
        "e2e": {"value": n_ex * world / e2e_s, "unit": "examples/s",
                "h2d_bytes_per_step": int(n_seeds * (tx.nbytes + ex.nbytes + 4 * N)),
                "d2h_bytes_per_step": int(n_seeds * (n_epochs * 8 * len(ey) + 10 * 24 + 10 * 2 * 4)),
                "path": "tmb.train(cfg, (x, y), (x_test, y_test), n_epochs=20) for seeds 0..4 in "
                        "turn (the public call is synchronous): host arrays in, per-epoch test "
                        "predictions and the model out",
                "test_accuracy_per_step": e2e_acc},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # N=1 only (contract)
        from oracle import oracle
        model_name, ncpu = host_desc()
        t = time.perf_counter()
        o_acc = []
        for sd in range(5):
            cfg = tmb.Config(**datasets.noisy_xor_config_kwargs(seed=sd))
            st, acc = oracle.train(cfg, tx, ty, n_epochs)
            _, pred = oracle.batch_votes(st.states, st.weights, oracle.augment_literals(ex))
            o_acc.append(float(np.mean(pred == ey)))
        dt = time.perf_counter() - t
        line["cpu_baseline"] = {"value": 5 * n_epochs * N / dt, "unit": "examples/s",
                                "cores": 1, "kind": "port",
                                "sample": f"oracle C port of executor.train, seeds 0..4 x 20 "
                                          f"epochs x 5000 examples ({dt:.1f}s, 1 thread)",
                                "host": model_name, "host_cores": ncpu,
                                "mean_test_accuracy_seeds_0_4": float(np.mean(o_acc))}
    return line


# -------------------------------------------------------- c3 inference --

def c3_inputs_device(n: int, start: int, data_seed: int = 3, F: int = 4096):
    """Device-side synthesis of the counter-based C3 inputs (same bits as
    datasets.inference_examples)."""
    from paper_2405_04212_b200 import datasets
    return datasets.inference_examples_device(data_seed, start, n, F)


def bench_c3_infer(args, rank, world, local, embedded=False):
    import torch

    import paper_2405_04212_b200 as tmb
    from paper_2405_04212_b200 import _lib, datasets
    F, C, K = 4096, 10000, 10
    N_total = args.c3_examples
    per = N_total // world
    start = rank * per
    n = per if rank < world - 1 else N_total - start
    m = datasets.inference_model(model_seed=11, n_features=F, n_clauses=C, n_classes=K)
    bank = tmb.DenseClauseBank(tmb.Config(n_literals=F, n_clauses=C, n_classes=K, s=2.0,
                                          threshold=100))
    bank.states[:] = m.states
    bank.weights[:] = m.weights
    model = tmb.CompiledModel.from_bank(bank)
    x = c3_inputs_device(n, start)
    pred = torch.empty(n, dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        model.infer_device(x, pred_dev=pred)
    _lib.call("tmb_infer_status", None)
    launches0 = _lib.launch_count()
    evs = []
    barrier(world)
    with ClockSampler(local) as clk:
        barrier(world)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            model.infer_device(x, pred_dev=pred)
            b.record(stream)
            evs.append((a, b))
        t1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    launches = _lib.launch_count() - launches0
    ms = max_over_ranks(t0.elapsed_time(t1), world)
    value = N_total * args.steps / (ms / 1e3)
    per_launch_ms = float(np.mean([a.elapsed_time(b) for a, b in evs]))
    bytes_ex = F + 8  # uint8 features in, int64 prediction out
    achieved = bytes_ex * n / (per_launch_ms / 1e3) / 1e9
    # parity sample against the CPU oracle
    parity = None
    if rank == 0:
        from oracle import oracle
        xs = x[:1024].cpu().numpy()
        _, op = oracle.batch_votes(m.states, m.weights, oracle.augment_literals(xs), nthreads=8)
        parity = bool(np.array_equal(pred[:1024].cpu().numpy(), op))
    # e2e: host (pinned) uint8 features -> tmbh_infer (3-deep pipeline of
    # ~48 MB chunks: H2D / kernel / D2H overlap) -> host predictions; beside
    # it the pinned H2D copy peak of the same bytes (one cudaMemcpyAsync)
    n_e2e = min(n, args.c3_e2e_examples)
    xh = torch.empty((n_e2e, F), dtype=torch.uint8).pin_memory()
    xh.copy_(x[:n_e2e])
    ph = np.empty(n_e2e, dtype=np.int64)
    from paper_2405_04212_b200.runtime import np_ptr
    _lib.call("tmbh_infer", model._h, ct_ptr(xh), n_e2e, None, np_ptr(ph), 0)
    xd_copy = torch.empty_like(xh, device="cuda")
    for _ in range(2):
        xd_copy.copy_(xh, non_blocking=True)
    torch.cuda.synchronize()
    ca, cb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ca.record(stream)
    for _ in range(3):
        xd_copy.copy_(xh, non_blocking=True)
    cb.record(stream)
    torch.cuda.synchronize()
    h2d_peak = 3 * xh.numel() / (ca.elapsed_time(cb) / 1e3) / 1e9
    del xd_copy
    barrier(world)
    t = time.perf_counter()
    for _ in range(args.steps):
        _lib.call("tmbh_infer", model._h, ct_ptr(xh), n_e2e, None, np_ptr(ph), 0)
    e2e_s = max_over_ranks(time.perf_counter() - t, world)
    e2e_value = n_e2e * world * args.steps / e2e_s
    # the same examples as bit-packed words (feature f = bit f%64 of word
    # f//64; the generator's raw stream words): device timing + e2e from
    # pinned host words through the public API
    xs_cpu = x[:args.c3_cpu_examples].cpu().numpy() if rank == 0 else None
    del x
    torch.cuda.empty_cache()
    W = (F + 63) // 64
    xb = torch.empty((n, W), dtype=torch.int64, device="cuda")
    from paper_2405_04212_b200.runtime import ptr, stream_ptr
    _lib.call("tmb_stream_u64_block", datasets.inference_stream_seed(3), start * W, n * W,
              ptr(xb), stream_ptr())
    predb = torch.empty(n, dtype=torch.int64, device="cuda")
    for _ in range(2):
        model.infer_device_packed(xb, pred_dev=predb)
    torch.cuda.synchronize()
    pa = torch.cuda.Event(enable_timing=True)
    pb = torch.cuda.Event(enable_timing=True)
    pa.record(stream)
    for _ in range(args.steps):
        model.infer_device_packed(xb, pred_dev=predb)
    pb.record(stream)
    torch.cuda.synchronize()
    packed_ms = max_over_ranks(pa.elapsed_time(pb), world) / args.steps
    packed_same = bool(torch.equal(predb, pred))
    xbh = xb[:n_e2e].cpu().pin_memory()
    prh = torch.empty(n_e2e, dtype=torch.int64).pin_memory()
    barrier(world)
    pe0 = torch.cuda.Event(enable_timing=True)
    pe1 = torch.cuda.Event(enable_timing=True)
    pe0.record(stream)
    for _ in range(args.steps):
        xbd = xbh.to("cuda", non_blocking=True)
        model.infer_device_packed(xbd, pred_dev=predb[:n_e2e])
        prh.copy_(predb[:n_e2e], non_blocking=True)
    pe1.record(stream)
    torch.cuda.synchronize()
    packed_e2e = n_e2e * world * args.steps / (max_over_ranks(pe0.elapsed_time(pe1), world) / 1e3)
    del xb
    tr_inf, tr_inf_src = ncu_traffic("k_infer_solo<0>")
    if tr_inf is not None:
        tr_inf *= (N_total / world) / (1 << 22)  # captured on the 2^22-example launch
    out = {
        "metric": "inference examples/sec (configs[2] batched CoTM inference)",
        "value": value, "unit": "examples/s", "n_gpus": world, "steps": args.steps,
        "ms_per_step": ms / args.steps,
        "config": {"workload": WORKLOADS["c3-infer"],
                   "examples": N_total, "sharding": f"contiguous example ranges over {world}",
                   "rules": model.n_rules, "l2": "inputs (17 GB) far larger than L2"},
        "gpu_launches": int(launches),
        "parity_sample_1024": parity,
        "roofline": {"kernel": "k_infer_solo (per-CTA bit-sliced rule evaluation, rule heads "
                               "streamed from L2)",
                     "bound": "hbm",
                     "achieved": achieved, "peak": HBM_PEAK, "unit": "GB/s",
                     "frac": achieved / HBM_PEAK, "traffic": tr_inf, "traffic_source": tr_inf_src,
                     "peak_source": HBM_PEAK_SRC,
                     "algorithmic_bytes_per_example": bytes_ex, "avg_launch_ms": per_launch_ms},
        "pipes_ncu": ncu_pipes("k_infer_solo<0>"),
        "bit_packed_input": {
            "note": "same examples and model, features as uint64 words (tmb_infer_packed); "
                    "not the reference's input format, so not the headline",
            "value": N_total / (packed_ms / 1e3), "unit": "examples/s", "ms_per_step": packed_ms,
            "same_predictions_as_uint8": packed_same,
            "hbm_bytes_per_example": 8 * W + 8,
            "e2e": {"value": packed_e2e, "unit": "examples/s", "h2d_bytes_per_step": n_e2e * 8 * W,
                    "d2h_bytes_per_step": n_e2e * 8,
                    "path": "pinned host uint64 words -> H2D -> tmb_infer_packed -> D2H"}},
        "clocks": clk.summary(),
        "e2e": {"value": e2e_value, "unit": "examples/s", "h2d_bytes_per_step": n_e2e * F,
                "d2h_bytes_per_step": n_e2e * 8,
                "path": f"pinned host uint8 [{n_e2e}, 4096] -> tmbh_infer (3-deep pipeline of "
                        "~48 MB chunks, buffers kept with the rule set) -> host int64 predictions",
                "h2d_gbs": n_e2e * F * args.steps / e2e_s / 1e9,
                "h2d_pinned_copy_peak_gbs": h2d_peak,
                "h2d_frac_of_peak": n_e2e * F * args.steps / e2e_s / 1e9 / h2d_peak},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # N=1 only (contract)
        from oracle import oracle
        _, ncpu = host_desc()
        xs = xs_cpu
        t = time.perf_counter()
        oracle.batch_votes(m.states, m.weights, oracle.augment_literals(xs), nthreads=ncpu,
                           want_votes=False)
        dt = time.perf_counter() - t
        out["cpu_baseline"] = {"value": len(xs) / dt, "unit": "examples/s", "cores": ncpu,
                               "kind": "port",
                               "sample": f"oracle C port of batch_votes, {len(xs)}-example "
                                         f"prefix, {ncpu} threads ({dt:.1f}s)"}
    torch.cuda.empty_cache()
    return out


def ct_ptr(t):
    import ctypes as ct
    return ct.c_void_p(t.data_ptr())



# ------------------------------------------------------- c4 / c5 rows --

def c4_ncu_sample():
    """DRAM bytes per example of the generic grid trainer from the newest
    committed ncu capture: tools/profile_round.sh captures the bench's own
    first timed c4-train launch (5000 steps after 3 warm-up launches); the
    round-1 summaries hold a 1000-step launch from a fresh model
    (tools/probes/c4_once.py)."""
    tot, src = ncu_traffic("k_train<")
    if tot is None:
        return None
    steps = 1000 if src.startswith("r01") else 5000
    return {"dram_bytes_per_example": tot / steps, "dram_bytes_per_launch": tot, "source": src,
            "sample": ("tools/probes/c4_once.py: 1000 steps from a fresh model" if steps == 1000
                       else "tools/profile_round.sh: the bench's first timed 5000-step launch")}


def bench_c4_train(args, rank, world, local):
    """configs[3]: bag-of-words CoTM training, 10^4 clauses x 2*10^4 literal
    positions (states HBM-resident, 200 MB).  Step = 5000 consecutive
    examples of the running epoch (a fifth of the 25000-example epoch)."""
    import ctypes as ct

    import torch

    import paper_2405_04212_b200 as tmb
    from paper_2405_04212_b200 import _lib, datasets
    (tx, ty), _ = datasets.bag_of_words(data_seed=4 + rank)
    cfg = tmb.Config(**datasets.bag_of_words_config_kwargs(seed=rank))
    sess = tmb.DenseTrainSession(cfg, tx, ty)
    step_n = 5000
    order = torch.from_numpy(sess.next_order().astype(np.int32)).cuda()
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    pos = 0

    def next_slice():
        # the next step_n examples of the running epoch (the next epoch's
        # shuffle once this one is used up: a step never trains fewer)
        nonlocal order, pos
        if pos + step_n > sess.N:
            order = torch.from_numpy(sess.next_order().astype(np.int32)).cuda()
            pos = 0
        sl = order[pos:pos + step_n]
        pos += step_n
        return sl

    for _ in range(args.warmup):
        sess.run_steps(next_slice())
    torch.cuda.synchronize()
    st0 = sess.states.cpu().numpy().copy()
    w0 = sess.weights.cpu().numpy().copy()
    c0 = sess.block_counters.cpu().numpy().copy()
    fb0 = sess.fb_counter
    stats0 = sess.stats_dict()
    snap = sess.snapshot()
    launches0 = _lib.launch_count()
    barrier(world)
    k_ms = []
    timed_slices = []
    with ClockSampler(local) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for i in range(args.steps):
            flush_l2(flush)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            sl = next_slice()
            timed_slices.append(sl)
            a.record(stream)
            sess.run_steps(sl)
            b.record(stream)
            k_ms.append((a, b))
        t_end.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    elapsed_ms = max_over_ranks(t_start.elapsed_time(t_end), world)
    launches = _lib.launch_count() - launches0
    per_launch_ms = float(np.mean([a.elapsed_time(b) for a, b in k_ms]))
    st1 = sess.stats_dict()
    d = {k: st1[k] - stats0[k] for k in st1}
    n_ex = args.steps * step_n
    value = n_ex * world / (elapsed_ms / 1e3)
    P = cfg.n_literal_positions
    # algorithmic HBM bytes: every Type I / II event reads and writes its
    # clause's P int8 states (HBM-resident); plus the literal row
    ev_ex = d["events"] / max(d["examples"], 1)
    bytes_ex = ev_ex * 2 * P + 4 * ((P + 31) // 32) + 8
    achieved = bytes_ex * step_n / (per_launch_ms / 1e3) / 1e9
    draws_ex = d["draws"] / max(d["examples"], 1)
    clocks = clk.summary()
    f_sm = (clocks["sm_mhz"] or 1965.0) * 1e6
    sm_count = torch.cuda.get_device_properties(local).multi_processor_count
    lp = live_peaks()
    int_s_ex = draws_ex / lp["draw_peak_per_s"]
    # e2e: the same slices from the same state through host buffers
    sess.restore(snap)
    from paper_2405_04212_b200.runtime import ptr, stream_ptr
    xp = torch.from_numpy(np.ascontiguousarray(tx)).pin_memory()
    st_host = torch.empty(sess.states.shape, dtype=torch.int8).pin_memory()
    w_host = torch.empty(sess.weights.shape, dtype=torch.int32).pin_memory()
    slices_h = [sl.cpu().pin_memory() for sl in timed_slices]
    barrier(world)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        xd = xp.to("cuda", non_blocking=True)
        _lib.call("tmb_pack_literals", ptr(xd), xp.shape[0], cfg.n_literals, 1,
                  ptr(sess.lit_words), stream_ptr())
        od = slices_h[i].to("cuda", non_blocking=True)
        sess.run_steps(od)
        st_host.copy_(sess.states, non_blocking=True)
        w_host.copy_(sess.weights, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1), world)
    line = {
        "metric": "train examples/sec (configs[3] bag-of-words CoTM training)",
        "value": value, "unit": "examples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "int8 TA states (HBM) / int32 weights / u64 SplitMix64",
        "data": "synthetic (datasets.bag_of_words: Zipf(1.1) documents, planted sets)",
        "config": {"workload": WORKLOADS["c4-train"],
                   "launch": sess.launch, "parallelism": f"replicas x{world}",
                   "l2": "256 MiB buffer written before every timed step"},
        "gpu_launches": int(launches),
        "work": {"events_per_example": ev_ex, "draws_per_example": draws_ex,
                 "type_i_per_example": d["type_i"] / max(d["examples"], 1),
                 "type_ii_per_example": d["type_ii"] / max(d["examples"], 1),
                 "state_updates_per_example": d["state_updates"] / max(d["examples"], 1)},
        # the binding resource is the integer pipe: every reference draw is
        # one SplitMix64 (two 64-bit multiplies) + compare, at the measured
        # per-SM draw rate; the HBM traffic of the states is secondary
        "roofline": {"kernel": "k_train<1, false> (grid mode, HBM-resident states, "
                               "grid-balanced byte-SIMD feedback)",
                     "bound": "int (SplitMix64 draws at the measured per-SM rate)",
                     "achieved": draws_ex * step_n / (per_launch_ms / 1e3) / 1e9,
                     "peak": lp["draw_peak_per_s"] / 1e9, "unit": "G draws/s",
                     "frac": int_s_ex * step_n / (per_launch_ms / 1e3),
                     "traffic": c4_ncu_sample(), "peak_source": lp["source"],
                     "draws_per_example": draws_ex,
                     "int_us_per_example": int_s_ex * 1e6,
                     "achieved_us_per_example": per_launch_ms * 1e3 / step_n,
                     "avg_launch_ms": per_launch_ms},
        "pipes_ncu": ncu_pipes("k_train<"),
        "roofline_hbm": {"achieved": achieved, "peak": HBM_PEAK, "unit": "GB/s",
                         "frac": achieved / HBM_PEAK, "peak_source": HBM_PEAK_SRC,
                         "algorithmic_bytes_per_example": bytes_ex,
                         "traffic_ncu_sample": c4_ncu_sample()},
        "clocks": clocks,
        "e2e": {"value": n_ex * world / (e2e_ms / 1e3), "unit": "examples/s",
                "h2d_bytes_per_step": int(tx.nbytes + 4 * step_n),
                "d2h_bytes_per_step": int(sess.states.numel() + 4 * sess.weights.numel()),
                "path": "pinned host features -> H2D -> tmb_pack_literals -> tmb_trainer_run "
                        "-> D2H model"},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # N=1 only (contract)
        from oracle import oracle
        x_lit = oracle.augment_literals(tx)
        rate, n_done, dt = oracle_train_rate(cfg, st0, w0, c0, fb0, x_lit, ty,
                                             timed_slices[0].cpu().numpy().astype(np.int64),
                                             args.cpu_seconds)
        model_name, ncpu = host_desc()
        line["cpu_baseline"] = {"value": rate, "unit": "examples/s", "cores": 1, "kind": "port",
                                "sample": f"oracle C port of executor.train, {n_done} examples of "
                                          f"the first timed step from the same model state "
                                          f"({dt:.1f}s, 1 thread)",
                                "host": model_name, "host_cores": ncpu}
    return line


def bench_c4_sweep(args, rank, world, local):
    """configs[3] sweep: the 8-point grid s in {1.5, 2, 3, 5} x T in {5000,
    10000} (datasets.SWEEP_GRID) of independent bag-of-words trainings, job j
    on rank j mod world (parallel.jobs_of; tuning.py:176-227 runs them one
    after another).  Step = every job trains its next --sweep-examples
    examples of epoch 1 (sessions persist across steps).  value = examples
    of all jobs / max-over-ranks time: total work is fixed, so scaling is
    strong.  The jobs' test accuracies (the sweep's result) are reported."""
    import torch

    import paper_2405_04212_b200 as tmb
    from paper_2405_04212_b200 import _lib, datasets, parallel
    (tx, ty), (ex, ey) = datasets.bag_of_words(data_seed=4)
    grid = datasets.SWEEP_GRID
    mine = parallel.jobs_of(len(grid), world, rank)
    step_n = args.sweep_examples
    jobs = []
    for j in mine:
        s_, t_ = grid[j]
        cfg = tmb.Config(**datasets.bag_of_words_config_kwargs(seed=j, s=s_, threshold=t_))
        sess = tmb.DenseTrainSession(cfg, tx, ty)
        order = torch.from_numpy(sess.next_order().astype(np.int32)).cuda()
        jobs.append([j, cfg, sess, order, 0])
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step(job):
        j, cfg, sess, order, pos = job
        if pos + step_n > sess.N:  # next epoch
            job[3] = order = torch.from_numpy(sess.next_order().astype(np.int32)).cuda()
            pos = 0
        sess.run_steps(order[pos:pos + step_n])
        job[4] = pos + step_n

    for _ in range(args.warmup):
        for job in jobs:
            step(job)
    torch.cuda.synchronize()
    stats0 = [job[2].stats_dict() for job in jobs]
    launches0 = _lib.launch_count()
    barrier(world)
    with ClockSampler(local) as clk:
        barrier(world)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            flush_l2(flush)
            for job in jobs:
                step(job)
        b.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    launches = _lib.launch_count() - launches0
    ms = max_over_ranks(a.elapsed_time(b), world)
    n_total = len(grid) * step_n * args.steps
    value = n_total / (ms / 1e3)
    ev = sum(job[2].stats_dict()["events"] - s0["events"] for job, s0 in zip(jobs, stats0))
    sweep_draws = sum(job[2].stats_dict()["draws"] - s0["draws"] for job, s0 in zip(jobs, stats0))
    n_mine = len(jobs) * step_n * args.steps
    # the sweep's result: test accuracy of every grid point (gathered)
    acc_mine = {job[0]: tmb.evaluate(job[2].model(), (ex, ey)) for job in jobs}
    if world > 1:
        import torch.distributed as dist
        parts = [None] * world
        dist.all_gather_object(parts, acc_mine)
        acc = {}
        for p in parts:
            acc.update(p)
    else:
        acc = acc_mine
    # e2e: per step and job, pinned host features -> H2D -> pack -> trainer ->
    # D2H model (a sweep driver that keeps no device state between steps)
    from paper_2405_04212_b200.runtime import ptr, stream_ptr
    xp = torch.from_numpy(np.ascontiguousarray(tx)).pin_memory()
    st_host = torch.empty(jobs[0][2].states.shape, dtype=torch.int8).pin_memory() if jobs else None
    w_host = torch.empty(jobs[0][2].weights.shape, dtype=torch.int32).pin_memory() if jobs else None
    barrier(world)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        for job in jobs:
            sess = job[2]
            xd = xp.to("cuda", non_blocking=True)
            _lib.call("tmb_pack_literals", ptr(xd), xp.shape[0], job[1].n_literals, 1,
                      ptr(sess.lit_words), stream_ptr())
            step(job)
            st_host.copy_(sess.states, non_blocking=True)
            w_host.copy_(sess.weights, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1), world)
    line = {
        "metric": "sweep train examples/sec (configs[3] 8-point s x T grid)",
        "value": value, "unit": "examples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "int8 TA states (HBM) / int32 weights / u64 SplitMix64",
        "data": "synthetic (datasets.bag_of_words: Zipf(1.1) documents, planted sets)",
        "config": {"workload": sweep_workload(world, step_n),
                   "grid": [list(g) for g in grid], "jobs_on_rank0": mine,
                   "parallelism": f"jobs round-robin over {world} GPU(s); no collective on "
                                  "the hot path",
                   "l2": "256 MiB buffer written before every timed step"},
        "gpu_launches": int(launches),
        "work": {"events_per_example_rank0": ev / max(n_mine, 1)},
        "sweep_result": {"test_accuracy": {f"s={grid[j][0]},T={grid[j][1]}": acc[j]
                                           for j in sorted(acc)},
                         "note": f"after {args.warmup + args.steps} steps of {step_n} "
                                 "examples per job"},
        "roofline": {"kernel": "k_train<1, false> (grid mode, HBM-resident states, "
                               "grid-balanced byte-SIMD feedback)",
                     "bound": "int (SplitMix64 draws at the measured per-SM rate)",
                     "achieved": sweep_draws / (ms / 1e3) / 1e9,
                     "peak": live_peaks()["draw_peak_per_s"] / 1e9, "unit": "G draws/s",
                     "frac": sweep_draws / (ms / 1e3) / live_peaks()["draw_peak_per_s"],
                     "draws_per_example_rank0": sweep_draws / max(n_mine, 1),
                     "peak_source": live_peaks()["source"],
                     "note": "the c4-train kernel; draws of rank 0's jobs over its timed region"},
        "clocks": clk.summary(),
        "e2e": {"value": n_total / (e2e_ms / 1e3), "unit": "examples/s",
                "h2d_bytes_per_step": int(len(jobs) * tx.nbytes),
                "d2h_bytes_per_step": int(len(jobs) * (jobs[0][2].states.numel()
                                                       + 4 * jobs[0][2].weights.numel()))
                if jobs else 0,
                "path": "per job and step: pinned host features -> H2D -> tmb_pack_literals "
                        "-> tmb_trainer_run -> D2H model"},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # N=1 only (contract)
        from oracle import oracle
        model_name, ncpu = host_desc()
        x_lit = oracle.augment_literals(tx)
        per, t = 6, time.perf_counter()
        for j, (s_, t_) in enumerate(grid):
            cfg = oracle.OracleCfg(**datasets.bag_of_words_config_kwargs(seed=j, s=s_,
                                                                          threshold=t_))
            st = oracle.new_train_state(cfg)
            order, _ = oracle.shuffle_permutation(len(ty), oracle.derive_stream(j, 0xD157), 0)
            oracle.train_steps(cfg, st, x_lit, ty, order[:per])
        dt = time.perf_counter() - t
        line["cpu_baseline"] = {"value": len(grid) * per / dt, "unit": "examples/s",
                                "cores": 1, "kind": "port",
                                "sample": f"oracle C port of executor.train, the first {per} "
                                          f"examples of each of the 8 grid points, run one "
                                          f"after another as tuning does ({dt:.1f}s, 1 thread)",
                                "host": model_name, "host_cores": ncpu}
    return line


def bench_c5_sparse(args, rank, world, local):
    """configs[4]: SparseTM on 10^6 Zipf documents (10^6-literal vocabulary,
    2000 clauses, capacity 64).  Headline = training documents/s, step =
    100000 consecutive documents of the epoch (the next epoch's shuffle when
    one runs out); every rank trains the same replica (same data and seed:
    training is sequential, "replicas only").  Secondary = inference over
    all 10^6 documents per step, the CSR rows SHARDED over the ranks by
    non-zeros (parallel.csr_shard), predictions gathered once."""
    import torch

    import paper_2405_04212_b200 as tmb
    from paper_2405_04212_b200 import _lib, datasets, parallel, sparse_train
    from paper_2405_04212_b200.executor import shuffle_permutation
    d = datasets.sparse_zipf(data_seed=5)
    cfg = tmb.Config(**datasets.sparse_config_kwargs(seed=0))
    sess = sparse_train.SparseTrainSession(cfg, d.indptr, d.indices, d.labels)
    step_n = 100_000
    cur = {"order": shuffle_permutation(sess.N, sess.shuffle_rng).astype(np.int32), "pos": 0}

    def next_slice():
        if cur["pos"] + step_n > sess.N:  # the next epoch's order
            cur["order"] = shuffle_permutation(sess.N, sess.shuffle_rng).astype(np.int32)
            cur["pos"] = 0
        o = cur["order"][cur["pos"]:cur["pos"] + step_n]
        cur["pos"] += step_n
        return o

    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        sess.run_steps(torch.from_numpy(next_slice()).cuda())
    torch.cuda.synchronize()
    timed = [next_slice() for _ in range(args.steps)]
    timed_dev = [torch.from_numpy(o).cuda() for o in timed]
    # model at the start of the timed region (CPU baseline starts from it)
    lits0, sts0, w0, bc0 = sess.engine.get_lists()
    fb0 = sess.fb_counter
    stats0 = sess.stats_dict()
    launches0 = _lib.launch_count()
    barrier(world)
    with ClockSampler(local) as clk:
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for od in timed_dev:
            sess.run_steps(od)
        b.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    t_ms = max_over_ranks(a.elapsed_time(b), world)
    st1 = sess.stats_dict()
    dd = {k: st1[k] - stats0[k] for k in st1}
    n_docs = args.steps * step_n
    value = n_docs * world / (t_ms / 1e3)
    nnz = 100
    csr_bytes = 4 * nnz + 8
    ev_doc = dd["events"] / max(dd["examples"], 1)
    # ---- sharded inference over all documents with the trained model
    eng = sess.engine
    lo, hi = parallel.csr_shard(d.indptr, world, rank)
    n_loc = hi - lo
    ip_loc = sess.indptr[lo:hi + 1] - sess.indptr[lo]
    ix_loc = sess.indices[int(d.indptr[lo]):int(d.indptr[hi])]
    for _ in range(2):
        eng.votes_and_pred(ip_loc, ix_loc, n_loc)
    torch.cuda.synchronize()
    barrier(world)
    ia = torch.cuda.Event(enable_timing=True)
    ib = torch.cuda.Event(enable_timing=True)
    ia.record(stream)
    for _ in range(args.steps):
        votes, pred = eng.votes_and_pred(ip_loc, ix_loc, n_loc)
    ib.record(stream)
    torch.cuda.synchronize()
    inf_ms = max_over_ranks(ia.elapsed_time(ib), world)
    inf_value = sess.N * args.steps / (inf_ms / 1e3)
    per_launch_inf_ms = ia.elapsed_time(ib) / args.steps
    tg = time.perf_counter()
    pred_all = parallel.gather_rows(pred.cpu().numpy(), sess.N)
    gather_s = time.perf_counter() - tg
    acc = float((pred_all == d.labels).mean())
    # e2e training: the timed chunks again from the same model, each chunk's
    # CSR rows staged (in consumption order) in pinned host memory by the
    # data loader before the timed region; timed per step: H2D of the chunk,
    # the trainer, D2H of the step's statistics
    eng.set_lists(lits0, sts0, w0, bc0)
    sess.fb_counter = fb0
    staged = []
    for o in timed:
        o = o.astype(np.int64)
        lens = d.indptr[o + 1] - d.indptr[o]
        ip = np.zeros(step_n + 1, dtype=np.int64)
        ip[1:] = np.cumsum(lens)
        gather = np.repeat(d.indptr[o] - ip[:-1], lens) + np.arange(ip[-1])
        staged.append((torch.from_numpy(ip).pin_memory(),
                       torch.from_numpy(d.indices[gather]).pin_memory(),
                       torch.from_numpy(d.labels[o].astype(np.int32)).pin_memory()))
    seq = torch.arange(step_n, dtype=torch.int32, device="cuda")
    st_h = torch.empty(6, dtype=torch.int64).pin_memory()
    h2d_tr = sum(int(x.numel() * x.element_size()) for x in staged[0])
    torch.cuda.synchronize()
    barrier(world)
    ta = torch.cuda.Event(enable_timing=True)
    tb = torch.cuda.Event(enable_timing=True)
    ta.record(stream)
    for ip_h, ix_h, lb_h in staged:
        sess.run_steps_on(ip_h.to("cuda", non_blocking=True), ix_h.to("cuda", non_blocking=True),
                          lb_h.to("cuda", non_blocking=True), seq)
        st_h.copy_(sess.stats, non_blocking=True)
    tb.record(stream)
    torch.cuda.synchronize()
    e2e_train = step_n * args.steps * world / (max_over_ranks(ta.elapsed_time(tb), world) / 1e3)
    lits1, sts1, w1, bc1 = eng.get_lists()
    e2e_same = bool(np.array_equal(bc1, sess.engine.get_lists()[3]))
    # e2e inference: this rank's host CSR shard -> device -> infer -> host
    a0, a1 = int(d.indptr[lo]), int(d.indptr[hi])
    ip_h = torch.from_numpy(np.ascontiguousarray(d.indptr[lo:hi + 1] - a0)).pin_memory()
    ix_h = torch.from_numpy(np.ascontiguousarray(d.indices[a0:a1])).pin_memory()
    pr_h = torch.empty(n_loc, dtype=torch.int64).pin_memory()
    barrier(world)
    ea = torch.cuda.Event(enable_timing=True)
    eb = torch.cuda.Event(enable_timing=True)
    ea.record(stream)
    for _ in range(args.steps):
        ipd = ip_h.to("cuda", non_blocking=True)
        ixd = ix_h.to("cuda", non_blocking=True)
        _, pd = eng.votes_and_pred(ipd, ixd, n_loc)
        pr_h.copy_(pd, non_blocking=True)
    eb.record(stream)
    torch.cuda.synchronize()
    e2e_inf = sess.N * args.steps / (max_over_ranks(ea.elapsed_time(eb), world) / 1e3)
    launches = _lib.launch_count() - launches0
    tr_tr, tr_tr_src = ncu_traffic("k_sparse_train")
    tr_in, tr_in_src = ncu_traffic("k_sparse_infer")
    line = {
        "metric": "SparseTM train documents/sec (configs[4])",
        "value": value, "unit": "documents/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "int32 literal ids / int8 states / u64 SplitMix64",
        "data": "synthetic (datasets.sparse_zipf: 10^6 Zipf(1.05) documents x 100 ids)",
        "config": {"workload": WORKLOADS["c5-sparse"],
                   "parallelism": f"replicas x{world} (online training is sequential; every "
                                  "rank trains the same replica)",
                   "l2": "per-step CSR chunk (40 MB) and the clause lists; each step streams "
                         "new documents"},
        "gpu_launches": int(launches),
        "work": {"events_per_document": ev_doc,
                 "draws_per_document": dd["draws"] / max(dd["examples"], 1)},
        "roofline": {"kernel": "k_sparse_train", "bound": "latency",
                     "achieved": value / world, "unit": "documents/s",
                     "peak": 1e9 / live_peaks()["l2_hop_ns"],
                     "frac": (value / world) * live_peaks()["l2_hop_ns"] / 1e9,
                     "floor": "one cross-SM L2 hop per document (every document is non-empty: "
                              "~1 100 applied events each, so no window of documents can be "
                              "decided together), measured live by tmb_microbench_pingpong",
                     "traffic": tr_tr, "traffic_source": tr_tr_src,
                     "hbm_gbs": csr_bytes * value / world / 1e9,
                     "hbm_frac": csr_bytes * value / world / 1e9 / HBM_PEAK,
                     "algorithmic_bytes_per_example": csr_bytes,
                     "note": "sequential training: one grid all-reduce per document plus the "
                             "per-event list merges; HBM carries only the document's CSR row"},
        "clocks": clk.summary(),
        "e2e": {"value": e2e_train, "unit": "documents/s",
                "h2d_bytes_per_step": h2d_tr, "d2h_bytes_per_step": 48,
                "same_model_as_device_run": e2e_same,
                "path": "per step: pinned host CSR chunk (100000 documents in consumption "
                        "order) + labels -> H2D -> tmb_sparse_train -> D2H step statistics"},
        "secondary": {"metric": "SparseTM inference documents/sec (configs[4], sharded)",
                      "value": inf_value, "unit": "documents/s", "n_gpus": world,
                      "scaling": "strong",
                      "sharding": f"CSR rows balanced by nnz over {world} rank(s) "
                                  "(parallel.csr_shard); predictions gathered once "
                                  f"({gather_s * 1e3:.1f} ms, outside the timed step)",
                      "rows_rank0": [lo, hi],
                      "e2e": {"value": e2e_inf, "unit": "documents/s",
                              "h2d_bytes_per_step": int(ip_h.numel() * 8 + ix_h.numel() * 4),
                              "d2h_bytes_per_step": int(8 * n_loc),
                              "path": "this rank's pinned host CSR shard -> H2D -> "
                                      "tmb_sparse_infer -> host predictions"},
                      "ms_per_step": inf_ms / args.steps, "accuracy_after_train": acc,
                      "roofline": {"kernel": "k_sparse_infer (inverted index)",
                                   "bound": "hbm (nominal; the binding cost is the postings' "
                                            "gathers from the L2-resident index and the "
                                            "per-warp shared counters, DESIGN.md 5.4)",
                                   "achieved": n_loc * (csr_bytes + 8) / (per_launch_inf_ms / 1e3)
                                   / 1e9,
                                   "peak": HBM_PEAK, "unit": "GB/s",
                                   "frac": n_loc * (csr_bytes + 8) / (per_launch_inf_ms / 1e3)
                                   / 1e9 / HBM_PEAK,
                                   "traffic": tr_in, "traffic_source": tr_in_src,
                                   "algorithmic_bytes_per_example": csr_bytes + 8}},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # N=1 only (contract)
        from oracle import oracle
        model_name, ncpu = host_desc()
        # the oracle from the SAME model state on the same documents, with the
        # real candidate set (the whole training set's actives)
        ob = oracle.SparseOracleBank(cfg, candidates=sess.candidates)
        ob.lits, ob.sts, ob.weights = lits0, sts0, w0.copy()
        docs = [d.row(int(i)) for i in timed[0]]
        labels = d.labels[timed[0]].astype(np.int64)
        n_tr, t0 = 0, time.perf_counter()
        bctr = [int(bc0[0])]
        fb = fb0
        while time.perf_counter() - t0 < args.cpu_seconds and n_tr < len(docs):
            _, bctr, fb = oracle.sparse_train_from(cfg, [ob], bctr, fb, docs[n_tr:n_tr + 1],
                                                   labels[n_tr:n_tr + 1])
            n_tr += 1
        dt = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": n_tr / dt, "unit": "documents/s", "cores": 1,
                                "kind": "port",
                                "sample": f"oracle C port of executor.train (sparse), the first "
                                          f"{n_tr} documents of the first timed step from the "
                                          f"same model state, real candidate set "
                                          f"({len(sess.candidates)} literals) ({dt:.1f}s, "
                                          f"1 thread)",
                                "host": model_name, "host_cores": ncpu}
    return line

# -------------------------------------------------------- reference arm --

def ref_package():
    """The UNMODIFIED reference (tsetlinkit) from baseline/_ref (pip-installed
    from /root/reference), with its default numba backend.
    Returns the module or None when it is not installed / numba is absent."""
    ref = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "tsetlinkit")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "numba_cache"))
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import tsetlinkit
        from tsetlinkit import kernels
    except Exception:  # noqa: BLE001 - fall back to the port
        return None
    if kernels.BACKEND_NAME != "numba":
        return None
    kernels.warmup()
    return tsetlinkit


class RefTrainer:
    """executor.train's serial driver (executor.py:296-330: eval_block /
    decide / update_block, one clause block) driving the reference's own
    DenseClauseBank, update_probabilities, sample_updates and numba kernels,
    started from a saved training state so it can time any epoch."""

    def __init__(self, tk, cfg_kwargs, x, state=None):
        from tsetlinkit.core import (FEEDBACK_STREAM, SHUFFLE_STREAM, Config, RngStream,
                                     augment_literals)
        from tsetlinkit.dense import DenseClauseBank
        self.tk = tk
        self.cfg = Config(**cfg_kwargs)
        self.bank = DenseClauseBank(self.cfg)
        self.blk_rng = RngStream.derive(self.cfg.seed, 0)
        self.fb_rng = RngStream.derive(self.cfg.seed, FEEDBACK_STREAM)
        self.sh_rng = RngStream.derive(self.cfg.seed, SHUFFLE_STREAM)
        if state is not None:
            self.bank.states[:] = state["states"]
            self.bank.weights[:] = state["weights"]
            self.blk_rng.counter = int(state["block_counters"][0])
            self.fb_rng.counter = int(state["fb_counter"])
            self.sh_rng.counter = int(state["shuffle_counter"])
        self.x_lit = augment_literals(x, self.cfg.negated_literals_enabled)
        self.votes_parts = np.zeros((1, self.cfg.n_classes), dtype=np.int64)

    def next_order(self):
        from tsetlinkit.executor import shuffle_permutation
        return shuffle_permutation(self.x_lit.shape[0], self.sh_rng)

    def steps(self, labels, order):
        from tsetlinkit.dense import EvalMode
        from tsetlinkit.feedback import sample_updates, update_probabilities
        bank, cfg, vp = self.bank, self.cfg, self.votes_parts
        for idx in order:
            lits = self.x_lit[idx]
            label = int(labels[idx])
            out = bank.clause_outputs(lits, EvalMode.TRAINING)
            vp[0] = bank.votes(out)
            dec = update_probabilities(vp.sum(axis=0), label, cfg.threshold, self.fb_rng)
            ut, un = sample_updates(dec, cfg.n_clauses, self.fb_rng)
            bank.apply_feedback(lits, out, label, dec.negative_class, ut, un, self.blk_rng)




def _c2_checkpoint(warmup: int):
    """Latest committed oracle checkpoint of the configs[1] bench model at or
    before the GPU arm's last warm-up epoch (tests/golden/c2_epoch{3,5}.npz)."""
    best = None
    for e in (3, 5):
        f = os.path.join(REPO, "tests", "golden", f"c2_epoch{e}.npz")
        if e <= warmup and os.path.exists(f):
            best = (e, f)
    if best is None:
        return 0, None
    g = np.load(best[1])
    return best[0], {k: g[k] for k in g.files}


def bench_reference(args, rank, world):
    """The reference's own CPU implementation on the host cores, rank 0 only.

    When baseline/_ref holds the unmodified reference (pip-installed from
    /root/reference) and numba imports, its own code runs ("kind":
    "reference"): the executor's serial-driver loop over its DenseClauseBank
    / feedback functions / numba kernels (training), its public train()
    (configs[0]), its numba clause_outputs_batch sharded over host threads
    (inference).  Otherwise, and for SparseTM (pure-Python reference, ~minutes
    per configs[4] document), the oracle's C restatement ("kind": "port")."""
    if rank != 0:
        return None
    from oracle import oracle

    from paper_2405_04212_b200 import datasets
    model_name, ncpu = host_desc()
    tk = None if args.ref_port else ref_package()
    kind = "reference" if tk is not None else "port"
    unit = "examples/s"
    extra = {}
    secs = []  # wall seconds of every timed step (a bounded sample of the workload's step)
    if args.workload == "c1-train":
        (tx, ty), (ex, ey) = datasets.noisy_xor()
        rates, accs = [], []
        for i in range(args.warmup + args.steps):
            kw = datasets.noisy_xor_config_kwargs(seed=i % 5)
            t = time.perf_counter()
            if tk is not None:
                run = tk.train(tk.Config(**kw), (tx, ty), n_epochs=20)
                st, w = run.model.states, run.model.weights
            else:
                ost, _ = oracle.train(oracle.OracleCfg(**kw), tx, ty, 20)
                st, w = ost.states, ost.weights
            dt = time.perf_counter() - t
            if i >= args.warmup:
                secs.append(dt)
                rates.append(20 * len(ty) / dt)
                _, pred = oracle.batch_votes(st, w, oracle.augment_literals(ex))
                accs.append(float(np.mean(pred == ey)))
        value = float(np.mean(rates))
        metric = "train examples/sec (configs[0] Noisy-XOR CoTM training)"
        sample = ("one 20-epoch train() of 5000 examples per step (model seeds 0..4 in turn), "
                  "1 thread" + (" (tsetlinkit.train, numba backend)" if tk else ""))
        cores = 1
        extra["test_accuracy_per_step"] = accs
    elif args.workload == "c3-infer":
        m = datasets.inference_model(model_seed=11)
        xs = datasets.inference_examples(3, 0, args.c3_cpu_examples)
        x_lit = oracle.augment_literals(xs)
        if tk is not None:
            from concurrent.futures import ThreadPoolExecutor

            from tsetlinkit.core import Config as RCfg
            from tsetlinkit.dense import DenseClauseBank as RBank
            bank = RBank(RCfg(n_literals=4096, n_clauses=10000, n_classes=10, s=2.0,
                              threshold=100))
            bank.states[:] = m.states
            bank.weights[:] = m.weights
            parts = np.array_split(np.arange(len(xs)), ncpu)
            pool = ThreadPoolExecutor(ncpu)

            def run_all():
                # batch_votes (dense.py:171-174; numba nogil kernel) per
                # thread shard, then argmax (executor.py:382)
                res = list(pool.map(lambda p: bank.batch_votes(x_lit[p]), parts))
                return np.argmax(np.concatenate(res), axis=1)
        else:
            def run_all():
                return oracle.batch_votes(m.states, m.weights, x_lit, nthreads=ncpu,
                                          want_votes=False)[1]
        rates = []
        for i in range(args.warmup + args.steps):
            t = time.perf_counter()
            run_all()
            if i >= args.warmup:
                secs.append(time.perf_counter() - t)
                rates.append(len(xs) / secs[-1])
        value = float(np.mean(rates))
        metric = "inference examples/sec (configs[2] batched CoTM inference)"
        sample = (f"{len(xs)}-example prefix per step, {ncpu} threads"
                  + (" (DenseClauseBank.batch_votes, numba nogil kernel per thread shard)"
                     if tk else ""))
        cores = ncpu
    elif args.workload in ("c4-train", "c4-sweep"):
        (tx, ty), _ = datasets.bag_of_words(data_seed=4)
        grid = datasets.SWEEP_GRID if args.workload == "c4-sweep" else [(2.0, 10000)]
        per_step = 8 if args.workload == "c4-train" else 2
        trainers = []
        for j, (s_, t_) in enumerate(grid):
            kw = datasets.bag_of_words_config_kwargs(seed=j if len(grid) > 1 else 0, s=s_,
                                                     threshold=t_)
            if tk is not None:
                tr = RefTrainer(tk, kw, tx)
                trainers.append((tr, tr.next_order(), None))
            else:
                cfg = oracle.OracleCfg(**kw)
                st = oracle.new_train_state(cfg)
                order, _ = oracle.shuffle_permutation(len(ty), oracle.derive_stream(cfg.seed,
                                                                                    0xD157), 0)
                trainers.append((cfg, order, st))
        x_lit = None if tk is not None else oracle.augment_literals(tx)
        rates, pos = [], 0
        for i in range(args.warmup + args.steps):
            t = time.perf_counter()
            for a, order, st in trainers:
                if tk is not None:
                    a.steps(ty, order[pos:pos + per_step])
                else:
                    oracle.train_steps(a, st, x_lit, ty, order[pos:pos + per_step])
            pos += per_step
            if i >= args.warmup:
                secs.append(time.perf_counter() - t)
                rates.append(per_step * len(trainers) / secs[-1])
        value = float(np.mean(rates))
        if args.workload == "c4-sweep":
            metric = "sweep train examples/sec (configs[3] 8-point s x T grid)"
            sample = (f"{per_step} consecutive examples of epoch 1 of each of the 8 grid points "
                      f"per step, run one after another as tuning does, 1 thread")
        else:
            metric = "train examples/sec (configs[3] bag-of-words CoTM training)"
            sample = f"{per_step} consecutive examples of epoch 1 per step, 1 thread"
        cores = 1
    elif args.workload == "c5-sparse":
        kind = "port"
        d = datasets.sparse_zipf(data_seed=5)
        cfg = oracle.OracleCfg(**datasets.sparse_config_kwargs(seed=0))
        cands = np.unique(d.indices).astype(np.int64)
        order, _ = oracle.shuffle_permutation(len(d), oracle.derive_stream(0, 0xD157), 0)
        banks = [oracle.SparseOracleBank(cfg, candidates=cands)]
        bctr, fb = [0], 0
        rates, pos, per_step = [], 0, 1
        for i in range(args.warmup + args.steps):
            docs = [d.row(int(k)) for k in order[pos:pos + per_step]]
            t = time.perf_counter()
            banks, bctr, fb = oracle.sparse_train_from(cfg, banks, bctr, fb, docs,
                                                       d.labels[order[pos:pos + per_step]])
            pos += per_step
            if i >= args.warmup:
                secs.append(time.perf_counter() - t)
                rates.append(per_step / secs[-1])
        value = float(np.mean(rates))
        metric = "SparseTM train documents/sec (configs[4])"
        sample = (f"{per_step} document(s) of epoch 1 per step with the full training set's "
                  f"candidate set ({cands.size} literals), 1 thread; the reference's "
                  "SparseClauseBank is pure Python, so its C restatement runs")
        cores = 1
        unit = "documents/s"
    else:
        (tx, ty), _ = c2_data(0)
        kw = datasets.mnist_shaped_config_kwargs(seed=0)
        # the GPU arm times epochs W+1..: start from the committed oracle
        # checkpoint of epoch W (bit-identical to the GPU arm's model there,
        # tests/test_gpu_parity.py) so the reference times the same epoch
        ep, ck = _c2_checkpoint(args.warmup)
        if tk is not None:
            tr = RefTrainer(tk, kw, tx, ck)
            order = tr.next_order()
        else:
            cfg = oracle.OracleCfg(**kw)
            if ck is not None:
                st = oracle.OracleTrainState(ck["states"].copy(), ck["weights"].copy(),
                                             ck["block_counters"].copy(), int(ck["fb_counter"]),
                                             int(ck["shuffle_counter"]))
            else:
                st = oracle.new_train_state(cfg)
            x_lit = oracle.augment_literals(tx)
            order, _ = oracle.shuffle_permutation(len(ty), oracle.derive_stream(0, 0xD157),
                                                  st.shuffle_counter)
        rates, pos = [], 0
        per_step = args.ref_examples
        for i in range(args.warmup + args.steps):
            if pos + per_step > len(ty):
                break
            t = time.perf_counter()
            if tk is not None:
                tr.steps(ty, order[pos:pos + per_step])
            else:
                oracle.train_steps(cfg, st, x_lit, ty, order[pos:pos + per_step])
            pos += per_step
            if i >= args.warmup:
                secs.append(time.perf_counter() - t)
                rates.append(per_step / secs[-1])
        value = float(np.mean(rates))
        metric = "train examples/sec (configs[1] MNIST-shaped CoTM training)"
        sample = (f"{per_step} consecutive examples of epoch {ep + 1} per step (warm-up steps "
                  f"advance the model; the GPU arm's first timed epoch is {args.warmup + 1}), "
                  f"from the committed epoch-{ep} checkpoint, 1 thread: training is "
                  f"sequential (n_blocks=1)"
                  + (" (tsetlinkit serial-driver loop, numba backend)" if tk else ""))
        cores = 1
    cpu = {"value": value, "unit": unit, "cores": cores, "kind": kind, "sample": sample,
           "host": model_name}
    if tk is not None and kind == "reference":
        from tsetlinkit import kernels as rk
        cpu["reference"] = {"package": "tsetlinkit (baseline/_ref, unmodified)",
                            "backend": rk.BACKEND_NAME}
    cpu.update(extra)
    return {"metric": metric, "value": value, "unit": unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * float(np.mean(secs)) if secs else None,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int8 / u64", "data": "synthetic", "impl": "reference",
            "config": {"workload": (sweep_workload(world, args.sweep_examples)
                                    if args.workload == "c4-sweep" else WORKLOADS[args.workload]),
                       "sample_per_step": sample},
            "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


# ------------------------------------------------------------------ main --

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c2-train",
                    choices=["c1-train", "c2-train", "c3-infer", "c4-train", "c4-sweep",
                             "c5-sparse"])
    ap.add_argument("--c3-examples", type=int, default=1 << 22)
    ap.add_argument("--c3-e2e-examples", type=int, default=1 << 20)
    ap.add_argument("--c3-cpu-examples", type=int, default=1 << 13)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-examples", type=int, default=1500)
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--sweep-examples", type=int, default=2500)
    ap.add_argument("--train-cta", type=int, default=0, help="0 = auto")
    ap.add_argument("--train-threads", type=int, default=0, help="0 = auto")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--set-option", action="append", default=[], metavar="NAME=INT",
                    help="tmb_set_option before the workload (A/B runs)")
    ap.add_argument("--ref-port", action="store_true",
                    help="reference arm: time the oracle port even when baseline/_ref exists")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        line = bench_reference(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return

    rank, world, local = dist_init()
    import paper_2405_04212_b200 as tmb
    tmb.runtime.require_device()
    for opt in args.set_option:
        name, val = opt.split("=")
        tmb._lib.call("tmb_set_option", name.encode(), int(val))
    if args.workload == "c3-infer":
        line = bench_c3_infer(args, rank, world, local)
        line.update({"higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                     "warmup": args.warmup, "dtype": "u8 features / int32 votes",
                     "data": "synthetic (counter-based Bernoulli(0.5) generator)"})
        line["scaling"] = "strong"
    elif args.workload == "c1-train":
        line = bench_c1_train(args, rank, world, local)
    elif args.workload == "c4-train":
        line = bench_c4_train(args, rank, world, local)
    elif args.workload == "c4-sweep":
        line = bench_c4_sweep(args, rank, world, local)
    elif args.workload == "c5-sparse":
        line = bench_c5_sparse(args, rank, world, local)
    else:
        line = bench_c2_train(args, rank, world, local)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
