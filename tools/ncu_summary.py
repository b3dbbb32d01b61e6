"""Summarise ncu reports / launch lists into profiles/ (run in the container).

    python tools/ncu_summary.py TAG
reads gpurun_out/TAG_prof_*.ncu-rep and TAG_*_launches.csv, writes
profiles/TAG_ncu_full_summary.json and profiles/TAG_launch_shares.json.
"""
import csv
import glob
import io
import json
import os
import subprocess
import sys

TAG = sys.argv[1] if len(sys.argv) > 1 else "r01"
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__cluster_dim_x", "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, v = rows[0], rows[1], rows[2]
    d = {"Kernel Name": v[h.index("Kernel Name")]}
    for k in KEYS:
        if k in h:
            i = h.index(k)
            d[k] = f"{v[i]} {units[i]}".strip()
    return d


summary = {}
for rep in sorted(glob.glob(f"gpurun_out/{TAG}_prof_*.ncu-rep")):
    summary[os.path.basename(rep)[:-8]] = raw(rep)
json.dump(summary, open(f"profiles/{TAG}_ncu_full_summary.json", "w"), indent=1)

shares = {}
for f in sorted(glob.glob(f"gpurun_out/{TAG}_*_launches.csv")):
    lines = [ln for ln in open(f) if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    per = {}
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        t = float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)
        name = r["Kernel Name"].split("(")[0]
        per.setdefault(name, [0, 0.0])
        per[name][0] += 1
        per[name][1] += t
    tot = sum(v[1] for v in per.values())
    shares[os.path.basename(f)] = {k: {"launches": v[0], "us_total": round(v[1], 1),
                                       "share": round(v[1] / tot, 4)}
                                   for k, v in sorted(per.items(), key=lambda x: -x[1][1])}
    os.system(f"cp {f} profiles/")
json.dump(shares, open(f"profiles/{TAG}_launch_shares.json", "w"), indent=1)
for b in glob.glob(f"gpurun_out/{TAG}_bench*.json") + glob.glob(f"gpurun_out/{TAG}_int_peaks.json"):
    os.system(f"cp {b} profiles/")
print(json.dumps(summary, indent=1))
print(json.dumps(shares, indent=1))
