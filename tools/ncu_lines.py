"""Aggregate ncu warp-stall samples per CUDA source line (run in the container).

    python tools/ncu_lines.py REPORT.ncu-rep [N]
Uses `ncu -i REP --page source --csv --print-source cuda,sass` (needs
-lineinfo and --import-source on at capture time)."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = defaultdict(lambda: defaultdict(int))
src = {}
hdr = None
fname = ""
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        idx = {k: i for i, k in enumerate(r) if k not in ("Source",)}
        stalls = [k for k in r if k.startswith("stall_") and "Not Issued" not in k]
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    try:
        s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    key = (fname, r[0])
    src[key] = r[1].strip()
    a = agg[key]
    a["samples"] += s
    a["inst"] += int(r[idx["Instructions Executed"]] or 0)
    a["wf"] += int(r[idx["L1 Wavefronts Shared"]] or 0)
    a["wfi"] += int(r[idx["L1 Wavefronts Shared Ideal"]] or 0)
    for k in stalls:
        a[k] += int(r[idx[k]] or 0)
tot = sum(a["samples"] for a in agg.values()) or 1
print(f"total samples {tot}")
for key, a in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]:
    st = sorted(((v, k[6:]) for k, v in a.items() if k.startswith("stall_")), reverse=True)[:3]
    sts = " ".join(f"{k}:{100 * v / max(a['samples'], 1):.0f}%" for v, k in st if v)
    print(f"{100 * a['samples'] / tot:5.1f}% {key[0]}:{key[1]:>5} inst={a['inst']:>10} wf={a['wf']:>10}/{a['wfi']:<10} "
          f"{src[key][:60]:60s} {sts}")
