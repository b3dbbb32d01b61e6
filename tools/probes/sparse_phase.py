"""Per-phase clock64 profile of the SparseTM trainer (configs[4] shapes).

Slots per CTA (tmb_sparse.cu k_sparse_train): 0-5 phases seen by thread 0,
6 / 7 / 8 Type I (output 0) / Type II / Type I (output 1) event cycles summed
over warps, 9 output-1 Type I events, 10 per-step slowest warp's event cycles.
"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2405_04212_b200 as tmb  # noqa: E402
from paper_2405_04212_b200 import _lib, datasets, sparse_train  # noqa: E402
n_docs = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
d = datasets.sparse_zipf(n_docs=n_docs)
cfg = tmb.Config(**datasets.sparse_config_kwargs(seed=0))
sess = sparse_train.SparseTrainSession(cfg, d.indptr, d.indices, d.labels)
sess.run_epoch(max_steps=50000)
torch.cuda.synchronize()
nc = 148
ph = torch.zeros(nc * 16, dtype=torch.int64, device="cuda")
_lib.call("tmb_set_option", b"sparse.phase_buffer", ph.data_ptr())
st0 = sess.stats_dict()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 20000
a.record()
sess.run_epoch(max_steps=n)
b.record()
torch.cuda.synchronize()
_lib.call("tmb_set_option", b"sparse.phase_buffer", 0)
st1 = sess.stats_dict()
dd = {k: st1[k] - st0[k] for k in st1}
clk = torch.cuda.get_device_properties(0).clock_rate * 1e3
raw = ph.cpu().numpy().reshape(nc, 16).astype(float)
p = raw / clk * 1e6 / n
print(f"{a.elapsed_time(b) * 1e3 / n:.2f} us/doc")
for q, name in enumerate(["loop top (act load, neg)", "eval", "votes+exchange", "flag bitmaps",
                          "events (warp 0)", "feedback merges"]):
    print(f"  {name:26s} mean {p[:, q].mean():7.3f}  max {p[:, q].max():7.3f} us/doc")
print("  stats", dd)
tot = raw / clk * 1e6
n1 = raw[:, 9].sum()
n0 = dd["type_i"] - n1
print(f"  Type I out=0  {tot[:, 6].sum() / max(n0, 1):.3f} us/event  ({n0 / n:.1f} per doc)")
print(f"  Type I out=1  {tot[:, 8].sum() / max(n1, 1):.3f} us/event  ({n1 / n:.1f} per doc)")
print(f"  Type II       {tot[:, 7].sum() / max(dd['type_ii'], 1):.3f} us/event  ({dd['type_ii'] / n:.1f} per doc)")
print(f"  slowest warp's events per step: mean over CTAs {p[:, 10].mean():.3f}  max {p[:, 10].max():.3f} us/doc")
nii = max(dd['type_ii'], 1)
print(f"  loop top up to the prefetch issue: mean {p[:, 15].mean():.3f} us/doc")
print(f"  Type II: cand rounds {raw[:, 11].sum() / nii:.2f}  stored n {raw[:, 12].sum() / nii:.1f}  ins {raw[:, 13].sum() / nii:.1f}  cand-loop {raw[:, 14].sum() / clk * 1e6 / nii:.3f} us")
