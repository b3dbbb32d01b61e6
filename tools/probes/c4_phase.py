"""Per-phase clock64 profile of the generic grid trainer (configs[3],
HBM-resident states, balanced feedback) over 1000 steps after 1000 warm-up
steps; optional tmb_set_option NAME=VALUE arguments."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2405_04212_b200 as tmb  # noqa: E402
from paper_2405_04212_b200 import _lib, datasets  # noqa: E402
from paper_2405_04212_b200.runtime import ptr  # noqa: E402

for a in sys.argv[1:]:
    n, v = a.split("=")
    _lib.load()
    _lib.call("tmb_set_option", n.encode(), int(v))
NAMES = ["eval(+votes)", "arrive", "precompute", "wait+decide", "flag bitmaps",
         "scan+events", "feedback", "wait for all CTAs' feedback"]
(tx, ty), _ = datasets.bag_of_words(n_train=6000, n_test=10)
cfg = tmb.Config(**datasets.bag_of_words_config_kwargs(seed=0))
sess = tmb.DenseTrainSession(cfg, tx, ty)
order = torch.from_numpy(sess.next_order().astype(np.int32)).cuda()
sess.run_steps(order[:1000])
nc = sess.launch["n_cta"]
ph = torch.zeros(nc * (8 + 3072 + 9), dtype=torch.int64, device="cuda")
_lib.call("tmb_trainer_set_profile", sess._h, ptr(ph))
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
sess.run_steps(order[1000:2000])
b.record()
torch.cuda.synchronize()
clk = torch.cuda.get_device_properties(0).clock_rate * 1e3
p = ph.cpu().numpy()[:nc * 8].reshape(nc, 8).astype(np.float64) / clk * 1e6 / 1000
print(f"launch {sess.launch}: {a.elapsed_time(b):.1f} us per example (profiled)")
for q in range(8):
    print(f"   {NAMES[q]:16s} mean {p[:, q].mean():8.2f}  max {p[:, q].max():8.2f} us/ex")
