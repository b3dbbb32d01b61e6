"""Time the C3 inference kernel with eval / transpose phases disabled (timing
experiment: which phase bounds the kernel)."""
import sys
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2405_04212_b200 as tmb  # noqa: E402
from paper_2405_04212_b200 import _lib, datasets  # noqa: E402

tmb.runtime.require_device()
_lib.call("tmb_set_option", b"infer.warp_specialized", 0 if "--legacy" in sys.argv else 1)
for a in sys.argv[1:]:
    if a.startswith("--mode="):
        _lib.call("tmb_set_option", b"infer.eval_mode", int(a[7:]))
N = 1 << 22
m = datasets.inference_model(model_seed=11)
bank = tmb.DenseClauseBank(tmb.Config(n_literals=4096, n_clauses=10000, n_classes=10, s=2.0,
                                      threshold=100))
bank.states[:] = m.states
bank.weights[:] = m.weights
model = tmb.CompiledModel.from_bank(bank)
x = bench.c3_inputs_device(N, 0)
pred = torch.empty(N, dtype=torch.int64, device="cuda")
for mode, name in ((0, "full"), (1, "skip eval"), (2, "skip transpose"), (3, "skip both"), (4, "no prefetch"), (7, "skip all")):
    _lib.call("tmb_set_option", b"infer.debug_skip", mode)
    for _ in range(2):
        model.infer_device(x, pred_dev=pred)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        model.infer_device(x, pred_dev=pred)
    b.record()
    torch.cuda.synchronize()
    print(f"{name:15s} {a.elapsed_time(b) / 3:8.2f} ms")
_lib.call("tmb_set_option", b"infer.debug_skip", 0)

# per-phase clock64 profile of thread 0 of every CTA (us per tile)
ph = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
_lib.call("tmb_set_option", b"infer.phase_buffer", ph.data_ptr())
model.infer_device(x, pred_dev=pred)
torch.cuda.synchronize()
_lib.call("tmb_set_option", b"infer.phase_buffer", 0)
clk = torch.cuda.get_device_properties(0).clock_rate * 1e3
p = ph.cpu().numpy().reshape(148, 8).astype(float) / clk * 1e6
tiles = (N // 128) / 33
ws = "--legacy" not in sys.argv
names = (["T: wait empty", "T: load+transpose", "T: publish", "T: loop", "E: wait full",
          "E: eval+sync", "E: arrive empty", "E: vempty+push+vfull"] if ws else
         ["prefetch", "zero+sync+eval", "sync", "transpose", "publish", "cluster.sync",
          "await", "finalize+loop"])
for q in range(8):
    print(f"  {names[q]:16s} {p[:, q].mean() / tiles:7.3f} us/tile (max CTA {p[:, q].max() / tiles:7.3f})")
