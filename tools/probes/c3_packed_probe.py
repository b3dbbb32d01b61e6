"""Timing probe of the bit-packed C3 path with debug ablations."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2405_04212_b200 as tmb  # noqa: E402
from paper_2405_04212_b200 import _lib, datasets  # noqa: E402
from paper_2405_04212_b200.runtime import ptr, stream_ptr  # noqa: E402
N, F = 1 << 22, 4096
W = F // 64
m = datasets.inference_model(model_seed=11)
bank = tmb.DenseClauseBank(tmb.Config(n_literals=F, n_clauses=10000, n_classes=10, s=2.0, threshold=100))
bank.states[:] = m.states
bank.weights[:] = m.weights
model = tmb.CompiledModel.from_bank(bank)
xb = torch.empty((N, W), dtype=torch.int64, device="cuda")
_lib.call("tmb_stream_u64_block", datasets.inference_stream_seed(3), 0, N * W, ptr(xb), stream_ptr())
pred = torch.empty(N, dtype=torch.int64, device="cuda")
for dbg, name in ((0, "full"), (32, "8 codes max"), (2, "skip transpose"), (1, "skip eval")):
    _lib.call("tmb_set_option", b"infer.debug_skip", dbg)
    for _ in range(2):
        model.infer_device_packed(xb, pred_dev=pred)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        model.infer_device_packed(xb, pred_dev=pred)
    b.record()
    torch.cuda.synchronize()
    print(f"{name:16s} {a.elapsed_time(b) / 3:7.2f} ms")
_lib.call("tmb_set_option", b"infer.debug_skip", 0)
