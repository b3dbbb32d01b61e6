"""configs[2] inference on the generic kernel (one CTA per tile, rules read
from L2) vs the warp-specialised cluster kernel, and how many SMs each uses."""
import sys
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2405_04212_b200 as tmb  # noqa: E402
from paper_2405_04212_b200 import _lib, datasets  # noqa: E402

N = 1 << 20
m = datasets.inference_model(model_seed=11)
bank = tmb.DenseClauseBank(tmb.Config(n_literals=4096, n_clauses=10000, n_classes=10, s=2.0,
                                      threshold=100))
bank.states[:] = m.states
bank.weights[:] = m.weights
model = tmb.CompiledModel.from_bank(bank)
x = bench.c3_inputs_device(N, 0)
pred = torch.empty(N, dtype=torch.int64, device="cuda")
for gen in (0, 1):
    _lib.call("tmb_set_option", b"infer.force_generic", gen)
    model.infer_device(x, pred_dev=pred)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(2):
        model.infer_device(x, pred_dev=pred)
    b.record()
    torch.cuda.synchronize()
    print(f"generic={gen}: {a.elapsed_time(b) / 2:.3f} ms per 2^20 examples")
_lib.call("tmb_set_option", b"infer.force_generic", 0)
