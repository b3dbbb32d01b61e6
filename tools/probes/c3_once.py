"""One C3 inference launch (for ncu)."""
import sys
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2405_04212_b200 as tmb  # noqa: E402
from paper_2405_04212_b200 import _lib, datasets  # noqa: E402

tmb.runtime.require_device()
_lib.call("tmb_set_option", b"infer.warp_specialized", 0 if "--legacy" in sys.argv else 1)
for a in sys.argv[1:]:
    if a.startswith("--dbg="):
        _lib.call("tmb_set_option", b"infer.debug_skip", int(a[6:]))
    if a.startswith("--mode="):
        _lib.call("tmb_set_option", b"infer.eval_mode", int(a[7:]))
N = 1 << 20
m = datasets.inference_model(model_seed=11)
bank = tmb.DenseClauseBank(tmb.Config(n_literals=4096, n_clauses=10000, n_classes=10, s=2.0,
                                      threshold=100))
bank.states[:] = m.states
bank.weights[:] = m.weights
model = tmb.CompiledModel.from_bank(bank)
x = bench.c3_inputs_device(N, 0)
pred = torch.empty(N, dtype=torch.int64, device="cuda")
model.infer_device(x, pred_dev=pred)
torch.cuda.synchronize()
print("ok")
