import sys, torch
sys.path.insert(0, ".")
import bench, paper_2405_04212_b200 as tmb
from paper_2405_04212_b200 import _lib, datasets
N = 1 << 22
m = datasets.inference_model(model_seed=11)
bank = tmb.DenseClauseBank(tmb.Config(n_literals=4096, n_clauses=10000, n_classes=10, s=2.0, threshold=100))
bank.states[:] = m.states; bank.weights[:] = m.weights
model = tmb.CompiledModel.from_bank(bank)
x = bench.c3_inputs_device(N, 0)
pred = torch.empty(N, dtype=torch.int64, device="cuda")
for mode, name in ((0, "full"), (3, "skip both"), (3 | 64, "skip both, no copies"), (64, "full, no copies (wrong)"), (1 | 64, "skip eval, no copies"), (2 | 64, "skip transpose, no copies")):
    _lib.call("tmb_set_option", b"infer.debug_skip", mode)
    for _ in range(2): model.infer_device(x, pred_dev=pred)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3): model.infer_device(x, pred_dev=pred)
    b.record(); torch.cuda.synchronize()
    print(f"{name:28s} {a.elapsed_time(b) / 3:7.3f} ms", flush=True)
_lib.call("tmb_set_option", b"infer.debug_skip", 0)
