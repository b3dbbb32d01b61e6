"""A/B timing of the k_infer_ws evaluator modes on the configs[2] workload
(2^22 examples x 4096 features, 10^4 rules x 20 includes); checks that every
mode predicts the same classes as the first one."""
import sys
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2405_04212_b200 as tmb  # noqa: E402
from paper_2405_04212_b200 import _lib, datasets  # noqa: E402

tmb.runtime.require_device()
N = 1 << 22
m = datasets.inference_model(model_seed=11)
bank = tmb.DenseClauseBank(tmb.Config(n_literals=4096, n_clauses=10000, n_classes=10, s=2.0,
                                      threshold=100))
bank.states[:] = m.states
bank.weights[:] = m.weights
model = tmb.CompiledModel.from_bank(bank)
x = bench.c3_inputs_device(N, 0)
ref = None
for mode in [int(a) for a in sys.argv[1:]] or [2, 0]:
    _lib.call("tmb_set_option", b"infer.eval_mode", mode)
    pred = torch.empty(N, dtype=torch.int64, device="cuda")
    for skip, name in ((0, "full"), (1, "skip eval"), (2, "skip transpose")):
        _lib.call("tmb_set_option", b"infer.debug_skip", skip)
        for _ in range(2):
            model.infer_device(x, pred_dev=pred)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            model.infer_device(x, pred_dev=pred)
        b.record()
        torch.cuda.synchronize()
        print(f"mode {mode} {name:15s} {a.elapsed_time(b) / 3:8.3f} ms", flush=True)
        if skip == 0:
            if ref is None:
                ref = pred.clone()
            print(f"   same predictions as first mode: {bool(torch.equal(ref, pred))}")
_lib.call("tmb_set_option", b"infer.debug_skip", 0)
_lib.call("tmb_set_option", b"infer.eval_mode", 2)
