"""A/B timing of the configs[2] inference kernels (2^22 examples x 4096
features, 10^4 rules x 20 includes): per-CTA solo kernel vs the 4-CTA
warp-specialised cluster kernel, uint8 and bit-packed input; checks that all
predict the same classes."""
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
xb = datasets.inference_examples_device(3, 0, N, 4096, packed=True)
ref = None
dbgs = [int(a) for a in sys.argv[1:]] or [0]
for solo, dbg in [(1, d) for d in dbgs] + ([(0, 0)] if dbgs == [0] else []):
    _lib.call("tmb_set_option", b"infer.solo", solo)
    _lib.call("tmb_set_option", b"infer.debug_skip", dbg)
    for packed in (False, True):
        pred = torch.empty(N, dtype=torch.int64, device="cuda")
        run = (lambda: model.infer_device_packed(xb, pred_dev=pred)) if packed else \
              (lambda: model.infer_device(x, pred_dev=pred))
        for _ in range(2):
            run()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            run()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 5
        gbs = N * 4104 / (ms / 1e3) / 1e9 if not packed else N * 520 / (ms / 1e3) / 1e9
        if ref is None:
            ref = pred.clone()
        print(f"solo={solo} dbg={dbg} packed={packed}: {ms:8.3f} ms  {N / ms / 1e3:8.1f} M ex/s  "
              f"{gbs:7.1f} GB/s  same={bool(torch.equal(ref, pred))}", flush=True)
_lib.call("tmb_set_option", b"infer.solo", 1)
_lib.call("tmb_set_option", b"infer.debug_skip", 0)
