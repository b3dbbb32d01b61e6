"""k_train_tiny timing ablations (train.debug_skip bits: 1 no feedback, 2 no
flag draws, 4 no barrier; results are wrong, timing only)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2405_04212_b200 as tmb  # noqa: E402
from paper_2405_04212_b200 import _lib, datasets  # noqa: E402
(tx, ty), _ = datasets.noisy_xor()
for dbg in (0, 1, 2, 3, 4, 7):
    _lib.call("tmb_set_option", b"train.debug_skip", dbg)
    cfg = tmb.Config(**datasets.noisy_xor_config_kwargs(seed=0))
    sess = tmb.DenseTrainSession(cfg, tx, ty)
    order = torch.from_numpy(np.tile(np.arange(len(ty), dtype=np.int32), 20)).cuda()
    sess.run_steps(order)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    sess.run_steps(order)
    b.record()
    torch.cuda.synchronize()
    print(dbg, sess.launch["kernel"], round(a.elapsed_time(b) * 1e3 / len(order), 4), "us/example")
_lib.call("tmb_set_option", b"train.debug_skip", 0)
