"""configs[1] trainer variants, us per example over epoch 4 (after 3 warm-up
epochs): fast path (smem states), generic grid kernel with HBM-resident states
with and without grid-balanced feedback."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2405_04212_b200 as tmb  # noqa: E402
from paper_2405_04212_b200 import datasets  # noqa: E402

(tx, ty), _ = datasets.mnist_shaped(n_train=60000, n_test=10)
variants = {
    "fast (smem states)": dict(),
    "generic, HBM states, balanced": dict(states_in_hbm=True, flag_keys=False, balanced_feedback=True),
    "generic, HBM states, unbalanced": dict(states_in_hbm=True, flag_keys=False, balanced_feedback=False),
    "generic, smem states": dict(flag_keys=False),
}
for name, kw in variants.items():
    cfg = tmb.Config(**datasets.mnist_shaped_config_kwargs(seed=0))
    sess = tmb.DenseTrainSession(cfg, tx, ty, **kw)
    for _ in range(3):
        sess.run_epoch()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    sess.run_epoch()
    b.record()
    torch.cuda.synchronize()
    print(f"{name:34s} {a.elapsed_time(b) * 1e3 / len(ty):6.3f} us/example  launch={sess.launch}",
          flush=True)
