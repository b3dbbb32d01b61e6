"""Debug: grid-balanced HBM feedback vs per-CTA feedback within one launch."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2405_04212_b200 as gpu  # noqa: E402
rs = np.random.default_rng(2003)
x = rs.integers(0, 2, size=(250, 27)).astype(np.uint8)
y = ((x[:, 0] + x[:, 3] * 2 + x[:, 9]) % 4).astype(np.int64)
P = int(sys.argv[1]) if len(sys.argv) > 1 else 27
x = rs.integers(0, 2, size=(250, P)).astype(np.uint8)
cfg = gpu.Config(n_literals=P, n_clauses=45, n_classes=4, s=2.5, threshold=9, seed=20,
                 n_blocks=3, n_literal_budget=6)


def run(k, bal):
    s = gpu.DenseTrainSession(cfg, x, y, n_cta=20, states_in_hbm=True, balanced_feedback=bal)
    order = torch.from_numpy(s.next_order().astype(np.int32)).cuda()
    s.run_steps(order[:k])
    m = s.model()
    return m.states, m.weights, s.stats_dict()


for k in (64,):
    a, b = run(k, True), run(k, False)
    same = np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    print(k, "same" if same else f"DIFF states {np.sum(a[0] != b[0])} rows {np.unique(np.argwhere(a[0] != b[0])[:, 0])[:8]} weights {np.sum(a[1] != b[1])}", a[2], b[2])
    if not same:
        break

# determinism of the balanced path
a1, a2 = run(250, True), run(250, True)
print("balanced run-to-run identical:", np.array_equal(a1[0], a2[0]) and np.array_equal(a1[1], a2[1]))
