import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2405_04212_b200 as gpu
from oracle import oracle
rs = np.random.default_rng(20 * 100 + 1)
x = rs.integers(0, 2, size=(250, 27)).astype(np.uint8)
y = ((x[:, 0] + x[:, 3] * 2 + x[:, 9]) % 4).astype(np.int64)
cfg = gpu.Config(n_literals=27, n_clauses=45, n_classes=4, s=2.5, threshold=9, seed=20, n_blocks=1, n_literal_budget=6)
for n_cta in (16, 20):
    sess = gpu.DenseTrainSession(cfg, x, y, n_cta=n_cta)
    order = sess.next_order()
    od = torch.from_numpy(order.astype(np.int32)).cuda()
    ost = oracle.new_train_state(cfg)
    xl = oracle.augment_literals(x)
    for step in range(250):
        sess.run_steps(od[step:step+1])
        oracle.train_steps(cfg, ost, xl, y, order[step:step+1])
        m = sess.model()
        if not (np.array_equal(m.states, ost.states) and np.array_equal(m.weights, ost.weights)):
            bad = np.argwhere(m.states != ost.states)
            print(n_cta, "first divergence at step", step, "clauses", np.unique(bad[:,0]) if len(bad) else None,
                  "w diff", np.argwhere(m.weights != ost.weights)[:5].tolist())
            break
    else:
        print(n_cta, "ok 250 single steps")
