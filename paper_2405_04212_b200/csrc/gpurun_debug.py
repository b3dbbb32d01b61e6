import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2405_04212_b200 as gpu
from paper_2405_04212_b200 import _lib
from paper_2405_04212_b200.runtime import ptr
from oracle import oracle
rs = np.random.default_rng(20 * 100 + 1)
x = rs.integers(0, 2, size=(250, 27)).astype(np.uint8)
y = ((x[:, 0] + x[:, 3] * 2 + x[:, 9]) % 4).astype(np.int64)
cfg = gpu.Config(n_literals=27, n_clauses=45, n_classes=4, s=2.5, threshold=9, seed=20, n_blocks=1, n_literal_budget=6)
for n_cta in (16, 20):
    sess = gpu.DenseTrainSession(cfg, x, y, n_cta=n_cta)
    tr = torch.zeros(4, dtype=torch.int64, device='cuda')
    _lib.call("tmb_trainer_set_trace", sess._h, ptr(tr))
    order = sess.next_order()
    od = torch.from_numpy(order.astype(np.int32)).cuda()
    ost = oracle.new_train_state(cfg)
    xl = oracle.augment_literals(x)
    for step in range(30):
        # oracle votes before the step
        outs = oracle.clause_outputs(ost.states, xl[order[step]], True, cfg.effective_budget)
        votes = outs.astype(np.int64) @ ost.weights.astype(np.int64)
        sess.run_steps(od[step:step+1])
        oracle.train_steps(cfg, ost, xl, y, order[step:step+1])
        t = tr.cpu().numpy()
        lab = y[order[step]]
        print(n_cta, step, "gpu neg/vl/vn/ev", t.tolist(), "oracle vl/vn", votes[lab], votes[t[0]])
        m = sess.model()
        if not (np.array_equal(m.states, ost.states) and np.array_equal(m.weights, ost.weights)):
            print("DIVERGED at", step); break
