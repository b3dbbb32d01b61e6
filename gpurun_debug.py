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
C = 45
fb_seed = oracle.derive_stream(cfg.seed, 0xFEED)
for trial in range(3):
  for n_cta in (16, 20):
    sess = gpu.DenseTrainSession(cfg, x, y, n_cta=n_cta)
    tr = torch.zeros(4 + 2*64, dtype=torch.int64, device='cuda')
    _lib.call("tmb_trainer_set_trace", sess._h, ptr(tr))
    order = sess.next_order()
    od = torch.from_numpy(order.astype(np.int32)).cuda()
    ost = oracle.new_train_state(cfg)
    xl = oracle.augment_literals(x)
    for step in range(250):
        lits = xl[order[step]]
        outs = oracle.clause_outputs(ost.states, lits, True, cfg.effective_budget)
        votes = outs.astype(np.int64) @ ost.weights.astype(np.int64)
        lab = y[order[step]]
        u = oracle.stream_u01(fb_seed, ost.fb_counter)
        neg, pt, pn = oracle.update_probabilities(votes, lab, cfg.threshold, u)
        ut, un = oracle.sample_updates(pt, pn, C, fb_seed, ost.fb_counter + 1)
        prev_states = ost.states.copy(); prev_w = ost.weights.copy(); prev_ctr = int(ost.block_counters[0])
        sess.run_steps(od[step:step+1])
        oracle.train_steps(cfg, ost, xl, y, order[step:step+1])
        t = tr.cpu().numpy()
        m = sess.model()
        if not (np.array_equal(m.states, ost.states) and np.array_equal(m.weights, ost.weights)):
            print("trial", trial, "n_cta", n_cta, "DIVERGED at", step, "gpu trace", t.tolist(), "oracle vl vn", votes[lab], votes[neg], "events", int(ut.sum()+un.sum()))
            print("  per-CTA vl/vn", t[4:4+2*n_cta].reshape(-1, 2).tolist())
            gctr = int(sess.block_counters.cpu().numpy()[0]); print("  block ctr gpu", gctr, "oracle", int(ost.block_counters[0]), "prev", prev_ctr)
            for j in np.unique(np.argwhere(m.states != ost.states)[:, 0]):
                d = np.flatnonzero(m.states[j] != ost.states[j])
                print("  clause", j, "out", outs[j], "ut", ut[j], "un", un[j], "w", prev_w[j].tolist(), "ndiff", len(d), "pos", d[:8].tolist(),
                      "prev", prev_states[j][d[:8]].tolist(), "gpu", m.states[j][d[:8]].tolist(), "orc", ost.states[j][d[:8]].tolist())
            break
