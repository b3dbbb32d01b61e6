"""configs[3] (bag-of-words, 10^4 clauses x 2*10^4 literals, states in HBM):
parity against the oracle on a prefix, then training throughput."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2405_04212_b200 as tmb  # noqa: E402
from paper_2405_04212_b200 import datasets  # noqa: E402

t0 = time.time()
(tx, ty), (ex, ey) = datasets.bag_of_words(n_train=6000, n_test=2000)
print("data", time.time() - t0, "s", tx.shape, "pos frac", ty.mean())
cfg = tmb.Config(**datasets.bag_of_words_config_kwargs(seed=0))
sess = tmb.DenseTrainSession(cfg, tx, ty)
print("launch", sess.launch)
order = sess.next_order().astype(np.int32)
od = torch.from_numpy(order).cuda()
# parity prefix
n_par = int(sys.argv[1]) if len(sys.argv) > 1 else 12
sess.run_steps(od[:n_par])
m = sess.model()
from oracle import oracle  # noqa: E402
st = oracle.new_train_state(cfg)
t1 = time.time()
oracle.train_steps(cfg, st, oracle.augment_literals(tx), ty, order[:n_par].astype(np.int64))
print("oracle", n_par, "examples in", round(time.time() - t1, 1), "s")
print("parity states", np.array_equal(m.states, st.states), "weights",
      np.array_equal(m.weights, st.weights))
# throughput on the rest of the epoch
for chunk in (2000, 3988):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0 = sess.stats_dict()
    a.record()
    sess.run_steps(od[n_par:n_par + chunk])
    b.record()
    torch.cuda.synchronize()
    s1 = sess.stats_dict()
    ms = a.elapsed_time(b)
    print(f"{chunk} examples: {ms:.1f} ms -> {chunk / ms * 1e3:.0f} ex/s; per ex:",
          {k: (s1[k] - s0[k]) / chunk for k in ("events", "type_i", "draws", "state_updates")})
    n_par += chunk
acc = tmb.evaluate(sess.model(), (ex, ey))
print("test accuracy after 1 epoch", acc)
