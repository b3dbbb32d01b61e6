"""One configs[3] training launch of 1000 steps (for ncu)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2405_04212_b200 as tmb  # noqa: E402
from paper_2405_04212_b200 import datasets  # noqa: E402
(tx, ty), _ = datasets.bag_of_words(n_train=6000, n_test=10)
cfg = tmb.Config(**datasets.bag_of_words_config_kwargs(seed=0))
sess = tmb.DenseTrainSession(cfg, tx, ty)
order = torch.from_numpy(sess.next_order().astype(np.int32)).cuda()
sess.run_steps(order[:1000])
sess.run_steps(order[1000:1300])
torch.cuda.synchronize()
print("ok", sess.launch)
