"""One SparseTM training launch of 5000 documents (for ncu)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2405_04212_b200 as tmb  # noqa: E402
from paper_2405_04212_b200 import datasets, sparse_train  # noqa: E402
d = datasets.sparse_zipf(n_docs=60000)
cfg = tmb.Config(**datasets.sparse_config_kwargs(seed=0))
sess = sparse_train.SparseTrainSession(cfg, d.indptr, d.indices, d.labels)
sess.run_epoch(max_steps=20000)
sess.run_epoch(max_steps=5000)
torch.cuda.synchronize()
print("ok")
