"""configs[1] bench model after 3 epochs, trained by the oracle (the C
restatement of tsetlinkit's executor.train, itself pinned to the reference's
fixtures).  It lets `bench.py --impl reference` time the same epoch (4) that
the GPU arm times, and `tests/test_gpu_parity.py` check 3 full configs[1]
epochs (180 000 examples) of the GPU trainer bit for bit.

    python tests/golden/make_c2_epoch3.py      (~4 min, 1 core)
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
from oracle import oracle  # noqa: E402

from paper_2405_04212_b200 import datasets  # noqa: E402

(tx, ty), _ = datasets.mnist_shaped(data_seed=7)
cfg = oracle.OracleCfg(**datasets.mnist_shaped_config_kwargs(seed=0))
t0 = time.time()
st, _ = oracle.train(cfg, tx, ty, 3)
print(f"3 epochs in {time.time() - t0:.0f} s")
np.savez_compressed(os.path.join(HERE, "c2_epoch3.npz"), states=st.states, weights=st.weights,
                    block_counters=st.block_counters, fb_counter=np.uint64(st.fb_counter),
                    shuffle_counter=np.uint64(st.shuffle_counter))
print("wrote", os.path.join(HERE, "c2_epoch3.npz"))
