"""configs[1] bench model after 5 epochs (the driver's bench runs with
--warmup 5, so its GPU arm times epochs 6..), trained by the oracle from the
committed 3-epoch state (tests/golden/c2_epoch3.npz, itself made by
make_c2_epoch3.py).  `bench.py --impl reference` starts from the checkpoint
of the GPU arm's last warm-up epoch, so both arms time the same epoch.

    python tests/golden/make_c2_epoch5.py      (~3 min, 1 core)
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
g = np.load(os.path.join(HERE, "c2_epoch3.npz"))
st = oracle.OracleTrainState(g["states"].copy(), g["weights"].copy(), g["block_counters"].copy(),
                             int(g["fb_counter"]), int(g["shuffle_counter"]))
t0 = time.time()
st, _ = oracle.train(cfg, tx, ty, 2, state=st)
print(f"epochs 4-5 in {time.time() - t0:.0f} s")
np.savez_compressed(os.path.join(HERE, "c2_epoch5.npz"), states=st.states, weights=st.weights,
                    block_counters=st.block_counters, fb_counter=np.uint64(st.fb_counter),
                    shuffle_counter=np.uint64(st.shuffle_counter))
print("wrote", os.path.join(HERE, "c2_epoch5.npz"))
