"""Executor: the training loop and evaluation (mirror of executor.py:36-383).

The reference runs four steps per example on host threads (input block ->
clause blocks evaluate -> feedback block decides -> clause blocks update,
executor.py:275-340).  Here one persistent cooperative CUDA kernel per epoch
runs all four steps for every example (csrc/tmb_train.cu); the host only
prepares data, draws the epoch permutation with the reference's Fisher-Yates
(executor.py:50-58, in C on the host), launches, and evaluates.  The trained
model is bit-identical to the reference's for the same Config, data and
n_epochs, for any n_jobs (n_blocks is model-semantic and honoured exactly).
"""

from __future__ import annotations

import ctypes as ct
import os
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import (FEEDBACK_STREAM, SHUFFLE_STREAM, Config, DataError, RngStream,
                   augment_literals, derive_stream)
from .dense import DenseClauseBank
from .runtime import np_ptr, ptr, require_device, stream_ptr
from .sparse import SparseClauseBank, SparseDataset


def partition_clauses(n_clauses: int, n_blocks: int) -> list[range]:
    """executor.py:36-47: contiguous ranges, sizes differing by at most one."""
    if not 1 <= n_blocks <= n_clauses:
        raise ValueError("n_blocks must be in [1, n_clauses]")
    base, extra = divmod(n_clauses, n_blocks)
    out, start = [], 0
    for b in range(n_blocks):
        size = base + (1 if b < extra else 0)
        out.append(range(start, start + size))
        start += size
    return out


def shuffle_permutation(n: int, rng: RngStream) -> np.ndarray:
    """executor.py:50-58: seeded Fisher-Yates (host C, libtmb200)."""
    perm = np.empty(max(n, 1), dtype=np.int64)
    new = ct.c_uint64()
    _lib.call("tmb_shuffle_permutation", n, rng.stream_seed & (2**64 - 1),
              rng.counter & (2**64 - 1), np_ptr(perm), ct.byref(new))
    rng.counter = int(new.value) if n > 1 else rng.counter
    return perm[:n]


@dataclass
class EpochMetric:
    epoch: int
    accuracy: float | None
    seconds: float


@dataclass
class TrainRun:
    config: Config
    epoch_metrics: list[EpochMetric]
    model: DenseClauseBank | SparseClauseBank


class _InputBlock:
    """executor.py:84-121: validation identical to the reference."""

    def __init__(self, cfg: Config, data, name: str):
        self.sparse = isinstance(data, SparseDataset)
        if self.sparse:
            if data.n_literals != cfg.n_literals:
                raise DataError(f"{name}: dataset universe {data.n_literals} does not "
                                f"match config n_literals {cfg.n_literals}")
            for ex in data.examples:
                ex.check_range(cfg.n_literals)
            self.data = data
            self.labels = data.labels
        else:
            x, y = data
            x = np.ascontiguousarray(x, dtype=np.uint8)
            if x.ndim != 2 or x.shape[1] != cfg.n_literals:
                raise DataError(f"{name}: feature width {x.shape[-1] if x.ndim else 0} "
                                f"does not match config n_literals {cfg.n_literals}")
            self.x = x
            self.labels = np.asarray(y, dtype=np.int64)
            if self.x.shape[0] != self.labels.shape[0]:
                raise DataError(f"{name}: example/label count mismatch")
        if len(self.labels) == 0:
            raise DataError(f"{name}: dataset is empty")
        if self.labels.min() < 0 or self.labels.max() >= cfg.n_classes:
            raise DataError(f"{name}: label outside [0, {cfg.n_classes})")

    def __len__(self) -> int:
        return len(self.labels)


def _resolve_jobs(n_jobs: int, n_blocks: int) -> int:
    """executor.py:267-272 (validation only: blocks run in parallel on the device)."""
    if n_jobs == -1:
        n_jobs = os.cpu_count() or 1
    if n_jobs < 1:
        raise ValueError("n_jobs must be positive or -1")
    return min(n_jobs, n_blocks)


# tmb_trainer_kernel kinds
TRAINER_KERNELS = ("k_train_warp", "k_train (cluster)", "k_train (grid)", "k_train_fast",
                   "k_train_spec", "k_train_tiny")


class DenseTrainSession:
    """Device-resident dense training state: the model (states, weights,
    per-block counters), the packed dataset and the fused-kernel trainer.

    ``run_epoch`` is one epoch of executor.train: shuffle (host), one
    cooperative kernel launch over all N examples."""

    def __init__(self, cfg: Config, x: np.ndarray, y: np.ndarray, n_cta: int = 0,
                 threads: int = 0, states: np.ndarray | None = None,
                 weights: np.ndarray | None = None, states_in_hbm: bool = False,
                 flag_keys: bool = True, balanced_feedback: bool = True,
                 warp_kernel: bool = True):
        import torch
        require_device()
        self.cfg = cfg
        self.N = int(x.shape[0])
        F, P, C, K = cfg.n_literals, cfg.n_literal_positions, cfg.n_clauses, cfg.n_classes
        self.W = (P + 31) // 32
        dev = torch.device("cuda", torch.cuda.current_device())
        init = np.full((C, P), cfg.init_state, np.int8) if states is None else states
        self.states = torch.from_numpy(np.ascontiguousarray(init, np.int8)).to(dev)
        w0 = np.zeros((C, K), np.int32) if weights is None else weights
        self.weights = torch.from_numpy(np.ascontiguousarray(w0, np.int32)).to(dev)
        self.block_counters = torch.zeros(cfg.n_blocks, dtype=torch.int64, device=dev)
        self.fb_counter = 0
        self.shuffle_rng = RngStream.derive(cfg.seed, SHUFFLE_STREAM)
        self.stats = torch.zeros(6, dtype=torch.int64, device=dev)
        self.set_data(x, y)
        tc = _lib.TrainCfg(F, P, C, K, cfg.n_blocks, cfg.threshold, cfg.effective_budget,
                           float(cfg.s), int(cfg.boost_true_positive), cfg.state_min,
                           cfg.state_max,
                           int(bool(states_in_hbm)) | (0 if flag_keys else 2) |
                           (0 if balanced_feedback else 4) | (0 if warp_kernel else 8),
                           cfg.seed & (2**64 - 1))
        self._h = ct.c_void_p()
        _lib.call("tmb_trainer_create", ct.byref(tc), ptr(self.states), ptr(self.weights),
                  ptr(self.block_counters), n_cta, threads, ct.byref(self._h))
        a, b, c, d = ct.c_int(), ct.c_int(), ct.c_int(), ct.c_int()
        _lib.call("tmb_trainer_info", self._h, ct.byref(a), ct.byref(b), ct.byref(c),
                  ct.byref(d))
        kind, win = ct.c_int(), ct.c_int()
        _lib.call("tmb_trainer_kernel", self._h, ct.byref(kind), ct.byref(win))
        self.launch = dict(n_cta=a.value, threads=b.value, smem_bytes=c.value,
                           states_in_smem=bool(d.value),
                           kernel=TRAINER_KERNELS[kind.value], spec_window=win.value)

    def set_data(self, x: np.ndarray, y: np.ndarray):
        """Upload raw features once and pack them to literal bit rows on the
        device (tmb_pack_literals: [N, ceil(P/32)] uint32)."""
        import torch
        x = np.ascontiguousarray(x, dtype=np.uint8)
        if x.size and int(x.max()) > 1:
            # the device packs literal bits; the inference and explain paths
            # reject non-0/1 bytes the same way
            raise DataError("train data: features must be 0/1")
        dev = self.states.device
        xd = torch.from_numpy(x).pin_memory().to(dev, non_blocking=True)
        self.lit_words = torch.empty((x.shape[0], self.W), dtype=torch.int32, device=dev)
        _lib.call("tmb_pack_literals", ptr(xd), x.shape[0], self.cfg.n_literals,
                  int(self.cfg.negated_literals_enabled), ptr(self.lit_words), stream_ptr())
        self.labels = torch.from_numpy(np.asarray(y, dtype=np.int32)).to(dev)
        self.N = int(x.shape[0])
        del xd

    def snapshot(self):
        """Device copy of the full training state (model + RNG counters)."""
        return (self.states.clone(), self.weights.clone(), self.block_counters.clone(),
                self.fb_counter, self.shuffle_rng.counter)

    def restore(self, snap):
        st, w, bc, fb, sh = snap
        self.states.copy_(st)
        self.weights.copy_(w)
        self.block_counters.copy_(bc)
        self.fb_counter = fb
        self.shuffle_rng.counter = sh

    def next_order(self) -> np.ndarray:
        return shuffle_permutation(self.N, self.shuffle_rng)

    def run_steps(self, order_dev, n_steps: int | None = None):
        """Launch the fused kernel over order_dev (device int32)."""
        n = int(order_dev.shape[0]) if n_steps is None else n_steps
        _lib.call("tmb_trainer_run", self._h, ptr(self.lit_words), ptr(self.labels),
                  ptr(order_dev), n, self.fb_counter & (2**64 - 1), ptr(self.stats),
                  stream_ptr())
        self.fb_counter += n * (1 + 2 * self.cfg.n_clauses)

    def run_epoch(self):
        import torch
        order = self.next_order().astype(np.int32)
        od = torch.from_numpy(order).to(self.states.device, non_blocking=False)
        self.run_steps(od)
        return od

    def compiled(self):
        from .inference import CompiledModel
        return CompiledModel.from_device_bank(self.states, self.weights, self.cfg.n_literals,
                                              self.cfg.negated_literals_enabled)

    def model(self) -> DenseClauseBank:
        import torch
        torch.cuda.current_stream().synchronize()
        bank = DenseClauseBank(self.cfg)
        bank.states[:] = self.states.cpu().numpy()
        bank.weights[:] = self.weights.cpu().numpy()
        return bank

    def stats_dict(self):
        v = self.stats.cpu().numpy()
        return dict(zip(["examples", "events", "type_i", "type_ii", "draws", "state_updates"],
                        [int(a) for a in v]))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.load().tmb_trainer_destroy(h)
            except Exception:
                pass
            self._h = None


def train(cfg: Config, train_data, eval_data=None, n_epochs: int = 1, n_jobs: int = 1,
          epoch_callback=None, observer=None) -> TrainRun:
    """executor.py:275-340 with the per-example loop on the GPU.

    ``observer(event, step, block)`` (a testing hook in the reference) is
    replayed after each epoch in the order the fused kernel guarantees:
    every block's "votes", then "decision", then every block's "update".
    """
    inp = _InputBlock(cfg, train_data, "train data")
    evl = _InputBlock(cfg, eval_data, "eval data") if eval_data is not None else None
    _resolve_jobs(n_jobs, cfg.n_blocks)
    if inp.sparse:
        from .sparse_train import train_sparse
        return train_sparse(cfg, inp, evl, n_epochs, epoch_callback, observer,
                            TrainRun, EpochMetric)
    metrics: list[EpochMetric] = []
    if n_epochs <= 0:
        return TrainRun(cfg, metrics, DenseClauseBank(cfg))
    sess = DenseTrainSession(cfg, inp.x, inp.labels)
    import torch
    for epoch in range(n_epochs):
        t0 = time.perf_counter()
        sess.run_epoch()
        if observer:
            torch.cuda.current_stream().synchronize()
            for step in range(len(inp)):
                for b in range(cfg.n_blocks):
                    observer("votes", (epoch, step), b)
                observer("decision", (epoch, step), None)
                for b in range(cfg.n_blocks):
                    observer("update", (epoch, step), b)
        accuracy = None
        if evl is not None:
            accuracy = _device_accuracy(sess.compiled(), evl.x, evl.labels)
        torch.cuda.current_stream().synchronize()
        metrics.append(EpochMetric(epoch, accuracy, time.perf_counter() - t0))
        if epoch_callback:
            epoch_callback(metrics[-1])
    return TrainRun(cfg, metrics, sess.model())


def _device_accuracy(model, x: np.ndarray, labels: np.ndarray) -> float:
    _, pred = model.votes_and_pred(x, want_votes=False)
    return float(np.mean(pred == labels))


def dataset_votes(bank, data) -> np.ndarray:
    """executor.py:355-372: inference-mode votes on a whole dataset."""
    if isinstance(data, SparseDataset):
        if bank.kind != "sparse":
            raise DataError("sparse data requires a sparse model")
        for ex in data.examples:
            ex.check_range(bank.n_literals)
        return bank.batch_votes(data.examples)
    x, _ = data
    x = np.ascontiguousarray(x, dtype=np.uint8)
    if bank.kind == "sparse":
        raise DataError("sparse model requires sparse data")
    if x.shape[1] != bank.cfg.n_literals:
        raise DataError(f"feature width {x.shape[1]} does not match model "
                        f"n_literals {bank.cfg.n_literals}")
    from .inference import CompiledModel
    votes, _ = CompiledModel.from_bank(bank).votes_and_pred(x, want_pred=False)
    return votes


def evaluate(bank, data) -> float:
    """executor.py:375-383: accuracy of argmax votes (ties -> lowest class)."""
    if isinstance(data, SparseDataset):
        labels = data.labels
        votes = dataset_votes(bank, data)
        return float(np.mean(np.argmax(votes, axis=1) == labels))
    x, y = data
    labels = np.asarray(y, dtype=np.int64)
    x = np.ascontiguousarray(x, dtype=np.uint8)
    if bank.kind == "sparse":
        raise DataError("sparse model requires sparse data")
    if x.shape[1] != bank.cfg.n_literals:
        raise DataError(f"feature width {x.shape[1]} does not match model "
                        f"n_literals {bank.cfg.n_literals}")
    from .inference import CompiledModel
    _, pred = CompiledModel.from_bank(bank).votes_and_pred(x, want_votes=False)
    return float(np.mean(pred == labels))
