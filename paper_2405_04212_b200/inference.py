"""Compiled-rule batched inference on the GPU (dense.py:171-174,
executor.py:355-383, predictor.py:45-96).

A ``CompiledModel`` is a device-resident include-list rule set: exactly the
rules ``compile_ruleset`` keeps (clauses with >= 1 include and a non-zero
weight row -- the dropped ones can never change a vote).  Evaluation is the
bit-sliced kernel of csrc/tmb_infer.cu; votes are identical to the
reference's int64 class sums and predictions follow np.argmax (ties to the
lowest class).
"""

from __future__ import annotations

import ctypes as ct

import numpy as np

from . import _lib
from .runtime import np_ptr, ptr, require_device, stream_ptr


def _bank_csr(states: np.ndarray, weights: np.ndarray):
    inc = states >= 0
    keep = inc.any(axis=1) & (weights != 0).any(axis=1)
    rows, cols = np.nonzero(inc[keep])
    counts = np.bincount(rows, minlength=int(keep.sum())).astype(np.int64)
    ptr_ = np.zeros(counts.size + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr_[1:])
    return ptr_, cols.astype(np.int64), np.ascontiguousarray(weights[keep], dtype=np.int32)


class CompiledModel:
    """Device rule set.  ``n_features`` is the width of the raw input rows the
    kernel reads; with ``negations`` the rules address [x, not x] positions."""

    def __init__(self, handle, n_features: int, n_classes: int, negations: bool):
        self._h = handle
        self.n_features = n_features
        self.n_classes = n_classes
        self.negations = negations

    # -- construction ---------------------------------------------------
    @classmethod
    def from_csr(cls, inc_ptr, inc_idx, weights, n_features: int, n_classes: int,
                 negations: bool):
        require_device()
        inc_ptr = np.ascontiguousarray(inc_ptr, dtype=np.int64)
        inc_idx = np.ascontiguousarray(inc_idx if len(inc_idx) else np.zeros(1), dtype=np.int64)
        weights = np.ascontiguousarray(weights, dtype=np.int32).reshape(-1, n_classes)
        if weights.size == 0:
            weights = np.zeros((1, n_classes), dtype=np.int32)
        h = ct.c_void_p()
        _lib.call("tmb_rules_from_csr", np_ptr(inc_ptr), np_ptr(inc_idx), inc_ptr.size - 1,
                  np_ptr(weights), n_classes, n_features, int(bool(negations)), ct.byref(h))
        return cls(h, n_features, n_classes, negations)

    @classmethod
    def from_bank(cls, bank, literal_input: bool = False):
        """From a (host) DenseClauseBank.  literal_input=True evaluates
        augmented literal rows [N, P] (DenseClauseBank.batch_votes); otherwise
        raw feature rows [N, F] (dataset_votes / evaluate)."""
        p, idx, w = _bank_csr(bank.states, bank.weights)
        if literal_input:
            return cls.from_csr(p, idx, w, bank.n_positions, bank.n_classes, False)
        return cls.from_csr(p, idx, w, bank.cfg.n_literals, bank.n_classes,
                            bank.cfg.negated_literals_enabled)

    @classmethod
    def from_device_bank(cls, states, weights, n_features: int, negations: bool):
        """From device tensors (the trainer's live model)."""
        require_device()
        C, P = states.shape
        K = weights.shape[1]
        h = ct.c_void_p()
        _lib.call("tmb_rules_from_bank", ptr(states), ptr(weights), C, P, K, n_features,
                  int(bool(negations)), ct.byref(h), stream_ptr())
        return cls(h, n_features, K, negations)

    @classmethod
    def from_ruleset(cls, rs):
        return cls.from_csr(*rs.csr(), rs.n_literals, rs.n_classes, rs.negated_literals_enabled)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.load().tmb_rules_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def n_rules(self) -> int:
        r = ct.c_int64()
        _lib.call("tmb_rules_info", self._h, ct.byref(r), None)
        return int(r.value)

    # -- evaluation -----------------------------------------------------
    def votes_and_pred(self, x: np.ndarray, want_votes: bool = True, want_pred: bool = True,
                       chunk: int = 0):
        """Host arrays in, host arrays out (tmbh_infer: a 3-deep pipeline of
        ~48 MB chunks -- H2D copy / kernel / D2H of the predictions overlap;
        chunk = examples per chunk, 0 = auto).  The device and pinned
        buffers stay with the rule set between calls (one call at a time)."""
        x = np.ascontiguousarray(x, dtype=np.uint8)
        if x.ndim != 2 or x.shape[1] != self.n_features:
            raise ValueError(f"expected [N, {self.n_features}] input, got {x.shape}")
        N = x.shape[0]
        votes = np.empty((N, self.n_classes), dtype=np.int64) if want_votes else None
        pred = np.empty(N, dtype=np.int64) if want_pred else None
        _lib.call("tmbh_infer", self._h, np_ptr(x), N,
                  np_ptr(votes) if want_votes else None,
                  np_ptr(pred) if want_pred else None, chunk)
        return votes, pred

    def infer_device(self, x_dev, votes_dev=None, pred_dev=None, labels_dev=None,
                     correct_dev=None):
        """Device tensors in/out on the current stream (asynchronous)."""
        N = x_dev.shape[0]
        _lib.call("tmb_infer", self._h, ptr(x_dev), N, ptr(votes_dev), ptr(pred_dev),
                  ptr(labels_dev), ptr(correct_dev), stream_ptr())

    # -- bit-packed input (bit-packed ingestion) ---------------
    def infer_device_packed(self, xb_dev, votes_dev=None, pred_dev=None, labels_dev=None,
                            correct_dev=None):
        """Device uint64 [N, W64] bit-packed features (feature f = bit f % 64
        of word f // 64, e.g. datasets.inference_examples(..., packed=True))
        on the current stream; same outputs as infer_device."""
        N, W64 = xb_dev.shape
        _lib.call("tmb_infer_packed", self._h, ptr(xb_dev), N, W64, ptr(votes_dev),
                  ptr(pred_dev), ptr(labels_dev), ptr(correct_dev), stream_ptr())

    def votes_and_pred_packed(self, xb: np.ndarray, want_votes: bool = True):
        """Host bit-packed rows in, host votes / predictions out."""
        import torch
        xb = np.ascontiguousarray(xb, dtype=np.uint64)
        if xb.ndim != 2 or xb.shape[1] * 64 < self.n_features:
            raise ValueError(f"expected [N, >= {(self.n_features + 63) // 64}] uint64 rows")
        N = xb.shape[0]
        xd = torch.from_numpy(xb.view(np.int64)).cuda()
        votes = torch.empty((N, self.n_classes), dtype=torch.int64, device="cuda") \
            if want_votes else None
        pred = torch.empty(N, dtype=torch.int64, device="cuda")
        self.infer_device_packed(xd, votes, pred)
        return (votes.cpu().numpy() if want_votes else None), pred.cpu().numpy()
