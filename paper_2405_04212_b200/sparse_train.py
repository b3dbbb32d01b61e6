"""SparseTM on the device (placeholder until csrc/tmb_sparse.cu lands)."""

from __future__ import annotations

from . import _lib


def _unsupported(*_a, **_k):
    raise _lib.TmbError(_lib.TMB_E_UNSUPPORTED, "SparseTM device path is not built yet")


train_sparse = _unsupported
sparse_outputs = _unsupported
sparse_batch_votes = _unsupported
sparse_apply_feedback = _unsupported
