"""The kernel-backend plugin, B200 edition.

Same module contract as the reference's backends (kernels/__init__.py:47-53:
``NAME, clause_outputs, clause_outputs_batch, bank_feedback, warmup``; the
functions of kernels/_numba.py:53-138), backed by libtmb200.so.  Arrays are
caller-owned numpy buffers exactly as in the reference: ``states`` and
``weights`` are mutated in place by ``bank_feedback``, which returns the new
event counter.  These per-call entry points are latency-bound by design (one
example per call, host<->device copies); ``executor.train`` uses the fused
persistent kernel instead.
"""

from __future__ import annotations

import ctypes as ct

import numpy as np

from . import _lib
from .runtime import np_ptr, require_device

NAME = "b200"

_MASK64 = (1 << 64) - 1


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def clause_outputs(states, lits, training, budget):
    """kernels/_numba.py:53-58: uint8 [C] outputs on one literal vector."""
    require_device()
    states = _c(states, np.int8)
    lits = _c(lits, np.uint8)
    C, P = states.shape
    out = np.empty(C, dtype=np.uint8)
    _lib.call("tmbh_clause_outputs", np_ptr(states), C, P, np_ptr(lits), int(bool(training)),
              int(budget), np_ptr(out))
    return out


def clause_outputs_batch(states, x_lit, training, budget):
    """kernels/_numba.py:61-68: uint8 [N, C] outputs for every row."""
    require_device()
    states = _c(states, np.int8)
    x_lit = _c(x_lit, np.uint8)
    C, P = states.shape
    N = x_lit.shape[0]
    out = np.empty((N, C), dtype=np.uint8)
    _lib.call("tmbh_clause_outputs_batch", np_ptr(states), C, P, np_ptr(x_lit), N,
              int(bool(training)), int(budget), np_ptr(out))
    return out


def _inplace(a, dtype, name):
    if not (isinstance(a, np.ndarray) and a.dtype == dtype and a.flags.c_contiguous
            and a.flags.writeable):
        raise TypeError(f"{name} must be a writeable C-contiguous {np.dtype(dtype)} array")
    return a


def bank_feedback(states, weights, lits, outputs, label, negative, update_target,
                  update_negative, s, boost, state_min, state_max, seed, counter):
    """kernels/_numba.py:101-125: one example's feedback, in place; returns
    the advanced event counter (as np.uint64, like the numba kernel)."""
    require_device()
    states = _inplace(states, np.int8, "states")
    weights = _inplace(weights, np.int32, "weights")
    lits = _c(lits, np.uint8)
    outputs = _c(outputs, np.uint8)
    ut = _c(update_target, np.uint8)
    un = _c(update_negative, np.uint8)
    C, P = states.shape
    K = weights.shape[1]
    new = ct.c_uint64()
    _lib.call("tmbh_bank_feedback", np_ptr(states), np_ptr(weights), C, P, K, np_ptr(lits),
              np_ptr(outputs), int(label), int(negative), np_ptr(ut), np_ptr(un), float(s),
              int(bool(boost)), int(state_min), int(state_max), int(seed) & _MASK64,
              int(counter) & _MASK64, ct.byref(new))
    return np.uint64(new.value)


def bank_feedback_draws(states, weights, lits, outputs, label, negative, update_target,
                        update_negative, s, boost, state_min, state_max, counter, draws):
    """Explicit-draws test hook: applied event i reads the uniform draws
    draws[i, :] instead of the stream (every applied event consumes a row,
    Type II included).  Runs the same device kernel as bank_feedback."""
    require_device()
    import torch

    from .runtime import ptr, stream_ptr, to_dev
    states = _inplace(states, np.int8, "states")
    weights = _inplace(weights, np.int32, "weights")
    draws = _c(draws, np.float64)
    C, P = states.shape
    K = weights.shape[1]
    if draws.ndim != 2 or draws.shape[1] != P:
        raise ValueError("draws must be [n_events, P]")
    ds, dw = to_dev(states), to_dev(weights)
    dl, do = to_dev(lits, np.uint8), to_dev(outputs, np.uint8)
    dut, dun = to_dev(update_target, np.uint8), to_dev(update_negative, np.uint8)
    dd = to_dev(draws)
    new = ct.c_uint64()
    _lib.call("tmb_bank_feedback_draws", ptr(ds), ptr(dw), C, P, K, ptr(dl), ptr(do),
              int(label), int(negative), ptr(dut), ptr(dun), float(s), int(bool(boost)),
              int(state_min), int(state_max), int(counter) & _MASK64, ptr(dd),
              draws.shape[0], ct.byref(new), stream_ptr())
    torch.cuda.current_stream().synchronize()
    states[...] = ds.cpu().numpy()
    weights[...] = dw.cpu().numpy()
    return np.uint64(new.value)


def warmup():
    """Load the library and touch every kernel once on tiny inputs."""
    states = np.zeros((2, 4), dtype=np.int8)
    weights = np.zeros((2, 2), dtype=np.int32)
    lits = np.array([1, 0, 1, 0], dtype=np.uint8)
    flags = np.array([True, False])
    clause_outputs(states, lits, True, 4)
    clause_outputs_batch(states, lits.reshape(1, -1), False, 4)
    bank_feedback(states, weights, lits, np.ones(2, dtype=np.uint8), 0, 1, flags, flags,
                  2.0, False, -127, 127, np.uint64(1), np.uint64(0))


BACKEND_NAME = NAME
