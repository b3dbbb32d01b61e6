# The INTEGRATION.md section-1 stub, verbatim: tsetlinkit/kernels/_b200.py as a
# maintainer of the reference would add it.  tools/run_reference_suite.py drops
# it into a copy of the installed reference (baseline/_ref) and runs the
# reference's own tests with TSETLINKIT_BACKEND=b200.
"""B200 backend: thin ctypes binding of libtmb200.so (host buffers)."""
import ctypes as ct
import os

import numpy as np

NAME = "b200"
_lib = ct.CDLL(os.environ.get("TMB200_LIB", "libtmb200.so"))
_vp, _i64, _i32, _u64, _f64 = ct.c_void_p, ct.c_int64, ct.c_int, ct.c_uint64, ct.c_double
_lib.tmbh_clause_outputs.argtypes = [_vp, _i64, _i64, _vp, _i32, _i64, _vp]
_lib.tmbh_clause_outputs_batch.argtypes = [_vp, _i64, _i64, _vp, _i64, _i32, _i64, _vp]
_lib.tmbh_bank_feedback.argtypes = [_vp, _vp, _i64, _i64, _i64, _vp, _vp, _i64, _i64, _vp, _vp,
                                    _f64, _i32, _i32, _i32, _u64, _u64, _vp]
_lib.tmb_last_error.restype = ct.c_char_p


def _p(a):
    return a.ctypes.data_as(_vp)


def _check(rc):
    if rc != 0:
        raise RuntimeError(_lib.tmb_last_error().decode())


def clause_outputs(states, lits, training, budget):        # kernels/_numba.py:53-58
    states = np.ascontiguousarray(states, np.int8)
    lits = np.ascontiguousarray(lits, np.uint8)
    out = np.empty(states.shape[0], np.uint8)
    _check(_lib.tmbh_clause_outputs(_p(states), states.shape[0], states.shape[1], _p(lits),
                                    int(training), int(budget), _p(out)))
    return out


def clause_outputs_batch(states, x_lit, training, budget):  # kernels/_numba.py:61-68
    states = np.ascontiguousarray(states, np.int8)
    x_lit = np.ascontiguousarray(x_lit, np.uint8)
    out = np.empty((x_lit.shape[0], states.shape[0]), np.uint8)
    _check(_lib.tmbh_clause_outputs_batch(_p(states), states.shape[0], states.shape[1],
                                          _p(x_lit), x_lit.shape[0], int(training),
                                          int(budget), _p(out)))
    return out


def bank_feedback(states, weights, lits, outputs, label, negative, update_target,
                  update_negative, s, boost, state_min, state_max, seed, counter):
    # kernels/_numba.py:101-125 -- states / weights are updated in place
    new = ct.c_uint64()
    c = lambda a, t: np.ascontiguousarray(a, t)  # noqa: E731
    _check(_lib.tmbh_bank_feedback(
        _p(states), _p(weights), states.shape[0], states.shape[1], weights.shape[1],
        _p(c(lits, np.uint8)), _p(c(outputs, np.uint8)), int(label), int(negative),
        _p(c(update_target, np.uint8)), _p(c(update_negative, np.uint8)), float(s),
        int(bool(boost)), int(state_min), int(state_max), int(seed), int(counter),
        ct.byref(new)))
    return np.uint64(new.value)


def warmup():
    clause_outputs(np.zeros((2, 4), np.int8), np.zeros(4, np.uint8), True, 4)
