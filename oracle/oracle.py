"""CPU parity oracle (TEST INFRASTRUCTURE ONLY).

Python glue over ``liboracle.so`` (``tm_oracle.c``), a plain-C restatement of
the reference ``tsetlinkit`` hot path.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this module, and only as the checker / the
CPU baseline -- never as the product.  Each function names the reference
file:line it restates (paths relative to
``/root/reference/pkg/src/tsetlinkit``).

Parity of this oracle with the reference is pinned by
``tests/test_oracle_golden.py`` against fixtures produced by importing the
reference itself (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes as ct
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

GOLDEN = 0x9E3779B97F4A7C15
MASK64 = (1 << 64) - 1
SHUFFLE_STREAM = 0xD157
FEEDBACK_STREAM = 0xFEED


def build(force: bool = False) -> str:
    """Compile liboracle.so with the committed Makefile (gcc only)."""
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "tm_oracle.c")):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ct.CDLL(_LIB_PATH)
        u64, i64, f64, i32 = ct.c_uint64, ct.c_int64, ct.c_double, ct.c_int
        vp = ct.c_void_p
        L.or_mix64.restype = u64
        L.or_mix64.argtypes = [u64]
        L.or_derive_stream.restype = u64
        L.or_derive_stream.argtypes = [u64, u64]
        L.or_stream_u64.restype = u64
        L.or_stream_u64.argtypes = [u64, u64]
        L.or_stream_u01.restype = f64
        L.or_stream_u01.argtypes = [u64, u64]
        L.or_stream_u64_block.argtypes = [u64, u64, i64, vp]
        L.or_stream_u01_block.argtypes = [u64, u64, i64, vp]
        L.or_clause_outputs.argtypes = [vp, i64, i64, vp, i32, i64, vp]
        L.or_clause_outputs_batch.argtypes = [vp, i64, i64, vp, i64, i32, i64, vp, i32]
        L.or_batch_votes.argtypes = [vp, vp, i64, i64, i64, vp, i64, vp, vp, i32]
        L.or_ruleset_votes.argtypes = [vp, vp, i64, vp, i64, vp, i64, i64, i32, vp, vp, i32]
        L.or_bank_feedback.restype = u64
        L.or_bank_feedback.argtypes = [vp, vp, i64, i64, i64, vp, vp, i64, i64, vp, vp,
                                       f64, i32, i32, i32, u64, u64]
        L.or_bank_feedback_draws.restype = u64
        L.or_bank_feedback_draws.argtypes = [vp, vp, i64, i64, i64, vp, vp, i64, i64, vp, vp,
                                             f64, i32, i32, i32, u64, vp, i64]
        L.or_update_probabilities.argtypes = [vp, i64, i64, i64, f64, vp, vp, vp]
        L.or_sample_updates.argtypes = [f64, f64, i64, u64, u64, vp, vp]
        L.or_shuffle_permutation.restype = u64
        L.or_shuffle_permutation.argtypes = [i64, u64, u64, vp]
        L.or_train_steps.argtypes = [vp, vp, vp, vp, vp, vp, i64, vp, vp]
        L.or_sparse_event.restype = i64
        L.or_sparse_event.argtypes = [vp, vp, i64, vp, i64, vp, i64, i32, i32, f64, i32,
                                      i32, i32, i64, u64, u64, vp, vp]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ct.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ------------------------------------------------------------------ RNG --

def mix64(z: int) -> int:                      # core.py:66-71
    return int(lib().or_mix64(z & MASK64))


def derive_stream(seed: int, index: int) -> int:  # core.py:74-85
    return int(lib().or_derive_stream(seed & MASK64, index & MASK64))


def stream_u64(seed: int, k: int) -> int:      # core.py:88-90
    return int(lib().or_stream_u64(seed & MASK64, k & MASK64))


def stream_u01(seed: int, k: int) -> float:    # core.py:93-95
    return float(lib().or_stream_u01(seed & MASK64, k & MASK64))


def stream_u64_block(seed: int, start: int, count: int) -> np.ndarray:  # core.py:98-104
    out = np.empty(count, dtype=np.uint64)
    lib().or_stream_u64_block(seed & MASK64, start & MASK64, count, _p(out))
    return out


def stream_u01_block(seed: int, start: int, count: int) -> np.ndarray:  # core.py:107-109
    out = np.empty(count, dtype=np.float64)
    lib().or_stream_u01_block(seed & MASK64, start & MASK64, count, _p(out))
    return out


# -------------------------------------------------------------- kernels --

def augment_literals(x, negations: bool = True) -> np.ndarray:  # core.py:232-242
    x = np.asarray(x, dtype=np.uint8)
    if not negations:
        return np.ascontiguousarray(x)
    return np.ascontiguousarray(np.concatenate([x, 1 - x], axis=-1))


def clause_outputs(states, lits, training: bool, budget: int) -> np.ndarray:  # _numba.py:53-58
    states = _c(states, np.int8)
    lits = _c(lits, np.uint8)
    out = np.empty(states.shape[0], dtype=np.uint8)
    lib().or_clause_outputs(_p(states), states.shape[0], states.shape[1], _p(lits),
                            int(bool(training)), int(budget), _p(out))
    return out


def clause_outputs_batch(states, x_lit, training: bool, budget: int,
                         nthreads: int = 1) -> np.ndarray:  # _numba.py:61-68
    states = _c(states, np.int8)
    x_lit = _c(x_lit, np.uint8)
    n = x_lit.shape[0]
    out = np.empty((n, states.shape[0]), dtype=np.uint8)
    lib().or_clause_outputs_batch(_p(states), states.shape[0], states.shape[1], _p(x_lit),
                                  n, int(bool(training)), int(budget), _p(out), nthreads)
    return out


def batch_votes(states, weights, x_lit, nthreads: int = 1, want_votes=True):
    """dense.py:171-174 + argmax (executor.py:382).  Returns (votes, pred)."""
    states = _c(states, np.int8)
    weights = _c(weights, np.int32)
    x_lit = _c(x_lit, np.uint8)
    n = x_lit.shape[0]
    C, P = states.shape
    K = weights.shape[1]
    votes = np.empty((n, K), dtype=np.int64) if want_votes else None
    pred = np.empty(n, dtype=np.int64)
    lib().or_batch_votes(_p(states), _p(weights), C, P, K, _p(x_lit), n,
                         _p(votes) if want_votes else None, _p(pred), nthreads)
    return votes, pred


def ruleset_votes(includes, weights, x, n_literals: int, negations: bool = True,
                  nthreads: int = 1, want_votes=True):
    """predictor.py:79-91 over a batch of raw feature rows."""
    x = _c(x, np.uint8).reshape(-1, n_literals)
    weights = _c(weights, np.int32).reshape(len(includes), -1) if len(includes) else \
        _c(weights, np.int32)
    K = weights.shape[1]
    ptr = np.zeros(len(includes) + 1, dtype=np.int64)
    for r, inc in enumerate(includes):
        ptr[r + 1] = ptr[r] + len(inc)
    idx = (np.concatenate([np.asarray(i, dtype=np.int64) for i in includes])
           if len(includes) else np.zeros(1, dtype=np.int64))
    idx = _c(idx, np.int64)
    n = x.shape[0]
    votes = np.empty((n, K), dtype=np.int64) if want_votes else None
    pred = np.empty(n, dtype=np.int64)
    w = weights if weights.size else np.zeros((1, K), dtype=np.int32)
    lib().or_ruleset_votes(_p(ptr), _p(idx), len(includes), _p(w), K, _p(x), n,
                           n_literals, int(bool(negations)),
                           _p(votes) if want_votes else None, _p(pred), nthreads)
    return votes, pred


def bank_feedback(states, weights, lits, outputs, label, negative, update_target,
                  update_negative, s, boost, state_min, state_max, seed, counter) -> int:
    """_numba.py:101-125; mutates states / weights in place, returns counter."""
    assert states.dtype == np.int8 and states.flags.c_contiguous
    assert weights.dtype == np.int32 and weights.flags.c_contiguous
    lits = _c(lits, np.uint8)
    outputs = _c(outputs, np.uint8)
    ut = _c(update_target, np.uint8)
    un = _c(update_negative, np.uint8)
    C, P = states.shape
    return int(lib().or_bank_feedback(
        _p(states), _p(weights), C, P, weights.shape[1], _p(lits), _p(outputs),
        int(label), int(negative), _p(ut), _p(un), float(s), int(bool(boost)),
        int(state_min), int(state_max), int(seed) & MASK64, int(counter) & MASK64))


def bank_feedback_draws(states, weights, lits, outputs, label, negative, update_target,
                        update_negative, s, boost, state_min, state_max, counter,
                        draws) -> int:
    """Explicit-draws test hook: applied event i reads draws[i, :]."""
    assert states.dtype == np.int8 and states.flags.c_contiguous
    assert weights.dtype == np.int32 and weights.flags.c_contiguous
    lits = _c(lits, np.uint8)
    outputs = _c(outputs, np.uint8)
    ut = _c(update_target, np.uint8)
    un = _c(update_negative, np.uint8)
    draws = _c(draws, np.float64)
    C, P = states.shape
    assert draws.ndim == 2 and draws.shape[1] == P
    return int(lib().or_bank_feedback_draws(
        _p(states), _p(weights), C, P, weights.shape[1], _p(lits), _p(outputs),
        int(label), int(negative), _p(ut), _p(un), float(s), int(bool(boost)),
        int(state_min), int(state_max), int(counter) & MASK64, _p(draws), draws.shape[0]))


def update_probabilities(votes, label: int, threshold: int, u: float):
    """feedback.py:33-44 given the negative-class draw u."""
    votes = _c(votes, np.int64)
    neg = ct.c_int64()
    pt = ct.c_double()
    pn = ct.c_double()
    lib().or_update_probabilities(_p(votes), votes.shape[0], int(label), int(threshold),
                                  float(u), ct.byref(neg), ct.byref(pt), ct.byref(pn))
    return int(neg.value), float(pt.value), float(pn.value)


def sample_updates(p_target, p_negative, n_clauses, fb_seed, fb_counter):
    """feedback.py:47-53: target draws then negative draws from fb_counter."""
    ut = np.empty(n_clauses, dtype=np.uint8)
    un = np.empty(n_clauses, dtype=np.uint8)
    lib().or_sample_updates(float(p_target), float(p_negative), n_clauses,
                            fb_seed & MASK64, fb_counter & MASK64, _p(ut), _p(un))
    return ut.astype(bool), un.astype(bool)


def shuffle_permutation(n: int, seed: int, counter: int):
    """executor.py:50-58.  Returns (perm, new_counter)."""
    perm = np.empty(max(n, 1), dtype=np.int64)
    c = int(lib().or_shuffle_permutation(n, seed & MASK64, counter & MASK64, _p(perm)))
    return perm[:n], c


def partition_clauses(n_clauses: int, n_blocks: int):  # executor.py:36-47
    base, extra = divmod(n_clauses, n_blocks)
    out, start = [], 0
    for b in range(n_blocks):
        size = base + (1 if b < extra else 0)
        out.append(range(start, start + size))
        start += size
    return out


# ------------------------------------------------------------- training --

class _TrainCfg(ct.Structure):
    _fields_ = [("n_literals", ct.c_int64), ("n_positions", ct.c_int64),
                ("n_clauses", ct.c_int64), ("n_classes", ct.c_int64),
                ("n_blocks", ct.c_int64), ("threshold", ct.c_int64),
                ("budget", ct.c_int64), ("s", ct.c_double), ("boost", ct.c_int),
                ("state_min", ct.c_int), ("state_max", ct.c_int), ("seed", ct.c_uint64)]


@dataclass
class OracleCfg:
    """Mirror of core.Config (core.py:156-229), the fields the hot path reads."""
    n_literals: int
    n_clauses: int
    n_classes: int
    s: float
    threshold: int
    n_literal_budget: int | None = None
    boost_true_positive: bool = False
    init_state: int = -1
    state_min: int = -127
    state_max: int = 127
    seed: int = 0
    n_blocks: int = 1
    negated_literals_enabled: bool = True
    sparse_floor: int = -15
    sparse_capacity: int | None = None

    @property
    def n_positions(self):                        # core.py:213-218
        return 2 * self.n_literals if self.negated_literals_enabled else self.n_literals

    @property
    def budget(self):                             # core.py:220-226
        if self.n_literal_budget is None:
            return self.n_positions
        return min(self.n_literal_budget, self.n_positions)


def as_oracle_cfg(cfg) -> OracleCfg:
    names = [f for f in OracleCfg.__dataclass_fields__]
    return OracleCfg(**{n: getattr(cfg, n) for n in names})


@dataclass
class OracleTrainState:
    states: np.ndarray
    weights: np.ndarray
    block_counters: np.ndarray
    fb_counter: int
    shuffle_counter: int


def new_train_state(cfg) -> OracleTrainState:
    cfg = as_oracle_cfg(cfg)
    return OracleTrainState(
        np.full((cfg.n_clauses, cfg.n_positions), cfg.init_state, dtype=np.int8),
        np.zeros((cfg.n_clauses, cfg.n_classes), dtype=np.int32),
        np.zeros(cfg.n_blocks, dtype=np.uint64), 0, 0)


def train_steps(cfg, st: OracleTrainState, x_lit, labels, order):
    """executor.py:326-330 inner loop (serial driver) over `order`."""
    cfg = as_oracle_cfg(cfg)
    tc = _TrainCfg(cfg.n_literals, cfg.n_positions, cfg.n_clauses, cfg.n_classes,
                   cfg.n_blocks, cfg.threshold, cfg.budget, float(cfg.s),
                   int(cfg.boost_true_positive), cfg.state_min, cfg.state_max,
                   cfg.seed & MASK64)
    x_lit = _c(x_lit, np.uint8)
    labels = _c(labels, np.int64)
    order = _c(order, np.int64)
    fb = ct.c_uint64(st.fb_counter)
    lib().or_train_steps(ct.byref(tc), _p(st.states), _p(st.weights), _p(x_lit),
                         _p(labels), _p(order), order.shape[0], _p(st.block_counters),
                         ct.byref(fb))
    st.fb_counter = int(fb.value)


def train(cfg, x, y, n_epochs: int = 1, eval_data=None, state: OracleTrainState | None = None,
          nthreads: int = 1):
    """executor.train (executor.py:275-340) for dense data.  Returns
    (OracleTrainState, [accuracy per epoch or None])."""
    ocfg = as_oracle_cfg(cfg)
    x_lit = augment_literals(x, ocfg.negated_literals_enabled)
    y = np.asarray(y, dtype=np.int64)
    st = state if state is not None else new_train_state(ocfg)
    shuffle_seed = derive_stream(ocfg.seed, SHUFFLE_STREAM)
    accs = []
    for _ in range(n_epochs):
        order, st.shuffle_counter = shuffle_permutation(len(y), shuffle_seed, st.shuffle_counter)
        train_steps(ocfg, st, x_lit, y, order)
        acc = None
        if eval_data is not None:
            ex, ey = eval_data
            _, pred = batch_votes(st.states, st.weights,
                                  augment_literals(ex, ocfg.negated_literals_enabled),
                                  nthreads=nthreads, want_votes=False)
            acc = float(np.mean(pred == np.asarray(ey, dtype=np.int64)))
        accs.append(acc)
    return st, accs


# --------------------------------------------------------------- sparse --

class SparseOracleBank:
    """SparseClauseBank (sparse.py:78-256) with the per-event merge walk in C."""

    def __init__(self, cfg, n_clauses=None, candidates=None):
        self.cfg = as_oracle_cfg(cfg)
        self.n_clauses = self.cfg.n_clauses if n_clauses is None else n_clauses
        self.lits = [np.empty(0, dtype=np.int64) for _ in range(self.n_clauses)]
        self.sts = [np.empty(0, dtype=np.int8) for _ in range(self.n_clauses)]
        self.weights = np.zeros((self.n_clauses, self.cfg.n_classes), dtype=np.int32)
        self.candidates = _c(candidates if candidates is not None else np.empty(0, np.int64),
                             np.int64)

    def included(self, j):                         # sparse.py:119-121
        return self.lits[j][self.sts[j] >= 0]

    def clause_outputs(self, active, training: bool):  # sparse.py:123-138
        active = np.asarray(active, dtype=np.int64)
        out = np.empty(self.n_clauses, dtype=np.uint8)
        for j in range(self.n_clauses):
            inc = self.included(j)
            if inc.size == 0:
                out[j] = 1 if training else 0
            elif training and inc.size > self.cfg.budget:
                out[j] = 0
            else:
                out[j] = 1 if np.all(np.isin(inc, active, assume_unique=True)) else 0
        return out

    def event(self, j, kind, output, active, seed, base):
        n_in = self.lits[j].size
        active = _c(active, np.int64)
        cap_extra = active.size if kind == 1 else self.candidates.size
        lo = np.empty(n_in + cap_extra + 1, dtype=np.int64)
        so = np.empty(n_in + cap_extra + 1, dtype=np.int8)
        li = _c(self.lits[j], np.int64)
        si = _c(self.sts[j], np.int8)
        cap = -1 if self.cfg.sparse_capacity is None else self.cfg.sparse_capacity
        n = lib().or_sparse_event(
            _p(li), _p(si), n_in, _p(active), active.size, _p(self.candidates),
            self.candidates.size, kind, int(output), float(self.cfg.s),
            int(self.cfg.boost_true_positive), self.cfg.sparse_floor, self.cfg.state_max,
            cap, seed & MASK64, base & MASK64, _p(lo), _p(so))
        self.lits[j] = lo[:n].copy()
        self.sts[j] = so[:n].copy()

    def apply_feedback(self, active, outputs, label, negative, ut, un, seed, counter):
        """sparse.py:222-249; returns the advanced block counter."""
        for j in range(self.n_clauses):
            for flag, cls, direction in ((ut[j], label, 1), (un[j], negative, -1)):
                if not flag:
                    continue
                w = self.weights[j, cls]
                type_i = (w >= 0) if direction == 1 else (w < 0)
                base = (counter << 32) & MASK64
                self.event(j, 1 if type_i else 2, int(outputs[j]), active, seed, base)
                if outputs[j] == 1:
                    self.weights[j, cls] += direction
                counter += 1
        return counter


def sparse_train(cfg, examples_active, labels, n_epochs=1, max_steps=None, candidates=None,
                 order=None, progress=None):
    """executor.train for a SparseDataset (executor.py:275-340 with the
    sparse branches at :88-97, :287-289).  examples_active: list (or any
    indexable) of sorted int64 arrays.  candidates: the training set's
    candidate literals when examples_active is only part of it (default: the
    union of examples_active, sparse.py:65-69).  order: explicit example
    order of ONE epoch instead of the shuffle (the caller applied
    shuffle_permutation itself).  Returns (banks per block, block counters,
    fb counter)."""
    ocfg = as_oracle_cfg(cfg)
    labels = np.asarray(labels, dtype=np.int64)
    if candidates is not None:
        cands = np.asarray(candidates, dtype=np.int64)
    else:
        cands = (np.unique(np.concatenate(list(examples_active))) if len(examples_active)
                 else np.empty(0, np.int64))
    ranges = partition_clauses(ocfg.n_clauses, ocfg.n_blocks)
    banks = [SparseOracleBank(ocfg, len(r), cands) for r in ranges]
    bseeds = [derive_stream(ocfg.seed, b) for b in range(ocfg.n_blocks)]
    bctr = [0] * ocfg.n_blocks
    fb_seed = derive_stream(ocfg.seed, FEEDBACK_STREAM)
    sh_seed = derive_stream(ocfg.seed, SHUFFLE_STREAM)
    fb, sh = 0, 0
    steps = 0
    for _ in range(n_epochs):
        if order is None:
            ep_order, sh = shuffle_permutation(len(labels), sh_seed, sh)
        else:
            ep_order = order
        for idx in ep_order:
            if max_steps is not None and steps >= max_steps:
                return banks, bctr, fb
            if progress is not None:
                progress(steps)
            fb = _sparse_step(ocfg, banks, ranges, bseeds, bctr, fb_seed, fb,
                              examples_active[idx], int(labels[idx]))
            steps += 1
    return banks, bctr, fb


def _sparse_step(ocfg, banks, ranges, bseeds, bctr, fb_seed, fb, act, label):
    """One example of executor.py:326-330 on sparse banks; updates bctr in
    place, returns the new feedback counter."""
    C = ocfg.n_clauses
    outs = [bk.clause_outputs(act, True) for bk in banks]
    votes = sum(o.astype(np.int64) @ bk.weights.astype(np.int64)
                for o, bk in zip(outs, banks))
    u = stream_u01(fb_seed, fb)
    neg, pt, pn = update_probabilities(votes, label, ocfg.threshold, u)
    ut, un = sample_updates(pt, pn, C, fb_seed, fb + 1)
    fb += 1 + 2 * C
    for b, (bk, r) in enumerate(zip(banks, ranges)):
        sl = slice(r.start, r.stop)
        bctr[b] = bk.apply_feedback(act, outs[b], label, neg, ut[sl], un[sl],
                                    bseeds[b], bctr[b])
    return fb


def sparse_train_from(cfg, banks, bctr, fb, docs, labels):
    """Continue sparse training from a given state (banks per block, block
    counters, feedback counter) over docs in the given order."""
    ocfg = as_oracle_cfg(cfg)
    ranges = partition_clauses(ocfg.n_clauses, ocfg.n_blocks)
    bseeds = [derive_stream(ocfg.seed, b) for b in range(ocfg.n_blocks)]
    fb_seed = derive_stream(ocfg.seed, FEEDBACK_STREAM)
    bctr = [int(c) for c in bctr]
    for act, label in zip(docs, labels):
        fb = _sparse_step(ocfg, banks, ranges, bseeds, bctr, fb_seed, fb, act, int(label))
    return banks, bctr, fb


def sparse_batch_votes(banks, examples_active):
    """sparse.py:140-147 summed over blocks (executor.py:343-352)."""
    K = banks[0].cfg.n_classes
    votes = np.zeros((len(examples_active), K), dtype=np.int64)
    for i, act in enumerate(examples_active):
        for bk in banks:
            votes[i] += bk.clause_outputs(act, False).astype(np.int64) @ bk.weights.astype(np.int64)
    return votes
