"""GTM1 model files, byte-identical to the reference's (
dataio.py:148-291): a GPU-trained dense bank, sparse bank or rule set saved
here loads in the reference and vice versa.

Layout (all little-endian, no padding):
  b"GTM1" | u16 version (1) | u8 kind (1 dense, 2 sparse, 3 rule set)
  dense / sparse: config record
      u64 n_literals, u32 n_clauses, u32 n_classes, f64 s, i32 threshold,
      u32 budget (0xFFFFFFFF = None), u8 boost, i8 init_state, i8 state_min,
      i8 state_max, u64 seed, u32 n_blocks, u8 negations, i8 sparse_floor,
      u32 sparse_capacity (0xFFFFFFFF = None)
  dense:  int8 states [C, P] | int32 weights [C, K]
  sparse: per clause u32 count, then count x (u32 literal, i8 state) |
          int32 weights [C, K]
  rule set: u64 n_literals, u32 n_rules, u32 n_classes, u8 negations, then
          per rule u32 count, u32 includes [count], int32 weights [K]
Loading checks the magic, the version, the kind and that nothing trails.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .core import Config, DataError

MAGIC = b"GTM1"
FORMAT_VERSION = 1
KIND_DENSE, KIND_SPARSE, KIND_RULESET = 1, 2, 3
UNLIMITED = 0xFFFFFFFF
_CFG = struct.Struct("<QIIdiIBbbbQIBbI")
_PAIR = np.dtype([("lit", "<u4"), ("st", "i1")])  # packed: 5 bytes per pair


class ModelFormatError(DataError):
    """Malformed / unsupported model file (dataio.py:35-36)."""


def _config_bytes(cfg: Config) -> bytes:
    return _CFG.pack(cfg.n_literals, cfg.n_clauses, cfg.n_classes, float(cfg.s), cfg.threshold,
                     UNLIMITED if cfg.n_literal_budget is None else cfg.n_literal_budget,
                     int(bool(cfg.boost_true_positive)), cfg.init_state, cfg.state_min,
                     cfg.state_max, cfg.seed, cfg.n_blocks, int(bool(cfg.negated_literals_enabled)),
                     cfg.sparse_floor, UNLIMITED if cfg.sparse_capacity is None else cfg.sparse_capacity)


def _config_from(fields) -> Config:
    (n_literals, n_clauses, n_classes, s, threshold, budget, boost, init_state, state_min,
     state_max, seed, n_blocks, negations, floor, capacity) = fields
    return Config(n_literals=n_literals, n_clauses=n_clauses, n_classes=n_classes, s=s,
                  threshold=threshold, n_literal_budget=None if budget == UNLIMITED else budget,
                  boost_true_positive=bool(boost), init_state=init_state, state_min=state_min,
                  state_max=state_max, seed=seed, n_blocks=n_blocks,
                  negated_literals_enabled=bool(negations), sparse_floor=floor,
                  sparse_capacity=None if capacity == UNLIMITED else capacity)


def model_bytes(model) -> bytes:
    """The GTM1 encoding of a DenseClauseBank, SparseClauseBank or RuleSet."""
    from .dense import DenseClauseBank
    from .predictor import RuleSet
    from .sparse import SparseClauseBank
    parts = [MAGIC, struct.pack("<H", FORMAT_VERSION)]
    if isinstance(model, DenseClauseBank):
        parts += [struct.pack("<B", KIND_DENSE), _config_bytes(model.cfg),
                  np.ascontiguousarray(model.states, dtype=np.int8).tobytes(),
                  np.ascontiguousarray(model.weights, dtype="<i4").tobytes()]
    elif isinstance(model, SparseClauseBank):
        parts += [struct.pack("<B", KIND_SPARSE), _config_bytes(model.cfg)]
        for lits, sts in zip(model.clause_literals, model.clause_states):
            rec = np.empty(len(lits), dtype=_PAIR)
            rec["lit"] = np.asarray(lits, dtype=np.int64)
            rec["st"] = np.asarray(sts, dtype=np.int8)
            parts += [struct.pack("<I", len(lits)), rec.tobytes()]
        parts.append(np.ascontiguousarray(model.weights, dtype="<i4").tobytes())
    elif isinstance(model, RuleSet):
        parts += [struct.pack("<B", KIND_RULESET),
                  struct.pack("<QII", model.n_literals, model.n_rules, model.n_classes),
                  struct.pack("<B", int(bool(model.negated_literals_enabled)))]
        for inc, row in zip(model.includes, model.weights):
            inc = np.asarray(inc, dtype="<u4")
            parts += [struct.pack("<I", inc.size), inc.tobytes(),
                      np.ascontiguousarray(row, dtype="<i4").tobytes()]
    else:
        raise TypeError(f"cannot serialize {type(model).__name__}")
    return b"".join(parts)


def save_model(model, path) -> None:
    Path(path).write_bytes(model_bytes(model))


class _Cursor:
    def __init__(self, raw: bytes):
        self.raw, self.pos = memoryview(raw), 0

    def take(self, n: int) -> memoryview:
        if self.pos + n > len(self.raw):
            raise ModelFormatError("truncated model file")
        out = self.raw[self.pos:self.pos + n]
        self.pos += n
        return out

    def unpack(self, fmt: str):
        st = struct.Struct("<" + fmt)
        return st.unpack(self.take(st.size))


def model_from_bytes(raw: bytes):
    from .dense import DenseClauseBank
    from .predictor import RuleSet
    from .sparse import SparseClauseBank
    cur = _Cursor(raw)
    if bytes(cur.take(4)) != MAGIC:
        raise ModelFormatError("bad magic: not a model file")
    (version,) = cur.unpack("H")
    if version != FORMAT_VERSION:
        raise ModelFormatError(f"unsupported model format version {version}")
    (kind,) = cur.unpack("B")
    if kind in (KIND_DENSE, KIND_SPARSE):
        cfg = _config_from(_CFG.unpack(cur.take(_CFG.size)))
        if kind == KIND_DENSE:
            model = DenseClauseBank(cfg)
            C, P, K = model.n_clauses, model.n_positions, model.n_classes
            model.states = np.frombuffer(cur.take(C * P), dtype=np.int8).reshape(C, P).copy()
        else:
            model = SparseClauseBank(cfg)
            C, K = model.n_clauses, model.n_classes
            lits, sts = [], []
            for _ in range(C):
                (count,) = cur.unpack("I")
                rec = np.frombuffer(cur.take(_PAIR.itemsize * count), dtype=_PAIR)
                lits.append(rec["lit"].astype(np.int64))
                sts.append(rec["st"].astype(np.int8))
            model.clause_literals, model.clause_states = lits, sts
        model.weights = np.frombuffer(cur.take(4 * C * K), dtype="<i4").reshape(C, K).astype(np.int32)
    elif kind == KIND_RULESET:
        n_literals, n_rules, n_classes = cur.unpack("QII")
        (negations,) = cur.unpack("B")
        includes, weights = [], np.empty((n_rules, n_classes), dtype=np.int32)
        for r in range(n_rules):
            (count,) = cur.unpack("I")
            includes.append(np.frombuffer(cur.take(4 * count), dtype="<u4").astype(np.int64))
            weights[r] = np.frombuffer(cur.take(4 * n_classes), dtype="<i4")
        model = RuleSet(n_literals, n_classes, bool(negations), tuple(includes), weights)
    else:
        raise ModelFormatError(f"unknown model kind {kind}")
    if cur.pos != len(cur.raw):
        raise ModelFormatError("trailing bytes after model payload")
    return model


def load_model(path):
    """Inverse of save_model; returns the same kind of object."""
    return model_from_bytes(Path(path).read_bytes())
