"""Sparse data and the SparseTM clause bank (mirror of sparse.py:28-285).

``SparseExample`` / ``SparseDataset`` keep the reference's validation and
layout.  ``SparseClauseBank`` keeps its caller-visible storage (per-clause
sorted ``clause_literals`` int64 / ``clause_states`` int8 lists and int32
``weights``); its evaluation and feedback run on the GPU through the
libtmb200 sparse engine (csrc/tmb_sparse.cu).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .core import Config
from .dense import ContractViolation, EvalMode


@dataclass(frozen=True)
class SparseExample:
    """Active literal indices (sorted, unique) plus a class label (sparse.py:28-48)."""

    active: np.ndarray
    label: int

    def __post_init__(self):
        active = np.asarray(self.active, dtype=np.int64)
        if active.ndim != 1:
            raise ContractViolation("active indices must be a 1-D sequence")
        if active.size and (np.any(np.diff(active) <= 0) or active[0] < 0):
            raise ContractViolation("active indices must be sorted, unique and non-negative")
        object.__setattr__(self, "active", active)

    def check_range(self, n_literals: int) -> None:
        if self.active.size and self.active[-1] >= n_literals:
            raise ContractViolation(f"active index {int(self.active[-1])} outside universe of "
                                    f"{n_literals} literals")


@dataclass
class SparseDataset:
    """A sparse example list with its declared literal universe (sparse.py:51-75)."""

    n_literals: int
    examples: list[SparseExample] = field(default_factory=list)

    def __len__(self) -> int:
        return len(self.examples)

    @property
    def labels(self) -> np.ndarray:
        return np.array([ex.label for ex in self.examples], dtype=np.int64)

    def candidate_literals(self) -> np.ndarray:
        if not self.examples:
            return np.empty(0, dtype=np.int64)
        return np.unique(np.concatenate([ex.active for ex in self.examples]))

    def densify(self) -> tuple[np.ndarray, np.ndarray]:
        x = np.zeros((len(self.examples), self.n_literals), dtype=np.uint8)
        for i, ex in enumerate(self.examples):
            x[i, ex.active] = 1
        return x, self.labels

    def to_csr(self):
        """(indptr int64 [N+1], indices int32 [nnz]) -- the device input format."""
        lens = np.array([ex.active.size for ex in self.examples], dtype=np.int64)
        indptr = np.zeros(lens.size + 1, dtype=np.int64)
        np.cumsum(lens, out=indptr[1:])
        idx = (np.concatenate([ex.active for ex in self.examples]).astype(np.int32)
               if self.examples and indptr[-1] else np.zeros(0, np.int32))
        return indptr, idx

    @classmethod
    def from_csr(cls, n_literals, indptr, indices, labels) -> "SparseDataset":
        ex = [SparseExample(np.asarray(indices[indptr[i]:indptr[i + 1]], dtype=np.int64),
                            int(labels[i])) for i in range(len(labels))]
        return cls(n_literals, ex)


class SparseClauseBank:
    """Sorted (literal, state) pair lists per clause (sparse.py:78-256)."""

    kind = "sparse"

    def __init__(self, cfg: Config, n_clauses: int | None = None,
                 candidate_literals: np.ndarray | None = None):
        if cfg.negated_literals_enabled:
            raise ContractViolation("sparse banks require negated_literals_enabled=False")
        self.cfg = cfg
        self.n_clauses = cfg.n_clauses if n_clauses is None else n_clauses
        self.n_literals = cfg.n_literals
        self.n_positions = cfg.n_literals
        self.n_classes = cfg.n_classes
        self.s = cfg.s
        self.boost_true_positive = cfg.boost_true_positive
        self.floor = cfg.sparse_floor
        self.state_max = cfg.state_max
        self.capacity = cfg.sparse_capacity
        self.budget = cfg.effective_budget
        if candidate_literals is None:
            candidate_literals = np.empty(0, dtype=np.int64)
        self.candidates = np.asarray(candidate_literals, dtype=np.int64)
        self.clause_literals: list[np.ndarray] = [np.empty(0, dtype=np.int64)
                                                  for _ in range(self.n_clauses)]
        self.clause_states: list[np.ndarray] = [np.empty(0, dtype=np.int8)
                                                for _ in range(self.n_clauses)]
        self.weights = np.zeros((self.n_clauses, self.n_classes), dtype=np.int32)

    # -- queries (host bookkeeping on the stored lists) -------------------
    def lookup(self, clause: int, literal: int) -> int:
        idx = self.clause_literals[clause]
        pos = int(np.searchsorted(idx, literal))
        if pos < idx.size and idx[pos] == literal:
            return int(self.clause_states[clause][pos])
        return self.floor

    def included_literals(self, clause: int) -> np.ndarray:
        idx = self.clause_literals[clause]
        return idx[self.clause_states[clause] >= 0]

    def memory_report(self) -> dict:
        """sparse.py:149-154: pairs and index+state bytes plus weights."""
        pairs = sum(int(a.size) for a in self.clause_literals)
        return {"pairs": pairs, "bytes": pairs * (4 + 1) + self.weights.size * 4}

    # -- evaluation on the device -----------------------------------------
    def evaluate_clause(self, clause: int, example: SparseExample, mode: EvalMode) -> int:
        return int(self.clause_outputs(example, mode)[clause])

    def clause_outputs(self, example: SparseExample, mode: EvalMode) -> np.ndarray:
        from .sparse_train import sparse_outputs
        return sparse_outputs(self, [example], mode)[0]

    def votes(self, outputs: np.ndarray) -> np.ndarray:
        return outputs.astype(np.int64) @ self.weights.astype(np.int64)

    def batch_votes(self, examples: list[SparseExample]) -> np.ndarray:
        from .sparse_train import sparse_batch_votes
        return sparse_batch_votes(self, examples)

    # -- feedback on the device -------------------------------------------
    def feedback(self, clause, cls, direction, update_sampled, clause_output, example, rng):
        """sparse.py:222-239 (one event)."""
        if direction not in (1, -1):
            raise ContractViolation("direction must be +1 or -1")
        if not update_sampled:
            return
        ut = np.zeros(self.n_clauses, dtype=bool)
        un = np.zeros(self.n_clauses, dtype=bool)
        outputs = np.zeros(self.n_clauses, dtype=np.uint8)
        outputs[clause] = clause_output
        other = (cls + 1) % self.n_classes
        if direction == 1:
            ut[clause] = True
            label, negative = cls, other
        else:
            un[clause] = True
            label, negative = other, cls
        self.apply_feedback(example, outputs, label, negative, ut, un, rng)

    def apply_feedback(self, example, outputs, label, negative, update_target,
                       update_negative, rng) -> None:
        from .sparse_train import sparse_apply_feedback
        sparse_apply_feedback(self, example, outputs, label, negative, update_target,
                              update_negative, rng)

    def copy(self) -> "SparseClauseBank":
        dup = SparseClauseBank(self.cfg, self.n_clauses, self.candidates)
        dup.clause_literals = [a.copy() for a in self.clause_literals]
        dup.clause_states = [a.copy() for a in self.clause_states]
        dup.weights = self.weights.copy()
        return dup


def sparse_lookup(bank, clause, literal):
    return bank.lookup(clause, literal)


def sparse_evaluate_clause(bank, clause, example, mode):
    return bank.evaluate_clause(clause, example, mode)


def sparse_feedback(bank, clause, cls, direction, update_sampled, clause_output, example, rng):
    bank.feedback(clause, cls, direction, update_sampled, clause_output, example, rng)


def sparse_memory_report(bank):
    return bank.memory_report()
