"""Cross-validation and random search over the GPU trainer (tuning.py of the
reference).

``stratified_kfold``, ``cross_validate``, ``SearchSpace`` and
``random_search`` keep the reference's semantics (fold assignment from the
KFOLD stream, fold model seed = derive_stream(seed, fold), one SEARCH-stream
draw per parameter in declaration order, the holdout split from the HOLDOUT
stream), so fold / trial models are bit-identical to the reference's.  Folds
and trials are independent trainings; with a torch.distributed group they run
one job per rank (one GPU each, ``parallel.run_jobs``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, fields

import numpy as np

from .core import (HOLDOUT_STREAM, KFOLD_STREAM, SEARCH_STREAM, Config, DataError, RngStream,
                   derive_stream)
from .executor import shuffle_permutation
from .sparse import SparseDataset


@dataclass
class CvReport:
    fold_accuracies: list
    mean: float
    std: float
    fold_assignments: np.ndarray


def labels_of(data) -> np.ndarray:
    if isinstance(data, SparseDataset):
        return data.labels
    return np.asarray(data[1], dtype=np.int64)


def subset(data, mask: np.ndarray):
    if isinstance(data, SparseDataset):
        return SparseDataset(data.n_literals, [ex for ex, m in zip(data.examples, mask) if m])
    x, y = data
    return np.asarray(x)[mask], np.asarray(y)[mask]


def stratified_kfold(labels, k: int, seed: int) -> np.ndarray:
    """Fold index per example: seeded shuffle within each class, then
    round-robin (tuning.py:157-173)."""
    labels = np.asarray(labels, dtype=np.int64)
    if k < 2:
        raise ValueError("k must be at least 2")
    rng = RngStream.derive(seed, KFOLD_STREAM)
    folds = np.empty(labels.shape[0], dtype=np.int64)
    for cls in np.unique(labels):
        idx = np.flatnonzero(labels == cls)
        if idx.size < k:
            raise DataError(f"class {int(cls)} has {idx.size} examples, fewer than k={k}")
        perm = shuffle_permutation(idx.size, rng)
        folds[idx[perm]] = np.arange(idx.size) % k
    return folds


def fold_configs(cfg, k: int, seed: int):
    """The k fold configurations of cross_validate (tuning.py:184)."""
    return [cfg.with_overrides(seed=derive_stream(seed, fold)) for fold in range(k)]


def cross_validate(cfg, data, k: int, n_epochs: int, seed: int, n_jobs: int = 1,
                   group=None, train_fn=None, evaluate_fn=None) -> CvReport:
    """tuning.py:176-191; with a process group the folds run one per rank."""
    from . import parallel
    from .executor import evaluate, train
    train_fn = train_fn or (lambda c, d, e: train(c, d, n_epochs=e, n_jobs=n_jobs).model)
    evaluate_fn = evaluate_fn or evaluate
    labels = labels_of(data)
    folds = stratified_kfold(labels, k, seed)
    cfgs = fold_configs(cfg, k, seed)

    def job(fold):
        held = folds == fold
        model = train_fn(cfgs[fold], subset(data, ~held), n_epochs)
        return evaluate_fn(model, subset(data, held))

    accs = parallel.run_jobs(k, job, group=group)
    mean = float(np.mean(accs))
    std = float(np.std(accs, ddof=1)) if k > 1 else 0.0
    return CvReport(list(accs), mean, std, folds)


# ---------------------------------------------------------------- search --
_KIND_OF = {f.name: str(f.type) for f in fields(Config)}


@dataclass(frozen=True)
class SearchSpace:
    """Ranges over Config fields (tuning.py:34-101): ``int`` (inclusive),
    ``uniform`` / ``loguniform`` (real) and ``cat`` (listed values), as
    ``(name, kind, spec)`` triples."""

    params: tuple

    def __post_init__(self):
        for name, kind, spec in self.params:
            if kind == "cat":
                if not spec:
                    raise ValueError(f"{name}: empty categorical list")
                continue
            if kind not in ("int", "uniform", "loguniform"):
                raise ValueError(f"{name}: unknown kind {kind!r}")
            lo, hi = spec
            if lo > hi:
                raise ValueError(f"{name}: lower bound {lo} above upper bound {hi}")
            if kind == "loguniform" and lo <= 0:
                raise ValueError(f"{name}: loguniform requires positive bounds")

    @classmethod
    def parse(cls, text: str) -> "SearchSpace":
        """One parameter per line, ``name kind lo hi`` or ``name cat v1,v2``;
        blank lines and ``#`` comments are skipped (tuning.py:59-80)."""
        out = []
        for no, raw in enumerate(text.splitlines(), start=1):
            line = raw.strip()
            if not line or line.startswith("#"):
                continue
            tok = line.split()
            if len(tok) == 3 and tok[1] == "cat":
                out.append((tok[0], "cat", tuple(_scalar(v) for v in tok[2].split(","))))
            elif len(tok) == 4 and tok[1] in ("int", "uniform", "loguniform"):
                cast = int if tok[1] == "int" else float
                out.append((tok[0], tok[1], (cast(tok[2]), cast(tok[3]))))
            else:
                raise ValueError(f"space line {no}: unrecognized spec {line!r}")
        return cls(tuple(out))

    def sample(self, rng: RngStream) -> dict:
        """One draw per parameter in declaration order (tuning.py:82-101)."""
        out = {}
        for name, kind, spec in self.params:
            u = rng.next_u01()
            if kind == "cat":
                out[name] = spec[min(len(spec) - 1, int(u * len(spec)))]
                continue
            lo, hi = spec
            if kind == "int":
                out[name] = min(hi, lo + int(u * (hi - lo + 1)))
            elif kind == "uniform":
                out[name] = lo + u * (hi - lo)
            else:
                out[name] = math.exp(math.log(lo) + u * (math.log(hi) - math.log(lo)))
        return out


def _scalar(tok: str):
    """true/false, then int, then float, else the string (tuning.py:104-114)."""
    if tok.lower() in ("true", "false"):
        return tok.lower() == "true"
    for cast in (int, float):
        try:
            return cast(tok)
        except ValueError:
            pass
    return tok


def _coerce(name: str, value):
    """Cast a sampled value to the Config field's type (tuning.py:117-124)."""
    kind = _KIND_OF.get(name, "")
    if kind in ("int", "int | None"):
        return value if isinstance(value, bool) else int(round(value))
    if kind == "float":
        return float(value)
    if kind == "bool":
        return bool(value)
    return value


@dataclass
class Trial:
    index: int
    params: dict
    config: Config
    accuracy: float


def random_search(space: SearchSpace, base_cfg, data, n_trials: int, n_epochs: int, seed: int,
                  cv_k: int | None = None, holdout_fraction: float = 0.2, n_jobs: int = 1,
                  group=None, train_fn=None, evaluate_fn=None) -> list:
    """tuning.py:194-227: draw ``n_trials`` configurations from the SEARCH
    stream, train each, score it on a stratified holdout shared by all
    trials (or by ``cv_k``-fold cross-validation), and rank by accuracy
    (ties keep the earlier trial).  All draws happen before any training --
    the stream advances only by sampling, so this is the reference's order --
    and with a process group the trials run one per rank."""
    from . import parallel
    from .executor import evaluate, train
    if n_trials < 1:
        raise ValueError("n_trials must be at least 1")
    train_fn = train_fn or (lambda c, d, e: train(c, d, n_epochs=e, n_jobs=n_jobs).model)
    evaluate_fn = evaluate_fn or evaluate
    rng = RngStream.derive(seed, SEARCH_STREAM)
    draws = [space.sample(rng) for _ in range(n_trials)]
    cfgs = [base_cfg.with_overrides(**{k: _coerce(k, v) for k, v in d.items()}) for d in draws]
    if cv_k is None:
        per_fold = max(2, int(round(1.0 / max(holdout_fraction, 1e-9))))
        hold = stratified_kfold(labels_of(data), per_fold,
                                derive_stream(seed, HOLDOUT_STREAM)) == 0
        fit, held = subset(data, ~hold), subset(data, hold)

        def job(t):
            return evaluate_fn(train_fn(cfgs[t], fit, n_epochs), held)
    else:
        def job(t):
            return cross_validate(cfgs[t], data, cv_k, n_epochs, seed, n_jobs,
                                  train_fn=train_fn, evaluate_fn=evaluate_fn).mean
    accs = parallel.run_jobs(n_trials, job, group=group)
    trials = [Trial(t, draws[t], cfgs[t], float(accs[t])) for t in range(n_trials)]
    return sorted(trials, key=lambda tr: (-tr.accuracy, tr.index))
