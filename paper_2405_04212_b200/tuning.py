"""Cross-validation over the GPU trainer (tuning.py:157-191 of the reference).

``stratified_kfold`` and ``cross_validate`` keep the reference's semantics
(fold assignment from the KFOLD stream, fold model seed =
derive_stream(seed, fold)), so fold models are bit-identical to the
reference's.  Folds are independent trainings; ``parallel.run_folds`` spreads
them over the ranks of a torch.distributed group (one GPU each).
``random_search`` / ``SearchSpace`` (the sampling utility) are outside the
B200 hot path ("Out of scope").
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import KFOLD_STREAM, DataError, RngStream, derive_stream
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
