"""The paper's listing-level API:
``TsetlinMachine`` / ``Trainer`` / ``get_predictor`` / ``predict_and_explain``
/ ``export_as_program``.  These names do not exist in the reference package
(it exposes Config / train / compile_ruleset); they are thin mappings onto
the same GPU-backed functions, as the north star asks.
"""

from __future__ import annotations

import numpy as np

from .core import Config
from .executor import TrainRun, train
from .predictor import (RuleSet, compile_ruleset, predict, predict_and_explain,
                        predict_and_explain_batch, predict_batch)


class TsetlinMachine:
    """``TsetlinMachine(n_literals, n_clauses, n_classes, s, threshold,
    n_literal_budget)`` -> a Config plus the trained model."""

    def __init__(self, n_literals: int, n_clauses: int, n_classes: int, s: float,
                 threshold: int, n_literal_budget: int | None = None, **kw):
        self.config = Config(n_literals=n_literals, n_clauses=n_clauses,
                             n_classes=n_classes, s=s, threshold=threshold,
                             n_literal_budget=n_literal_budget, **kw)
        self.model = None

    def get_predictor(self, explanation: str = "none", exclude_negative_clauses: bool = False):
        if self.model is None:
            raise RuntimeError("train the machine before asking for a predictor")
        return Predictor(compile_ruleset(self.model), explanation)


class Trainer:
    """``Trainer(tm, n_epochs, seed, n_jobs)`` with set_train_data /
    set_eval_data / train()."""

    def __init__(self, tm: TsetlinMachine, n_epochs: int = 1, seed: int | None = None,
                 n_jobs: int = 1, progress_bar: bool = False):
        self.tm = tm
        self.n_epochs = n_epochs
        self.n_jobs = n_jobs
        if seed is not None:
            tm.config = tm.config.with_overrides(seed=seed)
        self.train_data = None
        self.eval_data = None
        self.results: TrainRun | None = None

    def set_train_data(self, x, y):
        self.train_data = (np.asarray(x, dtype=np.uint8), np.asarray(y))

    def set_eval_data(self, x, y):
        self.eval_data = (np.asarray(x, dtype=np.uint8), np.asarray(y))

    def train(self) -> dict:
        if self.train_data is None:
            raise RuntimeError("set_train_data first")
        self.results = train(self.tm.config, self.train_data, self.eval_data,
                             n_epochs=self.n_epochs, n_jobs=self.n_jobs)
        self.tm.model = self.results.model
        accs = [m.accuracy for m in self.results.epoch_metrics]
        best = max((a for a in accs if a is not None), default=None)
        return {"train_time_of_epochs": [m.seconds for m in self.results.epoch_metrics],
                "eval_acc": accs, "best_eval_acc": best}


class Predictor:
    """``tm.get_predictor()``: predict / predict_and_explain /
    export_as_program over the compiled rule set."""

    def __init__(self, rules: RuleSet, explanation: str = "none"):
        self.rules = rules
        self.explanation = explanation

    def predict(self, x):
        x = np.asarray(x, dtype=np.uint8)
        if x.ndim == 2:
            return predict_batch(self.rules, x)
        return predict(self.rules, x)

    def predict_and_explain(self, x, level: str = "literal", for_class: int | None = None):
        return predict_and_explain(self.rules, x, level, for_class)

    def predict_and_explain_batch(self, x, level: str = "literal",
                                  for_class: int | None = None):
        return predict_and_explain_batch(self.rules, x, level, for_class)

    def export_as_program(self, path: str, name: str = "tm"):
        """C99 code generation (export_c.py) is outside the GPU hot path's
        scope ("Out of scope")."""
        raise NotImplementedError("export_as_program: C99 export is out of scope for the "
                                  "B200 build; use the reference's export_c on the RuleSet")
