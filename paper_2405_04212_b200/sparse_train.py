"""SparseTM on the device: training sessions and the SparseClauseBank
operations, over libtmb200's sparse engine (csrc/tmb_sparse.cu).

Mirrors executor.train for SparseDataset inputs (executor.py:275-340 with
the sparse branches at :88-97, :287-289): candidates are the union of the
training set's active literals, clause blocks keep their own streams and
counters, and the merged model is one SparseClauseBank in clause order.
"""

from __future__ import annotations

import ctypes as ct
import time

import numpy as np

from . import _lib
from .core import FEEDBACK_STREAM, SHUFFLE_STREAM, RngStream
from .dense import EvalMode
from .runtime import ptr, require_device, stream_ptr

DEFAULT_SLAB = 1024  # (literal, state) pairs per clause held on the device (initial)


def auto_slab(cfg, candidates, longest: int = 0) -> int:
    """Device slab (pairs per clause) for a bank over `candidates`.  With
    sparse_capacity=None a Type II event stores every candidate that is not
    active (sparse.py:192-210), so a list can hold the whole candidate set:
    size for it.  With a capacity, lists stay near it (stored pairs are kept,
    SURVEY 0.8) and start at DEFAULT_SLAB; training sessions grow the slab
    and replay the epoch if a list ever outgrows it."""
    n = DEFAULT_SLAB
    if cfg.sparse_capacity is None:
        n = max(n, int(len(candidates)) + 32)
    return max(n, int(longest) + 2 * (cfg.sparse_capacity or 64) + 64)


def _is_slab_overflow(err) -> bool:
    return isinstance(err, _lib.TmbError) and "slab" in str(err)


def _cfg_struct(cfg, n_clauses=None, n_blocks=None, slab=DEFAULT_SLAB):
    return _lib.SparseCfg(
        cfg.n_literals, cfg.n_clauses if n_clauses is None else n_clauses, cfg.n_classes,
        cfg.n_blocks if n_blocks is None else n_blocks, cfg.threshold, cfg.effective_budget,
        float(cfg.s), int(cfg.boost_true_positive), cfg.sparse_floor, cfg.state_max,
        -1 if cfg.sparse_capacity is None else int(cfg.sparse_capacity),
        cfg.seed & (2 ** 64 - 1), slab)


class SparseEngine:
    """Owns a device sparse model (tmb_sparse handle)."""

    def __init__(self, cfg, candidates, n_clauses=None, n_blocks=None, slab=DEFAULT_SLAB):
        require_device()
        self.cfg = cfg
        self.C = cfg.n_clauses if n_clauses is None else n_clauses
        self.K = cfg.n_classes
        self.n_blocks = cfg.n_blocks if n_blocks is None else n_blocks
        self.slab = (slab + 15) // 16 * 16
        cands = np.ascontiguousarray(candidates, dtype=np.int32)
        cs = _cfg_struct(cfg, self.C, self.n_blocks, self.slab)
        self._h = ct.c_void_p()
        _lib.call("tmb_sparse_create", ct.byref(cs), cands.ctypes.data_as(ct.c_void_p),
                  cands.size, ct.byref(self._h))

    @property
    def resident(self):
        """True if the trainer keeps the clause lists in shared memory."""
        out = (ct.c_int64 * 4)()
        _lib.call("tmb_sparse_layout", self._h, out)
        return bool(out[0])

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.load().tmb_sparse_destroy(h)
            except Exception:
                pass
            self._h = None

    # -- model transfer -----------------------------------------------------
    def set_lists(self, lits, sts, weights, block_counters=None):
        import torch
        lens = np.array([len(a) for a in lits], dtype=np.int32)
        if lens.size and lens.max(initial=0) > self.slab:
            raise _lib.TmbError(_lib.TMB_E_UNSUPPORTED, "clause list longer than the device slab")
        L = np.zeros((self.C, self.slab), dtype=np.int32)
        S = np.zeros((self.C, self.slab), dtype=np.int8)
        for j, (a, b) in enumerate(zip(lits, sts)):
            L[j, :len(a)] = a
            S[j, :len(b)] = b
        dev = torch.device("cuda")
        d = [torch.from_numpy(v).to(dev) for v in (lens, L, S, np.ascontiguousarray(weights, np.int32))]
        bc = None
        if block_counters is not None:
            bc = torch.from_numpy(np.asarray(block_counters, dtype=np.uint64).view(np.int64)).to(dev)
        _lib.call("tmb_sparse_set", self._h, ptr(d[0]), ptr(d[1]), ptr(d[2]), ptr(d[3]), ptr(bc),
                  stream_ptr())
        torch.cuda.current_stream().synchronize()

    def get_lists(self):
        import torch
        dev = torch.device("cuda")
        lens = torch.empty(self.C, dtype=torch.int32, device=dev)
        L = torch.zeros((self.C, self.slab), dtype=torch.int32, device=dev)
        S = torch.zeros((self.C, self.slab), dtype=torch.int8, device=dev)
        W = torch.empty((self.C, self.K), dtype=torch.int32, device=dev)
        BC = torch.empty(self.n_blocks, dtype=torch.int64, device=dev)
        _lib.call("tmb_sparse_get", self._h, ptr(lens), ptr(L), ptr(S), ptr(W), ptr(BC),
                  stream_ptr())
        torch.cuda.current_stream().synchronize()
        lens, L, S = lens.cpu().numpy(), L.cpu().numpy(), S.cpu().numpy()
        lits = [L[j, :lens[j]].astype(np.int64) for j in range(self.C)]
        sts = [S[j, :lens[j]].copy() for j in range(self.C)]
        return lits, sts, W.cpu().numpy(), BC.cpu().numpy().view(np.uint64)

    # -- compute ----------------------------------------------------------------
    def votes_and_pred(self, indptr_dev, indices_dev, n):
        import torch
        votes = torch.empty((n, self.K), dtype=torch.int64, device="cuda")
        pred = torch.empty(n, dtype=torch.int64, device="cuda")
        _lib.call("tmb_sparse_infer", self._h, ptr(indptr_dev), ptr(indices_dev), n, ptr(votes),
                  ptr(pred), stream_ptr())
        return votes, pred

    def outputs(self, indptr_dev, indices_dev, n):
        import torch
        out = torch.empty((n, self.C), dtype=torch.uint8, device="cuda")
        _lib.call("tmb_sparse_outputs", self._h, ptr(indptr_dev), ptr(indices_dev), n, ptr(out),
                  stream_ptr())
        return out


def _csr_dev(examples):
    import torch
    lens = np.array([ex.active.size for ex in examples], dtype=np.int64)
    indptr = np.zeros(lens.size + 1, dtype=np.int64)
    np.cumsum(lens, out=indptr[1:])
    idx = (np.concatenate([ex.active for ex in examples]).astype(np.int32)
           if len(examples) and indptr[-1] else np.zeros(1, np.int32))
    return (torch.from_numpy(indptr).cuda(), torch.from_numpy(np.ascontiguousarray(idx)).cuda(),
            len(examples))


class SparseTrainSession:
    """Device-resident sparse training (model, CSR data, RNG counters)."""

    def __init__(self, cfg, indptr, indices, labels, candidates=None, slab=None):
        import torch
        require_device()
        self.cfg = cfg
        indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        indices = np.ascontiguousarray(indices, dtype=np.int32)
        if candidates is None:
            candidates = np.unique(indices)
        self.candidates = np.asarray(candidates, dtype=np.int64)
        self.engine = SparseEngine(cfg, self.candidates,
                                   slab=auto_slab(cfg, self.candidates) if slab is None else slab)
        self.N = labels.shape[0]
        self.indptr = torch.from_numpy(indptr).cuda()
        self.indices = torch.from_numpy(indices if indices.size else np.zeros(1, np.int32)).cuda()
        self.labels = torch.from_numpy(np.asarray(labels, dtype=np.int32)).cuda()
        self.fb_counter = 0
        self.shuffle_rng = RngStream.derive(cfg.seed, SHUFFLE_STREAM)
        self.stats = torch.zeros(6, dtype=torch.int64, device="cuda")

    def run_steps(self, order_dev, n_steps=None):
        n = int(order_dev.shape[0]) if n_steps is None else n_steps
        _lib.call("tmb_sparse_train", self.engine._h, ptr(self.indptr), ptr(self.indices),
                  ptr(self.labels), ptr(order_dev), n, self.fb_counter & (2 ** 64 - 1),
                  ptr(self.stats), stream_ptr())
        self.fb_counter += n * (1 + 2 * self.cfg.n_clauses)

    def run_steps_on(self, indptr_dev, indices_dev, labels_dev, order_dev):
        """Like run_steps, on caller-provided device CSR rows / labels (a
        batch staged by a data loader) instead of the session's own copy."""
        n = int(order_dev.shape[0])
        _lib.call("tmb_sparse_train", self.engine._h, ptr(indptr_dev), ptr(indices_dev),
                  ptr(labels_dev), ptr(order_dev), n, self.fb_counter & (2 ** 64 - 1),
                  ptr(self.stats), stream_ptr())
        self.fb_counter += n * (1 + 2 * self.cfg.n_clauses)

    def run_epoch(self, max_steps=None):
        import torch
        from .executor import shuffle_permutation
        order = shuffle_permutation(self.N, self.shuffle_rng).astype(np.int32)
        if max_steps is not None:
            order = order[:max_steps]
        od = torch.from_numpy(order).cuda()
        self.run_steps(od)
        return od

    def snapshot(self):
        """Host copy of the training state (lists, weights, counters)."""
        return self.engine.get_lists(), self.fb_counter, self.shuffle_rng.counter

    def restore(self, snap, slab=None):
        """Back to a snapshot, optionally on a new engine with a larger slab."""
        (lits, sts, w, bc), fb, sh = snap
        if slab is not None and slab != self.engine.slab:
            self.engine = SparseEngine(self.cfg, self.candidates, slab=slab)
        self.engine.set_lists(lits, sts, w, bc)
        self.fb_counter = fb
        self.shuffle_rng.counter = sh

    def run_epoch_growing(self, max_steps=None):
        """run_epoch that survives a clause list outgrowing the device slab:
        the epoch is replayed from its start on a slab twice as large (the
        result is the same model; only the storage grew)."""
        snap = self.snapshot()
        while True:
            try:
                return self.run_epoch(max_steps)
            except _lib.TmbError as err:
                if not _is_slab_overflow(err):
                    raise
                self.restore(snap, slab=2 * self.engine.slab)

    def model(self):
        from .sparse import SparseClauseBank
        lits, sts, w, _ = self.engine.get_lists()
        bank = SparseClauseBank(self.cfg, candidate_literals=self.candidates)
        bank.clause_literals = lits
        bank.clause_states = sts
        bank.weights = w
        return bank

    def stats_dict(self):
        v = self.stats.cpu().numpy()
        return dict(zip(["examples", "events", "type_i", "type_ii", "draws", "state_updates"],
                        [int(a) for a in v]))


def train_sparse(cfg, inp, evl, n_epochs, epoch_callback, observer, TrainRun, EpochMetric):
    """executor.train for SparseDataset inputs (executor.py:275-340)."""
    import torch
    from .sparse import SparseClauseBank
    data = inp.data
    indptr, indices = data.to_csr()
    metrics = []
    cands = data.candidate_literals()
    if n_epochs <= 0:
        return TrainRun(cfg, metrics, SparseClauseBank(cfg, candidate_literals=cands))
    sess = SparseTrainSession(cfg, indptr, indices, inp.labels, candidates=cands)
    ev = None
    if evl is not None:
        ev = _csr_dev(evl.data.examples)
    for epoch in range(n_epochs):
        t0 = time.perf_counter()
        sess.run_epoch_growing()
        if observer:
            torch.cuda.current_stream().synchronize()
            for step in range(len(inp)):
                for b in range(cfg.n_blocks):
                    observer("votes", (epoch, step), b)
                observer("decision", (epoch, step), None)
                for b in range(cfg.n_blocks):
                    observer("update", (epoch, step), b)
        acc = None
        if ev is not None:
            _, pred = sess.engine.votes_and_pred(*ev)
            acc = float(np.mean(pred.cpu().numpy() == evl.labels))
        torch.cuda.current_stream().synchronize()
        metrics.append(EpochMetric(epoch, acc, time.perf_counter() - t0))
        if epoch_callback:
            epoch_callback(metrics[-1])
    return TrainRun(cfg, metrics, sess.model())


def _engine_for_bank(bank):
    eng = SparseEngine(bank.cfg, bank.candidates, n_clauses=bank.n_clauses, n_blocks=1,
                       slab=auto_slab(bank.cfg, bank.candidates,
                                      max((len(a) for a in bank.clause_literals), default=0)))
    eng.set_lists(bank.clause_literals, bank.clause_states, bank.weights)
    return eng


def sparse_outputs(bank, examples, mode):
    """SparseClauseBank.clause_outputs (sparse.py:123-138) for a batch."""
    eng = _engine_for_bank(bank)
    out = eng.outputs(*_csr_dev(examples)).cpu().numpy()
    if mode is EvalMode.TRAINING:
        # training conventions: empty clause -> 1, over budget -> 0
        n_inc = np.array([int((s >= 0).sum()) for s in bank.clause_states])
        out = out.copy()
        out[:, n_inc == 0] = 1
        out[:, n_inc > bank.budget] = 0
    return out


def sparse_batch_votes(bank, examples):
    """SparseClauseBank.batch_votes (sparse.py:140-147)."""
    eng = _engine_for_bank(bank)
    votes, _ = eng.votes_and_pred(*_csr_dev(examples))
    return votes.cpu().numpy()


def sparse_apply_feedback(bank, example, outputs, label, negative, update_target,
                          update_negative, rng):
    """SparseClauseBank.apply_feedback (sparse.py:241-249) on the device."""
    import torch
    eng = _engine_for_bank(bank)
    dev = torch.device("cuda")
    act = torch.from_numpy(np.ascontiguousarray(example.active, dtype=np.int32)
                           if example.active.size else np.zeros(1, np.int32)).to(dev)
    o = torch.from_numpy(np.ascontiguousarray(outputs, dtype=np.uint8)).to(dev)
    ut = torch.from_numpy(np.ascontiguousarray(update_target, dtype=np.uint8)).to(dev)
    un = torch.from_numpy(np.ascontiguousarray(update_negative, dtype=np.uint8)).to(dev)
    new = ct.c_uint64()
    _lib.call("tmb_sparse_feedback", eng._h, ptr(act), int(example.active.size), ptr(o),
              int(label), int(negative), ptr(ut), ptr(un), rng.stream_seed & (2 ** 64 - 1),
              rng.counter & (2 ** 64 - 1), ct.byref(new), stream_ptr())
    lits, sts, w, _ = eng.get_lists()
    bank.clause_literals = lits
    bank.clause_states = sts
    bank.weights = w
    rng.counter = int(new.value)
