"""Multi-GPU plumbing: one process per GPU over
torch.distributed (NCCL on the GPU box, gloo for CPU tests).

* Batched inference shards examples: contiguous ranges per rank, the model
  replicated; no collective on the hot path -- predictions are gathered once.
* Hyper-parameter grids and CV folds are independent trainings: job j runs on
  rank j mod world; results are gathered in job order.
* Per-example online training is sequential and is not
  sharded -- "replicas only".
"""

from __future__ import annotations

import os

import numpy as np


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) of n items for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world / rank")
    return n * rank // world, n * (rank + 1) // world


def csr_shard(indptr: np.ndarray, world: int, rank: int) -> tuple[int, int]:
    """Row range [lo, hi) of a CSR matrix for `rank` of `world`, balanced by
    non-zeros (the work of sparse inference is per posting): rank r starts
    at the first row whose prefix nnz reaches r/world of the total."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world / rank")
    indptr = np.asarray(indptr, dtype=np.int64)
    n = indptr.size - 1
    nnz = int(indptr[-1]) if n > 0 else 0

    def start(r):
        if r <= 0:
            return 0
        if r >= world:
            return n
        if nnz == 0:
            return n * r // world
        return int(np.searchsorted(indptr[:n], nnz * r // world, side="left"))

    return start(rank), start(rank + 1)


def jobs_of(n_jobs: int, world: int, rank: int) -> list[int]:
    """Round-robin job assignment (job j -> rank j mod world)."""
    return list(range(rank, n_jobs, world))


def world_info(group=None) -> tuple[int, int]:
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def init_from_env(backend: str | None = None):
    """Initialise torch.distributed from torchrun's environment (no-op for
    a single process).  Returns (world, rank, local_rank)."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return world, rank, local


def run_jobs(n_jobs: int, job, group=None) -> list:
    """Run job(j) for every j on its rank; every rank gets all results in
    job order (all_gather_object)."""
    import torch.distributed as dist
    world, rank = world_info(group)
    mine = {j: job(j) for j in jobs_of(n_jobs, world, rank)}
    if world == 1:
        return [mine[j] for j in range(n_jobs)]
    gathered = [None] * world
    dist.all_gather_object(gathered, mine, group=group)
    out = {}
    for part in gathered:
        out.update(part)
    return [out[j] for j in range(n_jobs)]


def run_sweep(configs, train_data, eval_data, n_epochs: int, group=None, train_fn=None,
              evaluate_fn=None) -> list:
    """Independent trainings of `configs` (e.g. configs[3]'s 8-point s x T
    grid), one job per config spread over the ranks; returns the evaluation
    accuracy of every config in order."""
    from .executor import evaluate, train
    train_fn = train_fn or (lambda c, d, e: train(c, d, n_epochs=e).model)
    evaluate_fn = evaluate_fn or evaluate
    return run_jobs(len(configs),
                    lambda j: evaluate_fn(train_fn(configs[j], train_data, n_epochs), eval_data),
                    group=group)


def gather_rows(local: np.ndarray, n_total: int, group=None) -> np.ndarray:
    """Reassemble per-rank contiguous shards (shard_range order)."""
    import torch.distributed as dist
    world, rank = world_info(group)
    if world == 1:
        return local
    gathered = [None] * world
    dist.all_gather_object(gathered, local, group=group)
    out = np.concatenate(gathered, axis=0)
    assert out.shape[0] == n_total
    return out


def sharded_predict(model, x: np.ndarray, group=None) -> np.ndarray:
    """Predictions of a CompiledModel for x [N, F] with the examples split
    over the ranks (each rank computes only its shard on its GPU)."""
    world, rank = world_info(group)
    lo, hi = shard_range(x.shape[0], world, rank)
    _, pred = model.votes_and_pred(x[lo:hi], want_votes=False)
    return gather_rows(pred, x.shape[0], group)


def sharded_sparse_predict(engine, indptr: np.ndarray, indices: np.ndarray, group=None):
    """Predictions of a device sparse model (sparse_train.SparseEngine) for a
    CSR document set, rows split over the ranks by csr_shard (each rank
    evaluates only its rows on its GPU), gathered once."""
    import torch
    world, rank = world_info(group)
    lo, hi = csr_shard(indptr, world, rank)
    a, b = int(indptr[lo]), int(indptr[hi])
    ip = torch.from_numpy(np.ascontiguousarray(indptr[lo:hi + 1] - a, dtype=np.int64)).cuda()
    ix = torch.from_numpy(np.ascontiguousarray(
        indices[a:b] if b > a else np.zeros(1, np.int32), dtype=np.int32)).cuda()
    _, pred = engine.votes_and_pred(ip, ix, hi - lo)
    return gather_rows(pred.cpu().numpy(), indptr.size - 1, group)
