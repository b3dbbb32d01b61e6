"""Seeded synthetic workloads with the shapes of BASELINE.json's five configs.

No public dataset is used or needed: BASELINE.json names only synthetic
inputs ("MNIST-shaped", "sentiment-shaped"), so every generator here is a
seeded numpy function of ``data_seed`` and the CPU oracle and the GPU consume
byte-identical arrays.  Choices that BASELINE.json leaves open are recorded in
the docstrings.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_MASK64 = (1 << 64) - 1
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def _mix64_vec(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _C1
    z = (z ^ (z >> np.uint64(27))) * _C2
    return z ^ (z >> np.uint64(31))


# --------------------------------------------------------------- config 1 --

def noisy_xor(data_seed: int = 2024, n_train: int = 5000, n_test: int = 5000,
              n_features: int = 12, flip_fraction: float = 0.4):
    """C1: 12 Bernoulli(0.5) features, label = x0 XOR x1; exactly 40 % of the
    training labels flipped (indices without replacement); clean test set."""
    rng = np.random.default_rng(data_seed)
    x = rng.integers(0, 2, size=(n_train + n_test, n_features)).astype(np.uint8)
    y = (x[:, 0] ^ x[:, 1]).astype(np.int64)
    tx, ty = x[:n_train], y[:n_train].copy()
    flip = rng.choice(n_train, size=int(round(flip_fraction * n_train)), replace=False)
    ty[flip] = 1 - ty[flip]
    return (tx, ty), (x[n_train:], y[n_train:])


def noisy_xor_config_kwargs(seed: int = 0) -> dict:
    """C1 model: 2 classes, 10 clauses, T=15, s=3.9, init at the boundary."""
    return dict(n_literals=12, n_clauses=10, n_classes=2, s=3.9, threshold=15,
                init_state=-1, seed=seed, n_blocks=1)


# --------------------------------------------------------------- config 2 --

def _prototypes(rng, n_classes=10, side=28):
    yy, xx = np.mgrid[0:side, 0:side].astype(np.float64)
    protos = np.zeros((n_classes, side, side), dtype=np.uint8)
    for c in range(n_classes):
        field = np.zeros((side, side))
        for _ in range(3):
            cy, cx = rng.uniform(6, 22, size=2)
            sigma = rng.uniform(2, 4)
            field += np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / (2 * sigma ** 2))
        protos[c] = (field > 0.5).astype(np.uint8)
    return protos


def mnist_shaped(data_seed: int = 7, n_train: int = 60000, n_test: int = 10000,
                 n_classes: int = 10, side: int = 28, max_shift: int = 2,
                 flip_p: float = 0.08):
    """C2: 10 class prototypes (3 thresholded Gaussian blobs each: centres
    U[6,22]^2, sigma U[2,4], threshold 0.5); an example is its prototype
    shifted by (dy, dx) ~ U{-2..2}^2 with zero fill, then each pixel flipped
    with p = 0.08.  Balanced classes, shuffled."""
    rng = np.random.default_rng(data_seed)
    protos = _prototypes(rng, n_classes, side)
    pad = np.pad(protos, ((0, 0), (max_shift, max_shift), (max_shift, max_shift)))

    def make(n):
        y = np.repeat(np.arange(n_classes), n // n_classes)
        y = np.concatenate([y, rng.integers(0, n_classes, size=n - y.size)])
        rng.shuffle(y)
        dy = rng.integers(-max_shift, max_shift + 1, size=n)
        dx = rng.integers(-max_shift, max_shift + 1, size=n)
        x = np.empty((n, side, side), dtype=np.uint8)
        for sy in range(-max_shift, max_shift + 1):
            for sx in range(-max_shift, max_shift + 1):
                sel = np.flatnonzero((dy == sy) & (dx == sx))
                if sel.size == 0:
                    continue
                win = pad[:, max_shift - sy:max_shift - sy + side,
                          max_shift - sx:max_shift - sx + side]
                x[sel] = win[y[sel]]
        flips = rng.random((n, side, side)) < flip_p
        x ^= flips.astype(np.uint8)
        return x.reshape(n, side * side), y.astype(np.int64)

    return make(n_train), make(n_test)


def mnist_shaped_config_kwargs(seed: int = 0) -> dict:
    return dict(n_literals=784, n_clauses=2000, n_classes=10, s=10.0, threshold=5000,
                seed=seed, n_blocks=1)


# --------------------------------------------------------------- config 3 --

def inference_stream_seed(data_seed: int) -> int:
    """Stream seed of the counter-based C3 example generator."""
    from .core import derive_stream
    return derive_stream(data_seed, 0)


def inference_examples(data_seed: int, start: int, count: int, n_features: int = 4096,
                       packed: bool = False) -> np.ndarray:
    """C3 inputs: Bernoulli(0.5) bits as a pure function of (data_seed,
    example index), so any shard or single example can be regenerated.
    Feature f of example e is bit (f % 64) of stream_u64(seed, e*W + f//64),
    W = ceil(F / 64).  Returns uint8 [count, F] (or uint64 [count, W] when
    packed)."""
    W = (n_features + 63) // 64
    seed = np.uint64(inference_stream_seed(data_seed))
    k = (np.arange(count * W, dtype=np.uint64) + np.uint64(start * W) + np.uint64(1))
    words = _mix64_vec(seed + _GOLDEN * k).reshape(count, W)
    if packed:
        return words
    bits = np.unpackbits(words.view(np.uint8).reshape(count, W * 8), axis=1,
                         bitorder="little")
    return np.ascontiguousarray(bits[:, :n_features])


def inference_examples_device(data_seed: int, start: int, count: int, n_features: int = 4096,
                              packed: bool = False):
    """Device twin of ``inference_examples`` (same bits): the stream words are
    filled by tmb_stream_u64_block on the current stream and expanded to
    uint8 [count, F] (or returned as int64 [count, W] words when packed)."""
    import torch

    from . import _lib
    from .runtime import ptr, stream_ptr
    W = (n_features + 63) // 64
    seed = inference_stream_seed(data_seed)
    if packed:
        words = torch.empty((count, W), dtype=torch.int64, device="cuda")
        _lib.call("tmb_stream_u64_block", seed, start * W, count * W, ptr(words), stream_ptr())
        return words
    x = torch.empty((count, n_features), dtype=torch.uint8, device="cuda")
    chunk = 1 << 18
    shifts = torch.arange(8, device="cuda", dtype=torch.uint8)
    for lo in range(0, count, chunk):
        m = min(chunk, count - lo)
        words = torch.empty(m * W, dtype=torch.int64, device="cuda")
        _lib.call("tmb_stream_u64_block", seed, (start + lo) * W, m * W, ptr(words),
                  stream_ptr())
        b = words.view(torch.uint8).view(m, W * 8)
        bits = (b.unsqueeze(-1) >> shifts) & 1
        x[lo:lo + m] = bits.view(m, W * 64)[:, :n_features]
        del words, b, bits
    return x


@dataclass
class InferenceModel:
    states: np.ndarray   # int8 [C, 2F]: 0 = include, -1 = exclude
    weights: np.ndarray  # int32 [C, K]


def inference_model(model_seed: int = 11, n_features: int = 4096, n_clauses: int = 10000,
                    n_classes: int = 10, n_includes: int = 20,
                    weight_range: int = 100) -> InferenceModel:
    """C3 model: each clause includes `n_includes` positions drawn uniformly
    without replacement from the 2F literal positions (state 0 = include,
    -1 = exclude); weights uniform ints in [-100, 100]."""
    rng = np.random.default_rng(model_seed)
    P = 2 * n_features
    states = np.full((n_clauses, P), -1, dtype=np.int8)
    keys = rng.random((n_clauses, P))
    inc = np.argpartition(keys, n_includes, axis=1)[:, :n_includes]
    np.put_along_axis(states, inc, 0, axis=1)
    weights = rng.integers(-weight_range, weight_range + 1,
                           size=(n_clauses, n_classes)).astype(np.int32)
    return InferenceModel(states, weights)


# --------------------------------------------------------------- config 4 --

def _zipf_probs(n: int, a: float) -> np.ndarray:
    p = 1.0 / np.arange(1, n + 1, dtype=np.float64) ** a
    return p / p.sum()


def _distinct_zipf_rows(rng, n_rows, n_tokens, vocab, a, rank_to_id):
    """Rows of `n_tokens` distinct ids drawn from a finite Zipf(a) over ranks
    1..vocab (duplicates redrawn), mapped through a fixed rank->id permutation."""
    cdf = np.cumsum(_zipf_probs(vocab, a))
    out = np.empty((n_rows, n_tokens), dtype=np.int64)
    for i in range(n_rows):
        got = np.empty(0, dtype=np.int64)
        need = n_tokens
        while need > 0:
            draw = np.searchsorted(cdf, rng.random(2 * need + 8), side="right")
            draw = np.minimum(draw, vocab - 1)
            got = np.concatenate([got, draw])
            _, first = np.unique(got, return_index=True)
            got = got[np.sort(first)]
            need = n_tokens - got.size
        out[i] = np.sort(rank_to_id[got[:n_tokens]])
    return out


def bag_of_words(data_seed: int = 4, n_train: int = 25000, n_test: int = 25000,
                 vocab: int = 10000, n_tokens: int = 150, a: float = 1.1,
                 n_planted: int = 200, noise: float = 0.1):
    """C4: documents of 150 distinct Zipf(1.1) word ids over a 10^4 vocabulary.
    Planted disjoint positive / negative sets of 200 ids each are drawn from
    ranks 20..1019 (frequent enough to be learnable); label = 1 iff
    count_pos - count_neg > 0 (ties -> 0), then 10 % of labels flipped."""
    rng = np.random.default_rng(data_seed)
    rank_to_id = rng.permutation(vocab)
    planted = rank_to_id[20 + rng.permutation(1000)[:2 * n_planted]]
    pos, neg = planted[:n_planted], planted[n_planted:]
    n = n_train + n_test
    rows = _distinct_zipf_rows(rng, n, n_tokens, vocab, a, rank_to_id)
    x = np.zeros((n, vocab), dtype=np.uint8)
    np.put_along_axis(x, rows, 1, axis=1)
    score = x[:, pos].sum(axis=1).astype(np.int64) - x[:, neg].sum(axis=1)
    y = (score > 0).astype(np.int64)
    flip = rng.random(n) < noise
    y[flip] = 1 - y[flip]
    return (x[:n_train], y[:n_train]), (x[n_train:], y[n_train:])


def bag_of_words_config_kwargs(seed: int = 0, s: float = 2.0, threshold: int = 10000) -> dict:
    return dict(n_literals=10000, n_clauses=10000, n_classes=2, s=s, threshold=threshold,
                seed=seed, n_blocks=1)


SWEEP_GRID = [(s, t) for s in (1.5, 2.0, 3.0, 5.0) for t in (5000, 10000)]


# --------------------------------------------------------------- config 5 --

@dataclass
class CSRDocs:
    n_literals: int
    indptr: np.ndarray   # int64 [N+1]
    indices: np.ndarray  # int32 [nnz], sorted within each row
    labels: np.ndarray   # int64 [N]

    def __len__(self):
        return self.labels.shape[0]

    def row(self, i):
        return self.indices[self.indptr[i]:self.indptr[i + 1]].astype(np.int64)


def sparse_zipf(data_seed: int = 5, n_docs: int = 1_000_000, vocab: int = 1_000_000,
                n_tokens: int = 100, a: float = 1.05, n_planted: int = 500,
                planted_lo: int = 100, planted_span: int = 5000) -> CSRDocs:
    """C5: documents of 100 distinct Zipf(1.05) ids over a 10^6 vocabulary,
    stored as CSR.  500 planted indicator ids per class are drawn from ranks
    100..5099 (planted_lo .. planted_lo + planted_span - 1); label = class
    with the larger planted count, ties broken by a coin from the data
    stream."""
    rng = np.random.default_rng(data_seed)
    rank_to_id = rng.permutation(vocab)
    planted = rank_to_id[planted_lo + rng.permutation(planted_span)[:2 * n_planted]]
    cls0, cls1 = np.sort(planted[:n_planted]), np.sort(planted[n_planted:])
    cdf = np.cumsum(_zipf_probs(vocab, a))
    indptr = np.arange(n_docs + 1, dtype=np.int64) * n_tokens
    indices = np.empty(n_docs * n_tokens, dtype=np.int32)
    chunk = 1 << 16
    for lo in range(0, n_docs, chunk):
        hi = min(lo + chunk, n_docs)
        m = hi - lo
        draw = np.minimum(np.searchsorted(cdf, rng.random((m, 2 * n_tokens)), side="right"),
                          vocab - 1)
        rows = np.empty((m, n_tokens), dtype=np.int64)
        for i in range(m):
            _, first = np.unique(draw[i], return_index=True)
            uniq = draw[i][np.sort(first)]
            while uniq.size < n_tokens:
                extra = np.minimum(np.searchsorted(cdf, rng.random(2 * n_tokens), side="right"),
                                   vocab - 1)
                cat = np.concatenate([uniq, extra])
                _, first = np.unique(cat, return_index=True)
                uniq = cat[np.sort(first)]
            rows[i] = np.sort(rank_to_id[uniq[:n_tokens]])
        indices[lo * n_tokens:hi * n_tokens] = rows.reshape(-1)
    c0 = np.isin(indices, cls0).reshape(n_docs, n_tokens).sum(axis=1)
    c1 = np.isin(indices, cls1).reshape(n_docs, n_tokens).sum(axis=1)
    coin = rng.integers(0, 2, size=n_docs)
    labels = np.where(c1 > c0, 1, np.where(c0 > c1, 0, coin)).astype(np.int64)
    return CSRDocs(vocab, indptr, indices, labels)


def sparse_config_kwargs(seed: int = 0) -> dict:
    """C5 model: 2000 clauses, T=2000, s=5.0, negations off; the "literal
    budget of 64" maps to sparse_capacity=64 and the absorbing threshold to
    the reference floor / evict rule (sparse_floor=-15)."""
    return dict(n_literals=1_000_000, n_clauses=2000, n_classes=2, s=5.0, threshold=2000,
                seed=seed, n_blocks=1, negated_literals_enabled=False,
                sparse_capacity=64, sparse_floor=-15)
