"""Feedback block (mirror of feedback.py:20-53).

On the training hot path this logic runs inside the fused kernel
(csrc/tmb_train.cu, step 5-6: every CTA recomputes the decision from the
all-reduced votes and random-access feedback-stream draws).  These host
functions keep the reference's public helpers with identical semantics;
``sample_updates`` evaluates its 2*C draws on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import RngStream


def clip_votes(v: int, threshold: int) -> int:
    """Clamp a vote sum to [-T, T] (feedback.py:20-22)."""
    return min(threshold, max(-threshold, v))


@dataclass(frozen=True)
class UpdateDecision:
    target_class: int
    negative_class: int
    p_target: float
    p_negative: float


def update_probabilities(votes: np.ndarray, label: int, threshold: int,
                         rng: RngStream) -> UpdateDecision:
    """feedback.py:33-44: one draw picks the negative class uniformly among
    the others; p_t = (T - clip(v_label)) / 2T, p_n = (T + clip(v_neg)) / 2T."""
    n_classes = votes.shape[0]
    u = rng.next_u01()
    negative = (label + 1 + int(u * (n_classes - 1))) % n_classes
    p_target = (threshold - clip_votes(int(votes[label]), threshold)) / (2.0 * threshold)
    p_negative = (threshold + clip_votes(int(votes[negative]), threshold)) / (2.0 * threshold)
    return UpdateDecision(label, negative, p_target, p_negative)


def _device_u53(stream_seed: int, start: int, count: int) -> np.ndarray:
    """Top-53-bit draws start..start+count-1 computed on the GPU."""
    import torch

    from . import _lib
    from .runtime import ptr, require_device, stream_ptr
    require_device()
    out = torch.empty(max(count, 1), dtype=torch.int64, device="cuda")
    _lib.call("tmb_stream_u64_block", int(stream_seed) & (2**64 - 1),
              int(start) & (2**64 - 1), count, ptr(out), stream_ptr())
    return out[:count].cpu().numpy().view(np.uint64) >> np.uint64(11)


def sample_updates(decision: UpdateDecision, n_clauses: int,
                   rng: RngStream) -> tuple[np.ndarray, np.ndarray]:
    """feedback.py:47-53: n_clauses target draws, then n_clauses negative
    draws; flag = u < p (compared exactly as integers: m < ceil(p * 2^53))."""
    import math
    m = _device_u53(rng.stream_seed, rng.counter, 2 * n_clauses)
    rng.counter += 2 * n_clauses
    t_t = np.uint64(min(math.ceil(decision.p_target * 2.0 ** 53), 2 ** 53))
    t_n = np.uint64(min(math.ceil(decision.p_negative * 2.0 ** 53), 2 ** 53))
    return m[:n_clauses] < t_t, m[n_clauses:] < t_n
