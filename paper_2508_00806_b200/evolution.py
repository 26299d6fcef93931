"""Adaptive policy evolution on the device (section 3.4; reference
evolve.py / simulate.py drift model).

The host trigger is the reference's: a TrackingSchedule with exponential
back-off (evolve.py:35-85: iterations 1, 2, 4, ..., max, then every max);
at a tracking iteration the tracked operators (linear / layer_norm / gelu,
evolve.py:30-32) are re-profiled -- here by counting the outlier channels of
the REAL activations on the device (the adc_detect_outliers kernel) instead of
reading a simulated trace (evolve.py:101-122) -- their compression rates are
updated, the plan is re-solved, and the fresh plan is adopted only if its
objective is strictly lower or the incumbent no longer fits (evolve.py:152-157).

``OutlierDrift`` reproduces the reference's synthetic shifting outlier
distribution (simulate.py:136-258: mean share decaying from 12% to 1% of the
channels with an AR(1) shock walk) and injects it into the model's residual
stream by scaling that many channels, so the drift is in the real tensors.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import codec as C
from .profiles import LayerKind, ModelProfile

TRACKED_KINDS = frozenset({LayerKind.LINEAR, LayerKind.LAYER_NORM, LayerKind.GELU})


@dataclass
class TrackingSchedule:
    """Powers of two up to max_interval, then every max_interval (evolve.py:35-85)."""

    max_interval: int = 512
    next_iteration: int = field(default=1, init=False)
    interval: int = field(default=1, init=False)
    last_seen: int = field(default=0, init=False)

    def __post_init__(self):
        m = self.max_interval
        if m < 1 or m & (m - 1):
            raise ValueError(f"max_interval must be a power of two, got {m}")

    def is_tracking(self, iteration: int) -> bool:
        if iteration <= self.last_seen:
            raise ValueError(f"iteration {iteration} observed after {self.last_seen}")
        self.last_seen = iteration
        while self.next_iteration < iteration:
            self._advance()
        if iteration != self.next_iteration:
            return False
        self._advance()
        return True

    def _advance(self):
        self.next_iteration += self.interval
        self.interval = min(self.interval * 2, self.max_interval)


@dataclass(frozen=True)
class OutlierDrift:
    """k(it) outlier channels (simulate.py:204-258 process), injected into x."""

    cols: int
    iterations: int
    seed: int = 0
    start_fraction: float = 0.12
    end_fraction: float = 0.01
    settle_iterations: int = 150
    amplitude: float = 6.0
    mean_reversion: float = 0.85
    factor: float = 30.0

    def counts(self) -> np.ndarray:
        steps = np.arange(1, self.iterations + 1, dtype=np.float64)
        mean = self.cols * (self.end_fraction + (self.start_fraction - self.end_fraction)
                            * np.exp(-(steps - 1) / self.settle_iterations))
        rng = np.random.default_rng([self.seed, 1])
        shocks = rng.standard_normal(self.iterations) * (self.amplitude / np.sqrt(steps))
        walk = np.empty(self.iterations)
        level = 0.0
        for i in range(self.iterations):
            level = self.mean_reversion * level + shocks[i]
            walk[i] = level
        return np.clip(np.rint(mean + walk), 0, self.cols // 2).astype(np.int64)

    def channels(self, device) -> torch.Tensor:
        g = torch.Generator(device="cpu")
        g.manual_seed(self.seed + 17)
        return torch.randperm(self.cols, generator=g).to(device)


def update_profile(profile: ModelProfile, measured: dict, k_margin: float = 2.0):
    """Re-measured compression rates of the tracked operators (evolve.py:101-122).

    ``measured``: op_id -> (k, cols, rows) from the device.  The rate is the
    reference size formula (codec.py:133-153) at the outlier capacity the hooks
    will reserve (2k + 8), so memory accounting matches what is held.
    Returns (profile, k_caps).
    """
    ops = []
    k_caps = {}
    for op in profile.operators:
        if op.id in measured and op.kind in TRACKED_KINDS:
            k, cols, rows = measured[op.id]
            cap = int(k * k_margin) + 8
            k_caps[op.id] = cap
            pay = C.packed_payload_bytes(C.Scheme.OUTLIER_SEPARATED, rows, cols, 128, min(cap, cols))
            ops.append(replace(op, compression_rate=min(1.0, pay / (2 * rows * cols))))
        else:
            ops.append(op)
    return replace(profile, operators=tuple(ops)), k_caps


def collect(pol) -> dict:
    """Read the tracking-iteration outlier counts (one synchronisation)."""
    per_op: dict[int, list] = {}
    for (op_id, _), (status, cols, rows) in pol.measured.items():
        per_op.setdefault(op_id, []).append((int(status[1].item()), cols, rows))
    return {op: (max(v[0] for v in vals), vals[0][1], vals[0][2]) for op, vals in per_op.items()}
