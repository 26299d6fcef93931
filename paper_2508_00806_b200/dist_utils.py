"""Cross-rank plumbing of the data-parallel path (one process per GPU).

The codec itself is rank-local (no data-path collective).
What does cross ranks:
  * timing: every reported time is the MAX over ranks (device-timed), and a
    whole-job rate is (units of all ranks) / that max;
  * the Adacc plan: the planner runs on rank-local device profiles, whose
    timings differ slightly per GPU; rank 0's plan is broadcast so every rank
    stores / compresses / recomputes the same operators (the reference's
    planner is deterministic for one profile, planner.py:16-19);
  * gradients: DDP's bucketed all-reduce (NCCL on GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def _active() -> bool:
    return dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1


def world_size() -> int:
    return dist.get_world_size() if _active() else 1


def max_over_ranks(value: float, device=None) -> float:
    """MAX of a per-rank scalar (a device time) over all ranks."""
    if not _active():
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_rate(units_per_rank: float, ms_local: float, device=None) -> tuple[float, float]:
    """(units of all ranks per second, max-over-ranks milliseconds)."""
    ms = max_over_ranks(ms_local, device)
    return world_size() * units_per_rank / (ms / 1e3), ms


def broadcast_plan(plan: dict, src: int = 0) -> dict:
    """Rank ``src``'s plan on every rank (op id -> action)."""
    if not _active():
        return plan
    box = [plan if dist.get_rank() == src else None]
    dist.broadcast_object_list(box, src=src)
    return box[0]


def plans_agree(plan: dict) -> bool:
    """True when every rank holds the same plan."""
    if not _active():
        return True
    items = [None] * dist.get_world_size()
    dist.all_gather_object(items, sorted(plan.items()))
    return all(i == items[0] for i in items)
