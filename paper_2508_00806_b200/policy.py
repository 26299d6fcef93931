"""Host-side policy maker: the exact retain / compress / recompute plan.

Restates the reference planner's model (/root/reference/pkg/src/actplan/planner.py)
for the host side of the B200 training loop, which runs where the reference
package is not installed:
  * cost of a choice: recompute -> compute_time_ms, compress ->
    compress_time_ms + decompress_time_ms, retain -> 0 (planner.py:75-80);
  * memory: recompute -> 0, compress -> ceil(mem_bytes * compression_rate),
    retain -> mem_bytes (planner.py:70-72, 83-88); activation memory is
    n_layers * per-block sum and must fit mem_budget - static (planner.py:98-104, 131-142);
  * the first operator (block input) is the checkpoint and cannot be
    recomputed (planner.py:1-9, 227);
  * ties: lowest objective, then lowest activation memory, then the
    lexicographically smallest choice vector with recompute < compress <
    retain (planner.py:16-19).
Block sizes here are <= 12 operators, so exhaustive vectorised enumeration is
exact and fast (3^11 = 177k assignments in ~10 ms).  The JSON profiles the
GPU profiler writes are the reference schema, so the reference's own ``solve``
accepts them too (tests/test_policy.py checks both agree).
"""

from __future__ import annotations

import itertools
import math
from dataclasses import dataclass

import numpy as np

from .errors import ValidationError
from .profiles import ModelProfile

RECOMPUTE, COMPRESS, RETAIN = 0, 1, 2
NAMES = {RECOMPUTE: "recompute", COMPRESS: "compress", RETAIN: "retain"}


class InfeasibleError(ValidationError):
    """No assignment fits the memory budget (errors.py:41-50)."""


@dataclass(frozen=True)
class Plan:
    choices: tuple
    objective_ms: float
    activation_bytes: int
    total_bytes: int

    def by_op(self, op_ids) -> dict:
        return {i: NAMES[c] for i, c in zip(op_ids, self.choices)}


def _tables(profile: ModelProfile):
    cost = np.array([[op.compute_time_ms, op.compress_time_ms + op.decompress_time_ms, 0.0]
                     for op in profile.operators])
    mem = np.array([[0, math.ceil(op.mem_bytes * op.compression_rate), op.mem_bytes]
                    for op in profile.operators], dtype=np.int64)
    return cost, mem


def evaluate(profile: ModelProfile, choices) -> Plan:
    cost, mem = _tables(profile)
    idx = np.arange(len(choices))
    c = np.asarray(choices)
    obj = float(sum(cost[i, c[i]] for i in idx))  # sequential sum, like block_cost
    act = int(profile.n_layers * mem[idx, c].sum())
    return Plan(tuple(int(v) for v in c), obj, act, profile.static_mem_bytes + act)


def solve(profile: ModelProfile) -> Plan:
    n = profile.n_operators
    if n > 12:
        raise ValidationError("exhaustive planner supports at most 12 operators per block")
    cost, mem = _tables(profile)
    room = (profile.mem_budget_bytes - profile.static_mem_bytes) // profile.n_layers
    grid = np.array(list(itertools.product((RECOMPUTE, COMPRESS, RETAIN), repeat=n)), dtype=np.int8)
    grid = grid[grid[:, 0] != RECOMPUTE]  # the checkpoint cannot be recomputed
    cols = np.arange(n)
    m = mem[cols, grid].sum(axis=1)
    ok = m <= room
    if not ok.any():
        floor = profile.static_mem_bytes + profile.n_layers * int(min(mem[0, 1], mem[0, 2]))
        raise InfeasibleError(
            f"no assignment fits: minimal achievable total is {floor} bytes, "
            f"budget is {profile.mem_budget_bytes} bytes")
    g = grid[ok]
    m = m[ok]
    # objective summed left to right in float64 (block_cost order)
    obj = np.zeros(len(g))
    for i in range(n):
        obj = obj + cost[i, g[:, i]]
    best = np.lexsort(tuple(g[:, i] for i in reversed(range(n))) + (m, obj))[0]
    return evaluate(profile, g[best])


def fixed_strategy(profile: ModelProfile, name: str) -> tuple:
    """retain-all / full-recompute / all-compress assignments (simulate.py strategy_choices)."""
    n = profile.n_operators
    if name == "retain-all":
        return (RETAIN,) * n
    if name == "all-compress":
        return (COMPRESS,) * n
    if name == "full-recompute":
        return (RETAIN,) + (RECOMPUTE,) * (n - 1)
    raise ValidationError(f"unknown strategy {name}")
