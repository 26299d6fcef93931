"""Host planner (policy.py) against the reference planner and brute force."""

import itertools
import math
import random

import pytest

from paper_2508_00806_b200 import policy as P
from paper_2508_00806_b200.profiles import LayerKind, ModelProfile, OperatorProfile


def random_profile(seed, n_ops=6):
    rng = random.Random(seed)
    kinds = list(LayerKind)
    ops = []
    for i in range(n_ops):
        mem = rng.choice([1, 2, 4, 8, 16, 32]) * (1 << 20)
        ops.append(OperatorProfile(i + 1, f"op{i + 1}", rng.choice(kinds), mem,
                                   rng.choice([0.125, 0.25, 0.5, 1.0, 2.0]),
                                   rng.choice([0.0625, 0.125, 0.25]), rng.choice([0.0625, 0.125]),
                                   rng.choice([0.125, 0.25, 0.27, 0.5])))
    n_layers = rng.choice([2, 4, 12])
    static = 1 << 30
    full = n_layers * sum(o.mem_bytes for o in ops)
    budget = static + int(full * rng.uniform(0.15, 1.1)) + 1
    return ModelProfile(tuple(ops), n_layers, static, budget, 4, 100.0)


def brute(profile):
    best = None
    for ch in itertools.product((0, 1, 2), repeat=profile.n_operators):
        if ch[0] == 0:
            continue
        plan = P.evaluate(profile, ch)
        if plan.total_bytes > profile.mem_budget_bytes:
            continue
        key = (plan.objective_ms, plan.activation_bytes, ch)
        if best is None or key < best[0]:
            best = (key, plan)
    return best[1] if best else None


@pytest.mark.parametrize("seed", range(60))
def test_solve_matches_brute_force(seed):
    prof = random_profile(seed, n_ops=5 + seed % 4)
    want = brute(prof)
    if want is None:
        with pytest.raises(P.InfeasibleError):
            P.solve(prof)
        return
    got = P.solve(prof)
    assert got.choices == want.choices
    assert got.objective_ms == want.objective_ms


@pytest.mark.parametrize("seed", range(40))
def test_solve_matches_reference_planner(seed, reference_codec):
    """Same assignment as the reference's branch-and-bound solve (planner.py:174)."""
    from actplan import planner as RP
    from actplan import profiles as RPR
    prof = random_profile(1000 + seed, n_ops=6 + seed % 5)
    ref = RPR.profile_from_dict(prof.to_dict())
    try:
        want = RP.solve(ref)
    except Exception as exc:  # InfeasibleError
        assert type(exc).__name__ == "InfeasibleError"
        with pytest.raises(P.InfeasibleError):
            P.solve(prof)
        return
    got = P.solve(prof)
    assert got.choices == tuple(int(c) for c in want.choices)
    assert got.objective_ms == want.objective_ms
    assert got.activation_bytes == want.activation_bytes


def test_fixed_strategies():
    prof = random_profile(3, 6)
    assert P.fixed_strategy(prof, "full-recompute")[0] == P.RETAIN
    assert set(P.fixed_strategy(prof, "full-recompute")[1:]) == {P.RECOMPUTE}
    assert P.fixed_strategy(prof, "all-compress") == (P.COMPRESS,) * 6


def test_profile_json_schema_roundtrip(tmp_path, reference_codec):
    """Profiles written here load with the reference's own schema checks (profiles.py:226)."""
    from actplan import profiles as RPR
    from paper_2508_00806_b200.profiles import save_profile
    prof = random_profile(7, 9)
    path = tmp_path / "p.json"
    save_profile(prof, path)
    ref = RPR.load_profile(path)
    assert ref.n_operators == 9 and ref.mem_budget_bytes == prof.mem_budget_bytes
