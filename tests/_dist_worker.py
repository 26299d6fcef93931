"""Body of the world_size-2 gloo tests (tests/test_dist_gloo.py), one process per rank on CPU."""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def run(rank: int, world: int, port: int, out_dir: str) -> None:
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch
    import torch.distributed as dist
    torch.set_num_threads(1)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_00806_b200 import dist_utils as D
    res = {}
    # bench / train timing: MAX over ranks, whole-job rate = all units / max time
    res["max"] = D.max_over_ranks(10.0 * (rank + 1))
    res["rate"], res["rate_ms"] = D.whole_job_rate(1000.0, 10.0 * (rank + 1))
    # the planner runs on rank-local profiles: rank 0's plan wins everywhere
    mine = {1: "retain", 2: "compress" if rank == 0 else "recompute", 3: "retain"}
    res["agree_before"] = D.plans_agree(mine)
    plan = D.broadcast_plan(mine)
    res["plan"] = sorted(plan.items())
    res["agree_after"] = D.plans_agree(plan)
    # DDP over the gradient all-reduce: different batches per rank, identical
    # weights after every step; the Adacc hooks stay inert on CPU tensors
    from paper_2508_00806_b200.gpt import GPTConfig
    from paper_2508_00806_b200.train import Trainer, plan_for
    tr = Trainer(GPTConfig.named("gpt-tiny"), 2, rank=rank, world=world, device=torch.device("cpu"),
                 ddp=True)
    tr.pol.plan = D.broadcast_plan(plan_for("all-compress"))
    losses = [float(tr.step(*tr.batch_at(s))) for s in range(2)]
    flat = torch.cat([p.detach().float().reshape(-1) for p in tr.model.parameters()])
    sums = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(sums, torch.tensor([flat.sum().item(), flat.abs().sum().item()], dtype=torch.float64))
    res["param_sums"] = [s.tolist() for s in sums]
    res["losses"] = losses
    first = tr.batch_at(7)[0].float().sum()
    others = [torch.zeros(()) for _ in range(world)]
    dist.all_gather(others, first)
    res["batches_per_rank"] = [float(o) for o in others]
    dist.destroy_process_group()
    Path(out_dir, f"rank{rank}.json").write_text(json.dumps(res))


if __name__ == "__main__":
    run(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4])
