"""Adacc-policy GPT training on B200 (BASELINE configs[1] and [3]).

    python -m paper_2508_00806_b200.train --model gpt-345m --batch 8 --steps 20 \
        --policy adacc --mem-cap-gb 40
    torchrun --nproc-per-node 8 -m paper_2508_00806_b200.train --model gpt-1.3b ...

Flow (Fig. 5): profile one block on the device (profiler.py) ->
plan with the exact planner under the HBM cap (policy.py; the reference's
``planner.solve`` accepts the same JSON) -> train with the plan applied by
saved-tensor hooks (hooks.py).  Data parallel over NCCL: the codec is
rank-local and the only collective is DDP's bucketed gradient all-reduce.
Synthetic learnable corpus (seeded Markov stream; no network for datasets).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import time

import torch
import torch.distributed as dist

from . import policy as P
from .dist_utils import broadcast_plan
from .gpt import BLOCK_OPS, GPT, GPTConfig, synthetic_batch
from .hooks import COMPRESS, RECOMPUTE, RETAIN, ActivationPolicy
from .profiler import profile_model
from .profiles import save_profile

STRATEGIES = ("retain-all", "full-recompute", "all-compress", "adacc")


def model_flops_per_token(cfg: GPTConfig, n_params: int) -> float:
    """Training FLOPs per token: 6 x parameters (forward + backward of every
    weight) + 12 x layers x seq x d_model for the attention score / context
    matmuls (forward 4 L s d, backward twice that).  Recomputation is not
    counted (it is overhead, not model work)."""
    return 6.0 * n_params + 12.0 * cfg.n_layer * cfg.seq * cfg.d_model


def peak_bf16_flops() -> tuple[float, str]:
    """Dense bf16 peak the MFU is quoted against: MEASURED_PEAKS.json's sustained
    cuBLAS figure when present, else the 2.25 PFLOP/s spec."""
    from pathlib import Path
    p = Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["bf16_tflops_sustained"]) * 1e12, "measured sustained cuBLAS bf16"
    except Exception:
        return 2.25e15, "B200 dense bf16 spec"


def codec_share(tr, batch) -> dict:
    """One profiled step: device time of the codec kernels (adc::) / all kernels."""
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        tr.step(*batch)
        torch.cuda.synchronize()
    tot = codec = 0.0
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            us = e.device_time if hasattr(e, "device_time") else e.cuda_time
            tot += us
            if "adc::" in e.name:
                codec += us
    return {"codec_kernel_us": round(codec, 1), "all_kernel_us": round(tot, 1),
            "share": round(codec / tot, 4) if tot else 0.0}


def plan_for(strategy: str, prof=None) -> dict:
    ids = [o.op_id for o in BLOCK_OPS]
    if strategy == "adacc":
        return P.solve(prof).by_op(ids)
    names = {P.RETAIN: RETAIN, P.COMPRESS: COMPRESS, P.RECOMPUTE: RECOMPUTE}
    n = len(ids)
    if strategy == "retain-all":
        ch = (P.RETAIN,) * n
    elif strategy == "all-compress":
        ch = (P.COMPRESS,) * n
    else:
        ch = (P.RETAIN,) + (P.RECOMPUTE,) * (n - 1)
    return {i: names[c] for i, c in zip(ids, ch)}


class Trainer:
    def __init__(self, cfg: GPTConfig, batch: int, *, lr: float = 3e-4, rank: int = 0,
                 world: int = 1, device=None, ddp: bool = False, lr_warmup: int = 0):
        self.cfg, self.batch, self.rank, self.world = cfg, batch, rank, world
        self.lr, self.lr_warmup = lr, int(lr_warmup)
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        torch.manual_seed(1234)
        model = GPT(cfg).to(self.device, dtype=torch.bfloat16)
        self.model = model
        self.net = model
        if ddp:
            from torch.nn.parallel import DistributedDataParallel as DDP
            on_gpu = self.device.type == "cuda"
            self.net = DDP(model, device_ids=[self.device.index] if on_gpu else None,
                           gradient_as_bucket_view=True, bucket_cap_mb=64)
        self.opt = torch.optim.AdamW(model.parameters(), lr=lr, betas=(0.9, 0.95), weight_decay=0.1,
                                     fused=self.device.type == "cuda")
        self.pol = ActivationPolicy(BLOCK_OPS)
        self.step_id = 0

    def batch_at(self, step):
        return synthetic_batch(step, self.rank, self.batch, self.cfg.seq, self.cfg.vocab, self.device)

    def _forward(self, idx, tgt, pol):
        # DDP wraps the module; our forward takes the policy as an argument
        return self.net(idx, tgt, pol, self.step_id)

    def step(self, idx, tgt) -> torch.Tensor:
        loss = self._forward(idx, tgt, self.pol)
        loss.backward()
        if self.lr_warmup:  # linear warm-up over the first lr_warmup steps of a run
            lr = self.lr * min(1.0, (self.step_id + 1) / self.lr_warmup)
            for g in self.opt.param_groups:
                g["lr"] = lr
        self.opt.step()
        self.opt.zero_grad(set_to_none=True)
        self.step_id += 1
        return loss.detach()

    def static_bytes(self) -> int:
        return torch.cuda.memory_allocated(self.device)

    def profile(self, mem_budget_bytes: int, base_step_ms: float):
        idx, tgt = self.batch_at(10**6)
        prof, k_caps = profile_model(self.model, BLOCK_OPS, lambda: (idx, tgt),
                                     mem_budget_bytes=mem_budget_bytes,
                                     static_mem_bytes=self.static_after_step,
                                     base_step_time_ms=base_step_ms, reference_batch=self.batch)
        return prof, k_caps


def _clone_state(sd):
    if isinstance(sd, dict):
        return {k: _clone_state(v) for k, v in sd.items()}
    if isinstance(sd, list):
        return [_clone_state(v) for v in sd]
    if isinstance(sd, torch.Tensor):
        return sd.detach().clone()
    return sd


def _calibrate(tr, prof, cap, snap_model, snap_opt, dev, world, rounds: int = 6):
    """Feed the measured peak back into the planner's budget.

    The reference cost model charges only n_layers x per-block activation
    bytes; transient memory of the chosen mix (a decompressed or recomputed
    tensor alive during its layer's backward) is not in it.  Solve, run two
    steps, and if the measured peak exceeds the cap shrink the budget by the
    overshoot and re-solve (at most ``rounds`` times; MAX over ranks)."""
    from dataclasses import replace
    budget = prof.mem_budget_bytes
    log = []
    plan = None
    for _ in range(rounds):
        p = replace(prof, mem_budget_bytes=max(budget, prof.static_mem_bytes + 1))
        try:
            plan = P.solve(p).by_op([o.op_id for o in BLOCK_OPS])
        except P.InfeasibleError:
            plan = plan_for("full-recompute")
        plan = broadcast_plan(plan)  # rank-local profiles differ slightly: rank 0 decides
        tr.pol.plan = plan
        tr.model.load_state_dict(snap_model)
        tr.opt.load_state_dict(_clone_state(snap_opt))
        torch.cuda.empty_cache()
        torch.cuda.reset_peak_memory_stats(dev)
        for s in range(2):
            tr.step(*tr.batch_at(500 + s))
        torch.cuda.synchronize()
        peak = torch.tensor([torch.cuda.max_memory_allocated(dev)], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(peak, op=dist.ReduceOp.MAX)
        peak = int(peak.item())
        same = bool(log) and log[-1]["plan"] == plan
        log.append({"budget_bytes": int(budget), "peak_bytes": peak, "plan": plan})
        if peak <= cap:
            break
        # shrink by the overshoot; if the last cut did not change the plan,
        # cut geometrically harder so the next solve has to move
        step = (peak - cap) + (64 << 20)
        if same:
            step = max(step, 2 * (log[-2]["budget_bytes"] - budget))
        budget -= step
    return plan, log


def _overrides(kinds: str) -> dict:
    """--int8-kinds softmax,score -> {LayerKind.SOFTMAX: "int8", ...} (EXTENSION codec)."""
    from .profiles import LayerKind
    return {LayerKind(k.strip()): "int8" for k in (kinds or "").split(",") if k.strip()}


def run(args) -> dict:
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=dev)
    cfg = GPTConfig.named(args.model)
    cfg.seq = args.seq or cfg.seq
    tr = Trainer(cfg, args.batch, rank=rank, world=world, device=dev, ddp=world > 1,
                 lr_warmup=getattr(args, "lr_warmup", 0))
    tr.pol.codec_overrides = _overrides(getattr(args, "int8_kinds", ""))
    if getattr(args, "codec_stream", False):
        tr.pol.codec_stream = torch.cuda.Stream(dev)
    total_hbm = torch.cuda.get_device_properties(dev).total_memory
    cap = int(args.mem_cap_gb * (1 << 30)) if args.mem_cap_gb else total_hbm
    # warm-up with retain-all to size static memory and the base step time
    tr.pol.plan = plan_for("retain-all")
    for s in range(2):
        tr.step(*tr.batch_at(s))
    torch.cuda.synchronize()
    tr.static_after_step = torch.cuda.memory_allocated(dev)
    t0 = time.perf_counter()
    tr.step(*tr.batch_at(2))
    torch.cuda.synchronize()
    base_ms = (time.perf_counter() - t0) * 1e3
    out = {"model": args.model, "params": tr.model.n_params(), "batch_per_gpu": args.batch,
           "seq": cfg.seq, "n_gpus": world, "mem_cap_bytes": cap, "lr": tr.lr, "lr_warmup": tr.lr_warmup,
           "int8_kinds": sorted(k.value for k in tr.pol.codec_overrides),
           "codec_stream": tr.pol.codec_stream is not None, "results": {}}
    prof = None
    if "adacc" in args.policy or args.profile_out:
        prof, k_caps = tr.profile(cap, base_ms)
        tr.pol.k_caps = k_caps
        if args.profile_out and rank == 0:
            save_profile(prof, args.profile_out)
        out["profile"] = prof.to_dict()
    losses_all = {}
    # every strategy starts from the same weights / optimizer state and sees
    # the same batches, so losses are comparable (retain vs recompute: equal)
    snap_model = {k: v.detach().clone() for k, v in tr.model.state_dict().items()}
    snap_opt = _clone_state(tr.opt.state_dict())
    for strategy in args.policy.split(","):
        plan = broadcast_plan(plan_for(strategy, prof))
        calib = []
        if strategy == "adacc" and cap < total_hbm:
            plan, calib = _calibrate(tr, prof, cap, snap_model, snap_opt, dev, world)
        tr.pol.plan = plan
        tr.model.load_state_dict(snap_model)
        tr.opt.load_state_dict(_clone_state(snap_opt))
        tr.step_id = 0
        torch.cuda.empty_cache()
        torch.cuda.reset_peak_memory_stats(dev)
        for s in range(args.warmup):
            tr.step(*tr.batch_at(100 + s))
        batches = [tr.batch_at(1000 + s) for s in range(args.steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        losses = []
        for idx, tgt in batches:
            losses.append(tr.step(idx, tgt))
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        tokens = args.batch * cfg.seq * world * args.steps
        err = tr.pol.check()
        peak = torch.cuda.max_memory_allocated(dev)
        lv = [float(l.item()) for l in losses]
        win = max(1, min(50, len(lv) // 10))
        tps = tokens / (ms / 1e3)
        peak_flops, peak_src = peak_bf16_flops()
        mfu = tps * model_flops_per_token(cfg, tr.model.n_params()) / (world * peak_flops)
        share = codec_share(tr, tr.batch_at(999)) if getattr(args, "codec_share", False) else None
        out["results"][strategy] = {
            "plan": plan, "tokens_per_s": tps, "ms_per_step": ms / args.steps,
            "peak_bytes": peak, "fits_cap": peak <= cap, "final_loss": lv[-1],
            "smoothed_final_loss": statistics.mean(lv[-win:]), "loss_window": win,
            "mean_loss": statistics.mean(lv), "mfu": round(mfu, 4), "mfu_peak": peak_src,
            "codec_share": share, "device_error_word": err,
            "compressed_tensors": tr.pol.stats.compressed, "recomputed_tensors": tr.pol.stats.recomputed,
            "calibration": calib,
        }
        if getattr(args, "loss_curve", False):
            out["results"][strategy]["losses"] = [round(v, 5) for v in lv[:: max(1, len(lv) // 100)]]
        losses_all[strategy] = lv
    return out


def evolve(args) -> dict:
    """Config 5: policy evolution under a shifting outlier distribution.

    Two arms from the same weights: STATIC keeps the plan solved at iteration
    1; ADAPTIVE re-profiles the tracked operators on the device at the
    TrackingSchedule's iterations, re-solves and swaps plans by the reference
    rule (evolve.py:125-166).  Both see the same drift and batches."""
    from dataclasses import replace
    from .evolution import TRACKED_KINDS, OutlierDrift, TrackingSchedule, collect, update_profile
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=dev)
    cfg = GPTConfig.named(args.model)
    cfg.seq = args.seq or cfg.seq
    tr = Trainer(cfg, args.batch, rank=rank, world=world, device=dev, ddp=world > 1)
    cap = int(args.mem_cap_gb * (1 << 30))
    n = args.evolve
    drift = OutlierDrift(cols=cfg.d_model, iterations=n, settle_iterations=max(1, args.settle))
    counts = drift.counts()
    chans = drift.channels(dev)

    def set_drift(it):
        scale = torch.ones(cfg.d_model, device=dev, dtype=torch.bfloat16)
        scale[chans[: int(counts[it - 1])]] = drift.factor
        tr.model.channel_scale = scale

    tr.pol.plan = plan_for("retain-all")
    set_drift(1)
    for s in range(2):
        tr.step(*tr.batch_at(s))
    torch.cuda.synchronize()
    tr.static_after_step = torch.cuda.memory_allocated(dev)
    t0 = time.perf_counter()
    tr.step(*tr.batch_at(2))
    torch.cuda.synchronize()
    base_ms = (time.perf_counter() - t0) * 1e3
    prof0, k_caps0 = tr.profile(cap, base_ms)
    snap_model = {k: v.detach().clone() for k, v in tr.model.state_dict().items()}
    snap_opt = _clone_state(tr.opt.state_dict())
    ids = [o.op_id for o in BLOCK_OPS]
    out = {"model": args.model, "iterations": n, "mem_cap_bytes": cap, "max_interval": args.max_interval,
           "drift_counts": [int(c) for c in counts[:: max(1, n // 32)]], "profile": prof0.to_dict(), "arms": {}}
    for arm in ("static", "adaptive"):
        tr.model.load_state_dict(snap_model)
        tr.opt.load_state_dict(_clone_state(snap_opt))
        tr.step_id = 0
        prof = prof0
        plan = P.solve(prof)
        tr.pol.plan = plan.by_op(ids)
        tr.pol.k_caps = dict(k_caps0)
        sched = TrackingSchedule(args.max_interval)
        log = []
        ms_total = 0.0
        torch.cuda.synchronize()
        for it in range(1, n + 1):
            set_drift(it)
            tracked = arm == "adaptive" and sched.is_tracking(it)
            tr.pol.measure_kinds = TRACKED_KINDS if tracked else frozenset()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            tr.step(*tr.batch_at(5000 + it))
            b.record()
            if tracked:
                measured = collect(tr.pol)  # the one synchronisation of a tracking iteration
                new_prof, caps = update_profile(prof0, measured)
                fresh = P.solve(new_prof)
                incumbent = P.evaluate(new_prof, plan.choices)
                forced = incumbent.total_bytes > new_prof.mem_budget_bytes
                adopt = forced or fresh.objective_ms < plan.objective_ms
                log.append({"iteration": it, "k": {str(k): v[0] for k, v in measured.items()},
                            "objective_old": plan.objective_ms, "objective_new": fresh.objective_ms,
                            "forced": forced, "changed": adopt})
                tr.pol.k_caps.update(caps)
                if adopt:
                    plan = fresh
                    tr.pol.plan = plan.by_op(ids)
                prof = new_prof
            b.synchronize()
            ms_total += a.elapsed_time(b)
        tokens = args.batch * cfg.seq * world * n
        t = torch.tensor([ms_total], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out["arms"][arm] = {"tokens_per_s": tokens / (float(t.item()) / 1e3), "final_plan": plan.by_op(ids),
                            "replans": sum(1 for e in log if e["changed"]), "tracking": log,
                            "device_error_word": tr.pol.check()}
    out["improvement_ratio"] = out["arms"]["adaptive"]["tokens_per_s"] / out["arms"]["static"]["tokens_per_s"]
    return out


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="gpt-345m")
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--seq", type=int, default=0)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--policy", default="retain-all,adacc")
    ap.add_argument("--mem-cap-gb", type=float, default=0.0)
    ap.add_argument("--profile-out", default="")
    ap.add_argument("--codec-share", action="store_true", help="profile one step: codec kernels' share of device time")
    ap.add_argument("--loss-curve", action="store_true", help="include a subsampled loss curve per strategy")
    ap.add_argument("--lr-warmup", type=int, default=0, help="linear learning-rate warm-up steps")
    ap.add_argument("--int8-kinds", default="",
                    help="layer kinds compressed with the int8 / f32-scale EXTENSION codec (e.g. softmax)")
    ap.add_argument("--codec-stream", action="store_true",
                    help="compress on a side stream overlapping the forward (decompress waits on its event)")
    ap.add_argument("--evolve", type=int, default=0, help="config 5: N iterations of policy evolution")
    ap.add_argument("--max-interval", type=int, default=64)
    ap.add_argument("--settle", type=int, default=150)
    args = ap.parse_args(argv)
    out = evolve(args) if args.evolve else run(args)
    if int(os.environ.get("RANK", "0")) == 0:
        print(json.dumps(out))
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
