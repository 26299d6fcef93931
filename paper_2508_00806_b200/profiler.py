"""GPU profiler: measured B200 costs -> the reference's OperatorProfile JSON.

Replaces the reference's CPU wall-clock ``measure_codec`` (codec.py:410-429)
and its hand-written profiles.  For one transformer block of
the real model on the real device it measures, per operator:
  mem_bytes          bytes of the activation autograd saves (distinct storages);
  compute_time_ms    single-hop recompute time: the operator's forward from
                     its inputs (CUDA events, median) -- SPEC.md:93;
  compress_time_ms / decompress_time_ms
                     the B200 codec on that very tensor (CUDA events, median);
  compression_rate   device bytes held when compressed / mem_bytes (payload of
                     codec.py:133-145 plus any outlier-capacity slack).
and emits a ``ModelProfile`` in the reference schema (profiles.py:37-55), so
either the reference's ``planner.solve`` or ``policy.solve`` plans from it.
"""

from __future__ import annotations

import statistics

import torch

from . import codec as C
from .hooks import RETAIN, ActivationPolicy
from .profiles import ModelProfile, OperatorProfile
from .slots import CodecSlot


class _Recorder(ActivationPolicy):
    """Retain-everything policy that records block 0's activations and recipes."""

    def __init__(self, ops, layer_of_interest: int = 0):
        super().__init__(ops, plan={})
        self.block = -1
        self.want = layer_of_interest
        self.recipes: dict[int, tuple] = {}
        self.saved: dict[int, dict] = {}   # op -> {storage ptr: base tensor}

    def tag(self, op_id, out, fn=None, inputs=()):
        if op_id == 1:
            self.block += 1
        if self.block == self.want and fn is not None:
            self.recipes[op_id] = (fn, tuple(inputs))  # strong refs: profiling pass only
        return super().tag(op_id, out, fn, inputs)

    def pack(self, t):
        if self.block == self.want and t.is_cuda and t.numel() >= self.min_numel and not (
                isinstance(t, torch.nn.Parameter) or (t.requires_grad and t.is_leaf)):
            base = t if t._base is None else t._base
            key = base.untyped_storage().data_ptr()
            tagged = self._lookup(key)
            op_id = tagged[0] if tagged else self._current
            if op_id is not None:
                self.saved.setdefault(op_id, {})[key] = base
        return t


_FLUSH: torch.Tensor | None = None


def _time(fn, reps: int) -> float:
    """Median device time of one ``fn()``: L2 flushed before each rep, and a
    device-side sleep queued ahead of the start event so the host has
    submitted ``fn``'s kernels before the GPU reaches them -- the measured
    interval is kernel time, not host launch latency (which a training step,
    where the host runs ahead of the device, never sees)."""
    global _FLUSH
    if _FLUSH is None:
        _FLUSH = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # 2x L2
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        _FLUSH.zero_()
        torch.cuda._sleep(1_000_000)  # ~0.5 ms of device time for the host to enqueue fn
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def profile_model(model, ops, batch_fn, *, mem_budget_bytes: int, static_mem_bytes: int,
                  base_step_time_ms: float, reference_batch: int, reps: int = 5,
                  k_margin: float = 2.0) -> tuple[ModelProfile, dict]:
    """Profile block 0 of ``model`` on one batch.  Returns (profile, k_caps)."""
    rec = _Recorder(ops)
    idx, tgt = batch_fn()
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    loss = model(idx, tgt, rec)
    loss.backward()  # peak of a retain-all step (activations + LM head + transients)
    torch.cuda.synchronize()
    step_peak = torch.cuda.max_memory_allocated() - before
    model.zero_grad(set_to_none=True)
    ops_out = []
    k_caps = {}
    by_id = {o.op_id: o for o in ops}
    for op_id in sorted(by_id):
        info = by_id[op_id]
        bases = list(rec.saved.get(op_id, {}).values())
        mem = sum(b.numel() * b.element_size() for b in bases)
        if mem == 0:
            mem = 1  # schema requires > 0; an operator autograd does not save costs nothing
        # recompute cost: the operator's own forward from its inputs
        if op_id in rec.recipes and op_id != 1:
            fn, inputs = rec.recipes[op_id]
            with torch.no_grad():
                compute_ms = _time(lambda: fn(*inputs), reps)
        else:
            compute_ms = 0.0
        # codec cost on the real tensors
        spec = C.scheme_for(info.kind)
        c_ms = d_ms = 0.0
        held = 0
        for b in bases:
            x = b.reshape(-1, b.shape[-1])
            if spec.scheme is C.Scheme.BIT_MASK:
                if b.dtype not in (torch.bool, torch.uint8):
                    held += mem
                    continue
            elif b.dtype not in (torch.bfloat16, torch.float16, torch.float32):
                held += b.numel() * b.element_size()
                continue
            k_cap = None
            if spec.scheme is C.Scheme.OUTLIER_SEPARATED:
                k = C.compress(x, spec).outlier_count if x.shape[1] > 1 else 0
                k_cap = max(32, int(k * k_margin) + 8)
                k_caps[op_id] = max(k_caps.get(op_id, 0), k_cap)
            slot = CodecSlot(x.shape[0], x.shape[1], spec, x.dtype, x.dtype if x.dtype != torch.bool else torch.uint8,
                             k_cap=k_cap, device=x.device)
            out = torch.empty((x.shape[0], x.shape[1]), dtype=slot.out_dtype, device=x.device)
            xs = x.contiguous()
            c_ms += _time(lambda: slot.compress(xs), reps)
            d_ms += _time(lambda: slot.decompress(out), reps)
            held += slot.codes.numel() + sum(t.numel() * t.element_size() for t in
                                             (slot.scales, slot.offsets, slot.idx, slot.val) if t is not None)
        rate = min(1.0, max(held, 1) / mem) if bases else 1.0
        ops_out.append(OperatorProfile(op_id, info.name, info.kind, int(mem), float(compute_ms),
                                       float(c_ms), float(d_ms), float(rate)))
    del loss
    torch.cuda.synchronize()
    # The planner charges n_layers * per-block activation bytes against
    # budget - static (planner.py:98-104, 131-142).  Everything else a step
    # holds at its peak (LM head logits, loss, transient workspaces) is folded
    # into static so that the plan's budget is the real HBM cap.
    act = model.cfg.n_layer * sum(op.mem_bytes for op in ops_out)
    static = int(static_mem_bytes) + max(0, int(step_peak) - act)
    budget = max(int(mem_budget_bytes), static + 1)
    prof = ModelProfile(tuple(ops_out), model.cfg.n_layer, static, budget,
                        int(reference_batch), float(base_step_time_ms))
    global _FLUSH
    _FLUSH = None  # the 256 MB L2-flush buffer is only needed while profiling
    return prof, k_caps
