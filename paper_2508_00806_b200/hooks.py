"""Saved-tensor hooks that apply an Adacc plan (section 3, planner.py:43-46):
each operator's saved activations are RETAINED, COMPRESSED after the forward
op and decompressed before its backward, or RECOMPUTED in the backward from
the operator's inputs.

``ActivationPolicy`` installs ``torch.autograd.graph.saved_tensors_hooks``.
Which operator a saved tensor belongs to is decided by its storage: the model
``tag``s the storages of the tensors each operator produces, together with a
recompute recipe (the operator's forward function and its input tensors); a
tensor saved while an operator is running that carries no tag (softmax saving
its own output) belongs to that operator.

* compress: the tensor's contiguous base is compressed once with the codec
  ``scheme_for(kind)`` names (codec.py:72-82) through the C-ABI, into a
  pooled :class:`~.slots.CodecSlot` (payload, side buffer, workspace and the
  outlier prediction allocated once per (operator, occurrence, shape) and
  reused every step: no allocation, no workspace fill, no synchronisation);
  every view of it (transposes, strided parts) is restored with
  ``as_strided`` from one shared decompression.  The model saves the fused
  QKV output ``[b, s, 3h]`` (gpt.py ``_QKScores`` / ``_Context``), so it is
  compressed per channel over its 3h columns like the reference's
  ``[tokens, 3h]`` QKV matrix.
* recompute: the pack hook stores the recipe with its inputs packed under
  their own operators' policies (so a recomputed tensor costs no memory and
  its inputs may themselves be compressed); the unpack hook re-runs the
  operator under ``no_grad`` -- single-hop recomputation from the previous
  checkpoint.  The first operator (the block input) is the
  checkpoint and is never recomputed (planner.py:1-9).
* retain: the tensor is kept.

Training mode never synchronises: outlier side buffers are sized from the
tracked outlier count (``k_caps``); errors accumulate in one device status
word read by ``check()``.  A tensor whose outlier count exceeds its capacity
keeps the first ``k_cap`` outliers exact and quantises the rest with their
groups (graceful, as the reference's fallback to symmetric).
"""

from __future__ import annotations

import contextlib
import weakref
from dataclasses import dataclass

import torch

from . import codec as C
from .profiles import LayerKind
from .slots import CodecSlot, Int8Slot

RETAIN, COMPRESS, RECOMPUTE = "retain", "compress", "recompute"


@dataclass
class OpInfo:
    op_id: int
    name: str
    kind: LayerKind


class _Base:
    """One packed base storage (compressed or recompute recipe), shared by views."""

    __slots__ = ("kind", "slot", "recipe", "shape", "dtype", "value", "src", "ready", "__weakref__")

    def __init__(self, kind, slot, recipe, shape, dtype, src, ready=None):
        self.kind, self.slot, self.recipe, self.shape, self.dtype = kind, slot, recipe, shape, dtype
        self.value = None
        self.src = src  # weakref to the packed base tensor: detects address reuse
        self.ready = ready  # event after the compress when it ran on the codec stream


@dataclass
class Stats:
    saved: int = 0
    compressed: int = 0
    recomputed: int = 0
    original_bytes: int = 0
    stored_bytes: int = 0


class ActivationPolicy:
    def __init__(self, ops: list[OpInfo], plan: dict[int, str] | None = None,
                 min_numel: int = 1 << 15, k_caps: dict[int, int] | None = None,
                 codec_overrides: dict[LayerKind, str] | None = None):
        self.ops = {o.op_id: o for o in ops}
        # kinds compressed with the int8 / float32-scale EXTENSION codec ("int8")
        # instead of the reference's scheme_for(kind) (not reference behaviour)
        self.codec_overrides = dict(codec_overrides or {})
        # optional side stream for the forward's compress calls: they start
        # when their activation is produced and overlap the next forward ops;
        # the backward's decompress waits for the compress's event
        self.codec_stream: torch.cuda.Stream | None = None
        self.plan = dict(plan or {})
        self.min_numel = min_numel
        self.k_caps = dict(k_caps or {})
        self.stats = Stats()
        self._tags: dict[int, tuple] = {}   # storage ptr -> (op_id, recipe)
        self._current: int | None = None
        self._enabled = True
        # storage ptr -> entry; weak: autograd's packed tuples are the only owners,
        # so a decompressed / recomputed value dies with its last saved tensor
        self._bases: weakref.WeakValueDictionary = weakref.WeakValueDictionary()
        self._pool: dict[tuple, CodecSlot] = {}   # (signature, occurrence) -> slot, reused every step
        self._occ: dict[tuple, int] = {}          # occurrences of a signature in this step
        self.status: torch.Tensor | None = None
        self.records: dict[int, list] = {}  # op_id -> compressed records of the last step (profiling)
        self.measure_kinds: frozenset = frozenset()   # tracking iterations: kinds to count outliers of
        self.measured: dict[int, list] = {}          # op_id -> [device [err, k], cols, rows]

    # -- model-facing -------------------------------------------------------
    def tag(self, op_id: int, out: torch.Tensor, fn=None, inputs=()):
        """Register ``out`` as operator ``op_id``'s activation, recomputable as fn(*inputs).

        Only weak references are kept (a tag must never keep a compressed or
        recomputed activation alive); a tag whose tensor has died is stale --
        its address may have been reused by the caching allocator.
        """
        recipe = None
        if fn is not None:
            recipe = (fn, tuple(weakref.ref(i) if isinstance(i, torch.Tensor) else i for i in inputs))
        self._tags[out.untyped_storage().data_ptr()] = (op_id, recipe, weakref.ref(out))
        return out

    def _lookup(self, key):
        hit = self._tags.get(key)
        if hit is None:
            return None
        if hit[2]() is None:  # stale: the tagged tensor is gone, the address was reused
            del self._tags[key]
            return None
        return hit

    @contextlib.contextmanager
    def op(self, op_id: int):
        prev = self._current
        self._current = op_id
        try:
            yield
        finally:
            self._current = prev

    @contextlib.contextmanager
    def paused(self):
        prev = self._enabled
        self._enabled = False
        try:
            yield
        finally:
            self._enabled = prev

    @contextlib.contextmanager
    def hooks(self):
        self._tags.clear()
        self._bases.clear()
        self._occ.clear()
        self.records = {}
        self.measured = {}
        if self.status is None and torch.cuda.is_available():
            # shared error word of this policy's codec calls (CPU runs -- the
            # gloo tests -- never compress: pack() keeps non-CUDA tensors)
            self.status = torch.zeros(2, dtype=torch.int32, device="cuda")
        with torch.autograd.graph.saved_tensors_hooks(self.pack, self.unpack):
            yield

    # -- hooks --------------------------------------------------------------
    def _choice(self, op_id):
        return self.plan.get(op_id, RETAIN)

    def pack(self, t: torch.Tensor):
        if (not self._enabled or not t.is_cuda or t.numel() < self.min_numel
                or isinstance(t, torch.nn.Parameter) or (t.requires_grad and t.is_leaf)):
            return t
        base = t if t._base is None else t._base
        key = base.untyped_storage().data_ptr()
        tagged = self._lookup(key)
        op_id, recipe = (tagged[0], tagged[1]) if tagged else (self._current, None)
        if op_id is None:
            return t
        if (self.measure_kinds and self.ops[op_id].kind in self.measure_kinds and base.is_contiguous()
                and base.dtype in (torch.bfloat16, torch.float16, torch.float32)):
            key_m = (op_id, key)
            if key_m not in self.measured:  # tracking iteration: device outlier count, no sync
                x = base.reshape(-1, base.shape[-1])
                self.measured[key_m] = [C.count_outliers_async(x), x.shape[1], x.shape[0]]
        choice = self._choice(op_id)
        if choice == RECOMPUTE and (recipe is None or op_id == 1):
            choice = RETAIN
        if choice == RETAIN:
            return t
        if not base.is_contiguous():
            return t
        self.stats.saved += 1
        entry = self._bases.get(key)
        if entry is not None and entry.src() is None:
            entry = None  # a dead base whose address was reused
        if entry is None:
            entry = self._make_entry(op_id, choice, base, recipe)
            if entry is None:
                return t
            self._bases[key] = entry
        if t is base or (t.shape == base.shape and t.stride() == base.stride()
                         and t.storage_offset() == base.storage_offset()):
            return (entry, None)
        return (entry, (tuple(t.shape), tuple(t.stride()), t.storage_offset() - base.storage_offset()))

    def _make_entry(self, op_id, choice, base, recipe):
        nbytes = base.numel() * base.element_size()
        if choice == RECOMPUTE:
            fn, inputs = recipe
            live = [i() if isinstance(i, weakref.ref) else i for i in inputs]
            if any(isinstance(i, weakref.ref) and v is None for i, v in zip(inputs, live)):
                return None  # an input is gone: cannot recompute, keep the tensor
            with self.op(None):
                packed_inputs = tuple(self.pack(i) if isinstance(i, torch.Tensor) else i for i in live)
            self.stats.recomputed += 1
            self.stats.original_bytes += nbytes
            return _Base(RECOMPUTE, None, (fn, packed_inputs), tuple(base.shape), base.dtype,
                         weakref.ref(base))
        kind = self.ops[op_id].kind
        if self.codec_overrides.get(kind) == "int8" and base.dtype in (torch.bfloat16, torch.float16, torch.float32):
            x = base.reshape(-1, base.shape[-1])
            slot = self._slot_int8(op_id, x)
            ready = self._launch_compress(slot, x)
            self.stats.compressed += 1
            self.stats.original_bytes += nbytes
            self.stats.stored_bytes += slot.device_bytes
            return _Base(COMPRESS, slot, None, tuple(base.shape), base.dtype, weakref.ref(base), ready)
        spec = C.scheme_for(kind)
        if spec.scheme is C.Scheme.BIT_MASK:
            if base.dtype not in (torch.bool, torch.uint8):
                return None
        elif base.dtype not in (torch.bfloat16, torch.float16, torch.float32):
            return None
        x = base.reshape(-1, base.shape[-1])
        k_cap = None
        if spec.scheme is C.Scheme.OUTLIER_SEPARATED:
            k_cap = self.k_caps.get(op_id, max(16, x.shape[1] // 32))
        slot = self._slot(op_id, spec, x, k_cap)
        ready = self._launch_compress(slot, x)
        self.stats.compressed += 1
        self.stats.original_bytes += nbytes
        self.stats.stored_bytes += slot.device_bytes
        self.records.setdefault(op_id, []).append(slot)
        return _Base(COMPRESS, slot, None, tuple(base.shape), base.dtype, weakref.ref(base), ready)

    def _launch_compress(self, slot, x):
        """Compress on the current stream, or on the codec stream after the
        producer (x is kept alive for that stream); returns the event the
        backward's decompress waits for (None on the current stream)."""
        cur = torch.cuda.current_stream(x.device)
        cs = self.codec_stream
        if cs is None:
            slot.compress_ptr(x.data_ptr(), cur.cuda_stream)
            return None
        cs.wait_stream(cur)
        slot.compress_ptr(x.data_ptr(), cs.cuda_stream)
        x.record_stream(cs)
        ev = torch.cuda.Event()
        ev.record(cs)
        return ev

    def _slot(self, op_id, spec, x, k_cap) -> CodecSlot:
        """The pooled slot of this (operator, shape, dtype, capacity)'s n-th
        occurrence in the step (one per layer), created on first use."""
        sig = (op_id, spec, tuple(x.shape), x.dtype, k_cap)
        n = self._occ.get(sig, 0)
        self._occ[sig] = n + 1
        slot = self._pool.get((sig, n))
        if slot is None:
            in_dt = torch.uint8 if x.dtype == torch.bool else x.dtype
            out_dt = torch.uint8 if spec.scheme is C.Scheme.BIT_MASK else x.dtype
            slot = CodecSlot(x.shape[0], x.shape[1], spec, in_dt, out_dt, k_cap=k_cap, device=x.device,
                             status=self.status)
            self._pool[(sig, n)] = slot
        return slot

    def _slot_int8(self, op_id, x) -> Int8Slot:
        sig = (op_id, "int8", tuple(x.shape), x.dtype)
        n = self._occ.get(sig, 0)
        self._occ[sig] = n + 1
        slot = self._pool.get((sig, n))
        if slot is None:
            slot = Int8Slot(x.shape[0], x.shape[1], 128, x.dtype, x.dtype, device=x.device, status=self.status)
            self._pool[(sig, n)] = slot
        return slot

    def _materialize(self, entry: _Base) -> torch.Tensor:
        if entry.value is not None:
            return entry.value
        if entry.kind == RECOMPUTE:
            fn, packed_inputs = entry.recipe
            inputs = [self.unpack(p) if isinstance(p, tuple) and p and isinstance(p[0], _Base) else p
                      for p in packed_inputs]
            with torch.no_grad(), self.paused():
                out = fn(*inputs)
            value = out.reshape(entry.shape)
        else:
            slot = entry.slot
            out = torch.empty((slot.rows, slot.cols), dtype=slot.out_dtype, device=slot.device)
            if entry.ready is not None:
                torch.cuda.current_stream(out.device).wait_event(entry.ready)
            slot.decompress_ptr(out.data_ptr(), torch.cuda.current_stream(out.device).cuda_stream)
            if entry.dtype == torch.bool:
                out = out.view(torch.bool)
            value = out.reshape(entry.shape)
        entry.value = value
        return value

    def unpack(self, packed):
        if isinstance(packed, torch.Tensor):
            return packed
        entry, view = packed
        full = self._materialize(entry)
        if view is None:
            return full
        size, stride, off = view
        return full.as_strided(size, stride, full.storage_offset() + off)

    def check(self) -> int:
        """Device error word accumulated since the last check (synchronises)."""
        if self.status is None:
            return 0
        if self.codec_stream is not None:
            self.codec_stream.synchronize()
        err = int(self.status[0].item()) & 0xffffffff
        self.status.zero_()
        return err
