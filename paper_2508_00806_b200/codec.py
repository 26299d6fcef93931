"""Device codec API -- the reference ``actplan.codec`` interface on B200.

Same names, argument meaning and error behaviour as
/root/reference/pkg/src/actplan/codec.py, but every array lives in HBM and
every byte of compute runs in the sm_100a kernels behind the C-ABI
(include/adacc.h, bound in ``_lib``).  There is no CPU fallback.

Differences a caller of the reference will notice:
  * arrays are ``torch`` tensors on the current CUDA device (numpy / lists are
    accepted as inputs and uploaded);
  * ``decompress`` returns a device tensor (float32 by default, bit-identical
    to the reference's float32 result; ``out_dtype=torch.bfloat16/float16``
    rounds that float32 value for training);
  * ``CompressedTensor.scales`` / ``offsets`` are float16 device tensors (the
    reference keeps the same float16 values in a float32 container).

The synchronous functions here ("parity mode") read the device error word and
outlier count back and raise the reference exception types.  Training code
uses :func:`compress_async` / :func:`decompress_into`, which never synchronise.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np
import torch

from . import _lib
from .errors import (CorruptPayloadError, NonBinaryMaskError, OutlierCapacityError,
                     ValidationError, raise_for_error_word)
from .profiles import LayerKind

MAGIC = b"ADC1"
DEFAULT_GROUP_SIZE = 128          # codec.py:42
DEFAULT_Z_THRESHOLD = 3.0         # codec.py:43
PER_CHANNEL = 0                   # codec.py:45
_HEADER = struct.Struct("<4sBIIIII")   # codec.py:52
SERIALIZED_HEADER_BYTES = _HEADER.size  # 25


class Scheme(IntEnum):
    """codec.py:56-60; values are the ADC1 scheme byte and the C-ABI ids."""

    SYMMETRIC_GROUP = 0
    ASYMMETRIC_GROUP = 1
    OUTLIER_SEPARATED = 2
    BIT_MASK = 3


@dataclass(frozen=True)
class SchemeSpec:
    """codec.py:63-69."""

    scheme: Scheme
    group_size: int = DEFAULT_GROUP_SIZE
    z_threshold: float = DEFAULT_Z_THRESHOLD


def scheme_for(kind: LayerKind) -> SchemeSpec:
    """Layer kind -> compressor (codec.py:72-82)."""
    kind = LayerKind(kind)
    if kind in (LayerKind.LINEAR, LayerKind.LAYER_NORM, LayerKind.GELU):
        return SchemeSpec(Scheme.OUTLIER_SEPARATED, DEFAULT_GROUP_SIZE, DEFAULT_Z_THRESHOLD)
    if kind is LayerKind.QKV_MATRIX:
        return SchemeSpec(Scheme.SYMMETRIC_GROUP, PER_CHANNEL)
    if kind in (LayerKind.SOFTMAX, LayerKind.SCORE):
        return SchemeSpec(Scheme.ASYMMETRIC_GROUP, DEFAULT_GROUP_SIZE)
    if kind is LayerKind.DROPOUT_MASK:
        return SchemeSpec(Scheme.BIT_MASK, 0)
    return SchemeSpec(Scheme.SYMMETRIC_GROUP, DEFAULT_GROUP_SIZE)


# ---------------------------------------------------------------------------
# sizes (codec.py:133-153), through the C-ABI
# ---------------------------------------------------------------------------
def _layout(scheme: int, rows: int, cols: int, group_size: int, k: int = 0):
    groups, code_bytes, total = (_lib.C.c_int64(), _lib.C.c_int64(), _lib.C.c_int64())
    st = _lib.lib().adc_payload_bytes(int(scheme), rows, cols, group_size, k,
                                      _lib.C.byref(groups), _lib.C.byref(code_bytes),
                                      _lib.C.byref(total))
    _lib.check(st, "payload_bytes")
    return groups.value, code_bytes.value, total.value


def packed_payload_bytes(scheme: Scheme, rows: int, cols: int, group_size: int,
                         outlier_count: int = 0) -> int:
    """Closed-form payload size in bytes (codec.py:133-145)."""
    return _layout(int(scheme), rows, cols, group_size, outlier_count)[2]


def outlier_separated_rate(rows: int, cols: int, outlier_count: int,
                           group_size: int = DEFAULT_GROUP_SIZE) -> float:
    """compressed/original implied by an outlier count (codec.py:148-153)."""
    return packed_payload_bytes(Scheme.OUTLIER_SEPARATED, rows, cols, group_size,
                                outlier_count) / (2 * rows * cols)


# ---------------------------------------------------------------------------
# the compressed record
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class CompressedTensor:
    """Device mirror of codec.py:85-130.

    ``packed_codes`` / ``mask_bits`` are uint8 device tensors in the reference
    byte layout; ``scales`` / ``offsets`` float16; ``outlier_indices`` int64
    (ascending); ``outlier_values`` float16 shaped (k, rows).
    """

    scheme: Scheme
    rows: int
    cols: int
    group_size: int
    scales: torch.Tensor | None
    offsets: torch.Tensor | None
    packed_codes: torch.Tensor | None
    outlier_indices: torch.Tensor | None = None
    outlier_values: torch.Tensor | None = None
    mask_bits: torch.Tensor | None = None
    # training-mode extras (not part of the reference record)
    k_dev: torch.Tensor | None = field(default=None, repr=False, compare=False)
    k_cap: int = field(default=0, repr=False, compare=False)
    shape: tuple | None = field(default=None, repr=False, compare=False)
    dtype: torch.dtype | None = field(default=None, repr=False, compare=False)

    @property
    def group_count(self) -> int:
        return 0 if self.scales is None else int(self.scales.numel())

    @property
    def outlier_count(self) -> int:
        return 0 if self.outlier_indices is None else int(self.outlier_indices.numel())

    @property
    def original_bytes(self) -> int:
        return self.rows * self.cols * (1 if self.scheme is Scheme.BIT_MASK else 2)

    @property
    def compressed_size_bytes(self) -> int:
        return packed_payload_bytes(self.scheme, self.rows, self.cols, self.group_size,
                                    self.outlier_count)

    @property
    def compression_ratio(self) -> float:
        return self.original_bytes / self.compressed_size_bytes

    @property
    def device_bytes(self) -> int:
        """HBM actually held by this record (includes any unused outlier capacity)."""
        return sum(t.numel() * t.element_size() for t in
                   (self.scales, self.offsets, self.packed_codes, self.outlier_indices,
                    self.outlier_values, self.mask_bits) if t is not None)

    def to_bytes(self) -> bytes:
        return serialize(self)


# ---------------------------------------------------------------------------
# input handling (codec.py:156-176)
# ---------------------------------------------------------------------------
_DT = {torch.float32: _lib.F32, torch.bfloat16: _lib.BF16, torch.float16: _lib.F16}


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise _lib.LibraryMissingError("a CUDA device is required: the codec has no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


def _as_device_matrix(x, *, allow_nd: bool = False) -> torch.Tensor:
    """Upload / view ``x`` as a C-contiguous (rows, cols) float matrix."""
    if isinstance(x, torch.Tensor):
        t = x
    else:
        try:
            arr = np.asarray(x)
            if arr.dtype == object or arr.dtype.kind not in "biuf":
                arr = np.asarray(x, dtype=np.float64)
        except (TypeError, ValueError) as exc:
            raise ValidationError(f"activation matrix must be numeric: {exc}") from exc
        t = torch.from_numpy(np.ascontiguousarray(arr))
    if t.dim() == 1:
        t = t.reshape(1, -1)
    if t.dim() != 2:
        if not allow_nd or t.dim() == 0:
            raise ValidationError(f"activation matrix must be 1-D or 2-D, got shape {tuple(t.shape)}")
        t = t.reshape(-1, t.shape[-1])
    if t.numel() == 0:
        raise ValidationError("activation matrix must have at least one element")
    dev = _device()
    if t.dtype not in _DT:
        # float64 / integer inputs: numpy's cast, as the reference's
        # np.asarray(x, dtype=float16) (codec.py:158) -- ONE RNE rounding to
        # float16.  torch's float64 -> float16 goes through float32 and rounds
        # twice (1 + 2^-11 + 2^-40 -> 1.0 instead of 1 + 2^-10).
        t = torch.from_numpy(np.ascontiguousarray(t.detach().cpu().numpy().astype(np.float16)))
    return t.to(dev, non_blocking=True).contiguous()


def _check_group_size(group_size: int) -> None:
    if group_size != PER_CHANNEL and group_size < 1:
        raise ValidationError(f"group_size must be positive or PER_CHANNEL, got {group_size}")


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


# ---------------------------------------------------------------------------
# compress (asynchronous core)
# ---------------------------------------------------------------------------
def compress_async(x: torch.Tensor, spec: SchemeSpec, *, k_cap: int | None = None,
                   status: torch.Tensor | None = None) -> CompressedTensor:
    """Launch one compression on the current stream and return at once.

    ``x`` is a CUDA tensor whose last dim is the channel dim (any rank).
    ``status`` is an int32 device tensor of 2 elements: [error word, k]; the
    error word is OR-ed, never cleared, so one status can cover many calls.
    Outlier buffers are sized for ``k_cap`` channels (default cols // 2, the
    reference's hard limit, so overflow is impossible).
    """
    scheme = Scheme(spec.scheme)
    shape, dtype = tuple(x.shape), x.dtype
    if scheme is Scheme.BIT_MASK:
        m = x.reshape(-1) if x.dim() != 2 else x
        rows, cols = (x.shape[0], x.shape[1]) if x.dim() == 2 else (1, x.numel())
        if m.dtype == torch.bool:
            m = m.view(torch.uint8)
        dt = _lib.U8 if m.dtype == torch.uint8 else _DT.get(m.dtype)
        if dt is None:
            m = m.to(torch.float32)
            dt = _lib.F32
        m = m.contiguous()
        bits = torch.empty((rows * cols + 7) // 8, dtype=torch.uint8, device=m.device)
        if status is None:
            status = torch.zeros(2, dtype=torch.int32, device=m.device)
        st = _lib.lib().adc_compress(int(scheme), m.data_ptr(), dt, rows, cols, 0, 0.0, 0,
                                     bits.data_ptr(), None, None, None, None, None,
                                     status.data_ptr(), None, 0, _stream())
        _lib.check(st, "compress")
        return CompressedTensor(scheme, rows, cols, 0, None, None, None, mask_bits=bits,
                                shape=shape, dtype=dtype, k_dev=status)
    _check_group_size(spec.group_size)
    if x.dim() != 2:
        x = x.reshape(-1, x.shape[-1])
    x = x.contiguous()
    if x.dtype not in _DT:
        raise ValidationError(f"unsupported activation dtype {x.dtype}")
    rows, cols = x.shape
    dev = x.device
    n_groups, code_bytes, _ = _layout(int(scheme), rows, cols, spec.group_size)
    codes = torch.empty(code_bytes, dtype=torch.uint8, device=dev)
    scales = torch.empty(n_groups, dtype=torch.float16, device=dev)
    offsets = (torch.empty(n_groups, dtype=torch.float16, device=dev)
               if scheme is Scheme.ASYMMETRIC_GROUP else None)
    shared = status is not None
    if status is None:
        status = torch.zeros(2, dtype=torch.int32, device=dev)
    idx = val = None
    kc = 0
    kbuf = status
    if scheme is Scheme.OUTLIER_SEPARATED:
        # k is per tensor (the decompress scatter reads it); only the error
        # word may be shared between calls
        if shared:
            kbuf = torch.zeros(2, dtype=torch.int32, device=dev)
        kc = cols // 2 if k_cap is None else int(k_cap)
        idx = torch.empty(max(kc, 1), dtype=torch.int32, device=dev)
        val = torch.empty((max(kc, 1), rows), dtype=torch.float16, device=dev)
    ws = None
    ws_bytes = 0
    if scheme is Scheme.OUTLIER_SEPARATED or spec.group_size == PER_CHANNEL:
        ws_bytes = _lib.lib().adc_workspace_bytes(int(scheme), rows, cols, spec.group_size)
        ws = torch.zeros(ws_bytes, dtype=torch.uint8, device=dev)
    st = _lib.lib().adc_compress(
        int(scheme), x.data_ptr(), _DT[x.dtype], rows, cols, spec.group_size,
        float(spec.z_threshold), kc, codes.data_ptr(), scales.data_ptr(), _ptr(offsets),
        _ptr(idx), _ptr(val), kbuf.data_ptr() + 4 if idx is not None else None,
        status.data_ptr(), _ptr(ws), ws_bytes, _stream())
    _lib.check(st, "compress")
    return CompressedTensor(scheme, rows, cols, spec.group_size, scales, offsets, codes,
                            outlier_indices=idx, outlier_values=val, k_dev=kbuf, k_cap=kc,
                            shape=shape, dtype=dtype)


def _finalize(ct: CompressedTensor) -> CompressedTensor:
    """Parity mode (private status = [error word, k]): synchronise, raise
    reference errors, trim outliers to k."""
    err, k = (int(v) for v in ct.k_dev.cpu().tolist())
    err &= 0xffffffff
    raise_for_error_word(err, rows=ct.rows, cols=ct.cols, k=k)
    if ct.scheme is not Scheme.OUTLIER_SEPARATED:
        return ct
    idx = ct.outlier_indices[:k].to(torch.int64)
    val = ct.outlier_values[:k].clone()
    return CompressedTensor(ct.scheme, ct.rows, ct.cols, ct.group_size, ct.scales, None,
                            ct.packed_codes, outlier_indices=idx, outlier_values=val,
                            k_dev=ct.k_dev, k_cap=ct.k_cap, shape=ct.shape, dtype=ct.dtype)


# ---------------------------------------------------------------------------
# public reference-shaped API
# ---------------------------------------------------------------------------
def quantize_symmetric(x, group_size: int = DEFAULT_GROUP_SIZE) -> CompressedTensor:
    """codec.py:245-252."""
    _check_group_size(group_size)
    return _finalize(compress_async(_as_device_matrix(x), SchemeSpec(Scheme.SYMMETRIC_GROUP, group_size)))


def quantize_asymmetric(x, group_size: int = DEFAULT_GROUP_SIZE) -> CompressedTensor:
    """codec.py:255-258."""
    _check_group_size(group_size)
    return _finalize(compress_async(_as_device_matrix(x), SchemeSpec(Scheme.ASYMMETRIC_GROUP, group_size)))


def compress_outlier_separated(x, group_size: int = DEFAULT_GROUP_SIZE,
                               threshold: float = DEFAULT_Z_THRESHOLD) -> CompressedTensor:
    """codec.py:308-341."""
    _check_group_size(group_size)
    return _finalize(compress_async(_as_device_matrix(x),
                                    SchemeSpec(Scheme.OUTLIER_SEPARATED, group_size, threshold)))


def _as_device_mask(mask) -> torch.Tensor:
    if isinstance(mask, (bytes, bytearray)):
        mask = np.frombuffer(bytes(mask), dtype=np.uint8)
    t = mask if isinstance(mask, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(mask)))
    if t.numel() == 0:
        raise ValidationError("mask must have at least one element")
    if t.dim() > 2:
        raise ValidationError(f"mask must be 1-D or 2-D, got shape {tuple(t.shape)}")
    if t.dtype not in (torch.bool, torch.uint8, torch.float32, torch.float16, torch.bfloat16):
        t = t.to(torch.float64)
        if not bool(((t == 0) | (t == 1)).all()):
            raise NonBinaryMaskError("mask bytes must be 0 or 1")
        t = t.to(torch.uint8)
    return t.to(_device()).contiguous()


def pack_bitmask(mask) -> CompressedTensor:
    """codec.py:344-369."""
    t = _as_device_mask(mask)
    return _finalize(compress_async(t, SchemeSpec(Scheme.BIT_MASK, 0)))


def unpack_bitmask(ct: CompressedTensor) -> torch.Tensor:
    """codec.py:372-378: uint8 0/1 tensor shaped (rows, cols)."""
    if ct.scheme is not Scheme.BIT_MASK:
        raise ValidationError(f"expected a bit mask, got {ct.scheme.name}")
    out = torch.empty((ct.rows, ct.cols), dtype=torch.uint8, device=ct.mask_bits.device)
    st = _lib.lib().adc_decompress(int(ct.scheme), ct.mask_bits.data_ptr(), None, None, None,
                                   None, None, 0, ct.rows, ct.cols, 0, out.data_ptr(), _lib.U8,
                                   _stream())
    _lib.check(st, "unpack_bitmask")
    return out


_OUT = {torch.float32: _lib.F32, torch.bfloat16: _lib.BF16, torch.float16: _lib.F16}


def decompress_into(ct: CompressedTensor, out: torch.Tensor) -> torch.Tensor:
    """Asynchronous decompression into a preallocated (rows, cols) tensor."""
    if ct.scheme is Scheme.BIT_MASK:
        dt = _lib.U8
        if out.dtype == torch.bool:
            out = out.view(torch.uint8)
        if out.dtype != torch.uint8:
            raise ValidationError("bit masks decompress to uint8/bool")
        st = _lib.lib().adc_decompress(int(ct.scheme), ct.mask_bits.data_ptr(), None, None, None,
                                       None, None, 0, ct.rows, ct.cols, 0, out.data_ptr(), dt,
                                       _stream())
        _lib.check(st, "decompress")
        return out
    if out.dtype not in _OUT:
        raise ValidationError(f"unsupported output dtype {out.dtype}")
    k_cap = 0
    k_ptr = None
    if ct.scheme is Scheme.OUTLIER_SEPARATED and ct.outlier_indices is not None:
        k_cap = ct.outlier_indices.numel() if ct.k_cap == 0 else ct.k_cap
        k_ptr = ct.k_dev.data_ptr() + 4
        if ct.outlier_indices.dtype != torch.int32:  # finalized record: k is exact
            k_cap = ct.outlier_count
    idx = ct.outlier_indices
    if idx is not None and idx.dtype != torch.int32:
        idx = idx.to(torch.int32)
    if k_cap and k_ptr is None:
        raise ValidationError("outlier record without a device count")
    st = _lib.lib().adc_decompress(
        int(ct.scheme), ct.packed_codes.data_ptr(), ct.scales.data_ptr(), _ptr(ct.offsets),
        _ptr(idx), _ptr(ct.outlier_values), k_ptr, k_cap, ct.rows, ct.cols, ct.group_size,
        out.data_ptr(), _OUT[out.dtype], _stream())
    _lib.check(st, "decompress")
    return out


def dequantize(ct: CompressedTensor, out_dtype: torch.dtype = torch.float32) -> torch.Tensor:
    """codec.py:261-286: (rows, cols) tensor; float32 is bit-identical to the reference."""
    if ct.scheme is Scheme.BIT_MASK:
        raise ValidationError("bit masks are restored with unpack_bitmask")
    dev = ct.packed_codes.device
    out = torch.empty((ct.rows, ct.cols), dtype=out_dtype, device=dev)
    if ct.scheme is Scheme.OUTLIER_SEPARATED and ct.outlier_indices is not None \
            and ct.outlier_indices.dtype != torch.int32:
        # finalized record: provide an exact device count for the scatter kernel
        k = ct.outlier_count
        status = torch.tensor([0, k], dtype=torch.int32, device=dev)
        ct = CompressedTensor(ct.scheme, ct.rows, ct.cols, ct.group_size, ct.scales, None,
                              ct.packed_codes, ct.outlier_indices.to(torch.int32),
                              ct.outlier_values.contiguous(), k_dev=status, k_cap=k)
    return decompress_into(ct, out)


def decompress(ct: CompressedTensor, out_dtype: torch.dtype = torch.float32) -> torch.Tensor:
    """codec.py:392-395."""
    if ct.scheme is Scheme.BIT_MASK:
        return unpack_bitmask(ct)
    return dequantize(ct, out_dtype)


def compress(x, spec: SchemeSpec) -> CompressedTensor:
    """codec.py:381-389 (``x`` is a mask for BIT_MASK)."""
    scheme = Scheme(spec.scheme)
    if scheme is Scheme.SYMMETRIC_GROUP:
        return quantize_symmetric(x, spec.group_size)
    if scheme is Scheme.ASYMMETRIC_GROUP:
        return quantize_asymmetric(x, spec.group_size)
    if scheme is Scheme.OUTLIER_SEPARATED:
        return compress_outlier_separated(x, spec.group_size, spec.z_threshold)
    return pack_bitmask(x)


# ---------------------------------------------------------------------------
# outlier detection (codec.py:289-305)
# ---------------------------------------------------------------------------
def channel_abs_sums(x) -> torch.Tensor:
    """float64 column sums of |f16(x)| (codec.py:289-291)."""
    t = _as_device_matrix(x)
    rows, cols = t.shape
    ws_bytes = _lib.lib().adc_workspace_bytes(int(Scheme.OUTLIER_SEPARATED), rows, cols, 0)
    ws = torch.zeros(ws_bytes, dtype=torch.uint8, device=t.device)
    sums = torch.empty(cols, dtype=torch.float64, device=t.device)
    status = torch.zeros(2, dtype=torch.int32, device=t.device)
    st = _lib.lib().adc_channel_abs_sums(t.data_ptr(), _DT[t.dtype], rows, cols, sums.data_ptr(),
                                         status.data_ptr(), ws.data_ptr(), ws_bytes, _stream())
    _lib.check(st, "channel_abs_sums")
    return sums


def detect_outlier_channels(x, threshold: float = DEFAULT_Z_THRESHOLD) -> torch.Tensor:
    """Ascending int64 indices of outlier channels (codec.py:294-305)."""
    t = _as_device_matrix(x)
    rows, cols = t.shape
    ws_bytes = _lib.lib().adc_workspace_bytes(int(Scheme.OUTLIER_SEPARATED), rows, cols, 0)
    ws = torch.zeros(ws_bytes, dtype=torch.uint8, device=t.device)
    idx = torch.empty(cols, dtype=torch.int32, device=t.device)
    status = torch.zeros(2, dtype=torch.int32, device=t.device)
    st = _lib.lib().adc_detect_outliers(t.data_ptr(), _DT[t.dtype], rows, cols, float(threshold),
                                        cols, idx.data_ptr(), status.data_ptr() + 4,
                                        status.data_ptr(), ws.data_ptr(), ws_bytes, _stream())
    _lib.check(st, "detect_outlier_channels")
    err, k = (int(v) for v in status.cpu().tolist())
    raise_for_error_word(err & 0xffffffff, rows=rows, cols=cols, k=k)
    return idx[:k].to(torch.int64)


def count_outliers_async(x: torch.Tensor, threshold: float = DEFAULT_Z_THRESHOLD) -> torch.Tensor:
    """Launch outlier detection on a (rows, cols) CUDA tensor without
    synchronising; returns the int32 device pair [error word, k].  Used at
    policy-evolution tracking iterations (section 3.4)."""
    rows, cols = x.shape
    ws_bytes = _lib.lib().adc_workspace_bytes(int(Scheme.OUTLIER_SEPARATED), rows, cols, 0)
    ws = torch.zeros(ws_bytes, dtype=torch.uint8, device=x.device)
    idx = torch.empty(1, dtype=torch.int32, device=x.device)
    status = torch.zeros(2, dtype=torch.int32, device=x.device)
    st = _lib.lib().adc_detect_outliers(x.data_ptr(), _DT[x.dtype], rows, cols, float(threshold), 0,
                                        idx.data_ptr(), status.data_ptr() + 4, status.data_ptr(),
                                        ws.data_ptr(), ws_bytes, _stream())
    _lib.check(st, "count_outliers")
    return status


# ---------------------------------------------------------------------------
# measurement (codec.py:398-429), CUDA events instead of perf_counter
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class CodecReport:
    scheme: Scheme
    compress_ms: float
    decompress_ms: float
    ratio: float
    original_bytes: int
    compressed_bytes: int


def measure_codec(x, spec: SchemeSpec, *, repeats: int = 5,
                  out_dtype: torch.dtype | None = None) -> CodecReport:
    """Device time of one compress / decompress cycle (median of ``repeats``).

    Timed with CUDA events on the launching stream around the asynchronous
    launch sequence; the ratio comes from the finalized (exact-k) record.
    """
    t = _as_device_mask(x) if Scheme(spec.scheme) is Scheme.BIT_MASK else _as_device_matrix(x, allow_nd=True)
    ct = _finalize(compress_async(t, spec))
    k_cap = max(ct.outlier_count, 1) if ct.scheme is Scheme.OUTLIER_SEPARATED else None
    if ct.scheme is Scheme.BIT_MASK:
        out = torch.empty((ct.rows, ct.cols), dtype=torch.uint8, device=t.device)
    else:
        out = torch.empty((ct.rows, ct.cols), dtype=out_dtype or t.dtype, device=t.device)
    c_ms, d_ms = [], []
    for _ in range(repeats + 1):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        work = compress_async(t, spec, k_cap=k_cap)
        e1.record()
        decompress_into(work, out)
        e2.record()
        e2.synchronize()
        c_ms.append(e0.elapsed_time(e1))
        d_ms.append(e1.elapsed_time(e2))
    c_ms, d_ms = sorted(c_ms[1:]), sorted(d_ms[1:])
    return CodecReport(ct.scheme, c_ms[len(c_ms) // 2], d_ms[len(d_ms) // 2], ct.compression_ratio,
                       ct.original_bytes, ct.compressed_size_bytes)


# ---------------------------------------------------------------------------
# ADC1 wire format (codec.py:432-546), host side
# ---------------------------------------------------------------------------
def _np(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def serialize(ct: CompressedTensor) -> bytes:
    """25-byte header, group metadata, codes, outliers (codec.py:432-459)."""
    header = _HEADER.pack(MAGIC, int(ct.scheme), ct.rows, ct.cols, ct.group_size,
                          ct.group_count, ct.outlier_count)
    if ct.scheme is Scheme.BIT_MASK:
        return header + _np(ct.mask_bits).tobytes()
    parts = [header]
    if ct.offsets is None:
        parts.append(_np(ct.scales).astype("<f2").tobytes())
    else:
        meta = np.stack([_np(ct.scales), _np(ct.offsets)], axis=1).astype("<f2")
        parts.append(meta.tobytes())
    parts.append(_np(ct.packed_codes).tobytes())
    if ct.outlier_count:
        parts.append(_np(ct.outlier_indices).astype("<u4").tobytes())
        parts.append(_np(ct.outlier_values).astype("<f2").tobytes())
    return b"".join(parts)


def serialize_device(ct: CompressedTensor) -> torch.Tensor:
    """ADC1 bytes (codec.py:432-459) assembled on the device (adc_serialize):
    a uint8 device tensor equal to ``serialize(ct)``."""
    rows, cols = ct.rows, ct.cols
    dev = (ct.mask_bits if ct.scheme is Scheme.BIT_MASK else ct.packed_codes).device
    idx = val = kd = None
    k_cap = 0
    if ct.scheme is Scheme.OUTLIER_SEPARATED and ct.outlier_count:
        if ct.outlier_indices.dtype == torch.int32 and ct.k_dev is not None:  # async record: (k_cap, rows)
            idx, val, kd, k_cap = ct.outlier_indices, ct.outlier_values, ct.k_dev, ct.k_cap
        else:  # parity record: trimmed to k
            idx = ct.outlier_indices.to(torch.int32).contiguous()
            val = ct.outlier_values.contiguous()
            k_cap = int(idx.numel())
            kd = torch.tensor([0, k_cap], dtype=torch.int32, device=dev)
    cap = _HEADER.size + packed_payload_bytes(ct.scheme, rows, cols, ct.group_size, k_cap)
    out = torch.empty((cap + 15) // 16 * 16, dtype=torch.uint8, device=dev)
    meta = torch.zeros(2, dtype=torch.int64, device=dev)  # [length, error word]
    codes = ct.mask_bits if ct.scheme is Scheme.BIT_MASK else ct.packed_codes
    st = _lib.lib().adc_serialize(int(ct.scheme), _ptr(ct.scales), _ptr(ct.offsets), codes.data_ptr(),
                                  _ptr(idx), _ptr(val), None if kd is None else kd.data_ptr() + 4, k_cap,
                                  rows, cols, ct.group_size, out.data_ptr(), out.numel(), meta.data_ptr(),
                                  meta.data_ptr() + 8, _stream())
    _lib.check(st, "serialize")
    length = int(meta[0].item())
    return out[:length]


def _header_error(v: int, buf_len: int, raw: bytes, h) -> CorruptPayloadError:
    """The reference's message for an adc_parse_header verdict (codec.py:464-493)."""
    if v == _lib.WIRE_TRUNCATED:
        return CorruptPayloadError(f"payload truncated: {buf_len} bytes is shorter than the header")
    if v == _lib.WIRE_BAD_MAGIC:
        return CorruptPayloadError(f"bad magic {bytes(raw[:4])!r}")
    if v == _lib.WIRE_BAD_SCHEME:
        return CorruptPayloadError(f"unknown scheme byte {h.scheme}")
    if v == _lib.WIRE_BAD_SHAPE:
        return CorruptPayloadError(f"invalid shape {h.rows}x{h.cols}")
    if v == _lib.WIRE_OUTLIERS_NOT_ALLOWED:
        return CorruptPayloadError(f"{Scheme(h.scheme).name} cannot carry outliers")
    if v == _lib.WIRE_TOO_MANY_OUTLIERS:
        return CorruptPayloadError(f"outlier count {h.outlier_count} exceeds half of {h.cols} channels")
    if v == _lib.WIRE_BAD_GROUP_COUNT:
        return CorruptPayloadError(f"group count {h.group_count} does not match shape (want {h.expected_groups})")
    if v == _lib.WIRE_SIZE_MISMATCH:
        return CorruptPayloadError(f"payload size mismatch: expected {h.total_bytes} bytes, got {buf_len}")
    return CorruptPayloadError(f"invalid group size {h.group_size}")


_CONTENT_ERRORS = ((_lib.ERR_BAD_SCALE, "scales must be finite and non-negative"),
                   (_lib.ERR_BAD_OFFSET, "offsets must be finite"),
                   (_lib.ERR_BAD_INDEX_RANGE, "outlier index out of range"),
                   (_lib.ERR_BAD_INDEX_ORDER, "outlier indices must be strictly increasing"))


def deserialize(buf) -> CompressedTensor:
    """Parse + validate an ADC1 payload into a device record (codec.py:462-546).

    ``buf`` is ``bytes`` (uploaded once) or a uint8 CUDA tensor already in HBM.
    The header is checked by ``adc_parse_header`` (host, 25 bytes); the
    content -- scale / offset finiteness, outlier index range and order -- is
    checked by the device kernel that splits the payload into the record's
    arrays (``adc_deserialize``).  Errors are the reference's
    ``CorruptPayloadError`` messages, raised in the reference's order.
    """
    if isinstance(buf, torch.Tensor):
        if buf.dtype != torch.uint8 or buf.dim() != 1:
            raise ValidationError("device payload must be a 1-D uint8 tensor")
        blob_dev, n = buf, buf.numel()
        head = bytes(buf[:_HEADER.size].cpu().numpy().tobytes()) if n else b""
    else:
        blob = bytes(buf)
        blob_dev, n, head = None, len(blob), blob[:_HEADER.size]
    h = _lib.WireHeader()
    verdict = _lib.lib().adc_parse_header(head, n, _lib.C.byref(h))
    if verdict != _lib.WIRE_OK:
        raise _header_error(verdict, n, head, h)
    dev = _device()
    if blob_dev is None:
        blob_dev = torch.frombuffer(bytearray(blob), dtype=torch.uint8).to(dev)
    else:
        blob_dev = blob_dev.contiguous()
    scheme, rows, cols, k = Scheme(h.scheme), int(h.rows), int(h.cols), int(h.outlier_count)
    gc = int(h.group_count)
    is_mask = scheme is Scheme.BIT_MASK
    codes = torch.empty(int(h.code_bytes), dtype=torch.uint8, device=dev)
    scales = None if is_mask else torch.empty(gc, dtype=torch.float16, device=dev)
    offsets = torch.empty(gc, dtype=torch.float16, device=dev) if scheme is Scheme.ASYMMETRIC_GROUP else None
    idx = torch.empty(k, dtype=torch.int32, device=dev) if k else None
    val = torch.empty((k, rows), dtype=torch.float16, device=dev) if k else None
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    st = _lib.lib().adc_deserialize(blob_dev.data_ptr(), _lib.C.byref(h), _ptr(scales), _ptr(offsets),
                                    codes.data_ptr(), _ptr(idx), _ptr(val), err.data_ptr(), _stream())
    _lib.check(st, "deserialize")
    word = int(err.item()) & 0xffffffff
    for bit, msg in _CONTENT_ERRORS:
        if word & bit:
            raise CorruptPayloadError(msg)
    if is_mask:
        return CompressedTensor(scheme, rows, cols, 0, None, None, None, mask_bits=codes)
    return CompressedTensor(scheme, rows, cols, int(h.group_size), scales, offsets, codes,
                            outlier_indices=None if idx is None else idx.to(torch.int64),
                            outlier_values=val)


# ---------------------------------------------------------------------------
# int8 extension (no reference counterpart; parity unpinned, see
# include/adacc.h adc_compress_int8 and oracle/int8_oracle.py)
# ---------------------------------------------------------------------------
@dataclass
class Int8Tensor:
    """Symmetric group int8 codes with float32 scales (payload N + 4*G bytes)."""
    rows: int
    cols: int
    group_size: int
    codes: torch.Tensor   # int8 (rows*cols,)
    scales: torch.Tensor  # float32 (n_groups,)
    status: torch.Tensor  # int32 [error word, unused]
    shape: tuple = ()

    @property
    def compressed_size_bytes(self) -> int:
        return self.codes.numel() + 4 * self.scales.numel()

    @property
    def compression_ratio(self) -> float:
        return 2 * self.rows * self.cols / self.compressed_size_bytes


def quantize_int8(x, group_size: int = DEFAULT_GROUP_SIZE, *, check: bool = True) -> Int8Tensor:
    """int8 extension compress (device); raises the reference's errors in check mode."""
    if group_size < 1:
        raise ValidationError(f"group_size must be positive, got {group_size}")
    shape = tuple(x.shape) if hasattr(x, "shape") else ()
    t = _as_device_matrix(x)
    rows, cols = t.shape
    n = rows * cols
    dev = t.device
    codes = torch.empty(n, dtype=torch.int8, device=dev)
    scales = torch.empty((n + group_size - 1) // group_size, dtype=torch.float32, device=dev)
    status = torch.zeros(2, dtype=torch.int32, device=dev)
    st = _lib.lib().adc_compress_int8(t.data_ptr(), _DT[t.dtype], rows, cols, group_size, codes.data_ptr(),
                                      scales.data_ptr(), status.data_ptr(), _stream())
    _lib.check(st, "compress_int8")
    ct = Int8Tensor(rows, cols, group_size, codes, scales, status, shape)
    if check:
        raise_for_error_word(int(status[0].item()) & 0xffffffff, rows=rows, cols=cols, k=0)
    return ct


def dequantize_int8(ct: Int8Tensor, out_dtype: torch.dtype = torch.float32) -> torch.Tensor:
    y = torch.empty((ct.rows, ct.cols), dtype=out_dtype, device=ct.codes.device)
    st = _lib.lib().adc_decompress_int8(ct.codes.data_ptr(), ct.scales.data_ptr(), ct.rows, ct.cols,
                                        ct.group_size, y.data_ptr(), _DT[out_dtype], _stream())
    _lib.check(st, "decompress_int8")
    return y


@dataclass
class Int4F32Tensor:
    """Symmetric group int4 codes with float32 scales (payload ceil(N/2) + 4*G bytes)."""
    rows: int
    cols: int
    group_size: int
    codes: torch.Tensor   # uint8 (ceil(rows*cols/2),), the reference nibble order
    scales: torch.Tensor  # float32 (n_groups,)
    status: torch.Tensor  # int32 [error word, unused]
    shape: tuple = ()

    @property
    def compressed_size_bytes(self) -> int:
        return self.codes.numel() + 4 * self.scales.numel()

    @property
    def compression_ratio(self) -> float:
        return 2 * self.rows * self.cols / self.compressed_size_bytes


def quantize_int4_f32(x, group_size: int = DEFAULT_GROUP_SIZE, *, check: bool = True) -> Int4F32Tensor:
    """int4 / float32-scale extension compress (device); the reference's errors in check mode."""
    if group_size < 1:
        raise ValidationError(f"group_size must be positive, got {group_size}")
    shape = tuple(x.shape) if hasattr(x, "shape") else ()
    t = _as_device_matrix(x)
    rows, cols = t.shape
    n = rows * cols
    dev = t.device
    codes = torch.empty((n + 1) // 2, dtype=torch.uint8, device=dev)
    scales = torch.empty((n + group_size - 1) // group_size, dtype=torch.float32, device=dev)
    status = torch.zeros(2, dtype=torch.int32, device=dev)
    st = _lib.lib().adc_compress_int4f32(t.data_ptr(), _DT[t.dtype], rows, cols, group_size, codes.data_ptr(),
                                         scales.data_ptr(), status.data_ptr(), _stream())
    _lib.check(st, "compress_int4f32")
    ct = Int4F32Tensor(rows, cols, group_size, codes, scales, status, shape)
    if check:
        raise_for_error_word(int(status[0].item()) & 0xffffffff, rows=rows, cols=cols, k=0)
    return ct


def dequantize_int4_f32(ct: Int4F32Tensor, out_dtype: torch.dtype = torch.float32) -> torch.Tensor:
    y = torch.empty((ct.rows, ct.cols), dtype=out_dtype, device=ct.codes.device)
    st = _lib.lib().adc_decompress_int4f32(ct.codes.data_ptr(), ct.scales.data_ptr(), ct.rows, ct.cols,
                                           ct.group_size, y.data_ptr(), _DT[out_dtype], _stream())
    _lib.check(st, "decompress_int4f32")
    return y

