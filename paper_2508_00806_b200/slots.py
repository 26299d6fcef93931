"""Preallocated compressor slots: the zero-overhead launch path.

A :class:`CodecSlot` owns every device buffer one (shape, scheme) activation
needs -- payload, outlier side buffer, workspace, status word -- allocated
once, and issues the C-ABI calls with cached raw pointers.  This is what the
bench, the profiler and the training hooks use on the hot path: no torch
allocation and no host synchronisation per call, so the step can also be
captured into a CUDA graph.

Memory of a slot is the reference payload (codec.py:133-145) plus
``k_cap * (4 + 2 * rows)`` bytes of outlier capacity.
"""

from __future__ import annotations

import torch

from . import _lib
from .codec import PER_CHANNEL, CompressedTensor, Scheme, SchemeSpec, _layout

_IN = {torch.float32: _lib.F32, torch.bfloat16: _lib.BF16, torch.float16: _lib.F16,
       torch.uint8: _lib.U8, torch.bool: _lib.U8}


class CodecSlot:
    def __init__(self, rows: int, cols: int, spec: SchemeSpec, in_dtype: torch.dtype,
                 out_dtype: torch.dtype | None = None, *, k_cap: int | None = None,
                 device=None, status: torch.Tensor | None = None):
        self.rows, self.cols, self.spec = int(rows), int(cols), spec
        self.scheme = Scheme(spec.scheme)
        self.in_dtype = in_dtype
        self.out_dtype = out_dtype or (torch.uint8 if self.scheme is Scheme.BIT_MASK else in_dtype)
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        g = spec.group_size if self.scheme is not Scheme.BIT_MASK else 0
        self.group = g
        n_groups, code_bytes, _ = _layout(int(self.scheme), self.rows, self.cols, g)
        self.codes = torch.empty(code_bytes, dtype=torch.uint8, device=dev)
        self.scales = self.offsets = self.idx = self.val = self.ws = None
        self.k_cap = 0
        # status = [error word, k]; shared across slots when the caller passes one
        self.status = status if status is not None else torch.zeros(2, dtype=torch.int32, device=dev)
        if self.scheme is not Scheme.BIT_MASK:
            self.scales = torch.empty(n_groups, dtype=torch.float16, device=dev)
            if self.scheme is Scheme.ASYMMETRIC_GROUP:
                self.offsets = torch.empty(n_groups, dtype=torch.float16, device=dev)
        self.k_status = self.status
        if self.scheme is Scheme.OUTLIER_SEPARATED:
            self.k_cap = self.cols // 2 if k_cap is None else int(k_cap)
            self.idx = torch.empty(max(self.k_cap, 1), dtype=torch.int32, device=dev)
            self.val = torch.empty((max(self.k_cap, 1), self.rows), dtype=torch.float16, device=dev)
            # each outlier slot keeps its own k (shared status would race on k)
            self.k_status = torch.zeros(2, dtype=torch.int32, device=dev)
        self.ws_bytes = 0
        if self.scheme is Scheme.OUTLIER_SEPARATED or (self.scheme is not Scheme.BIT_MASK
                                                       and g == PER_CHANNEL):
            self.ws_bytes = _lib.lib().adc_workspace_bytes(int(self.scheme), self.rows, self.cols, g)
            self.ws = torch.zeros(self.ws_bytes, dtype=torch.uint8, device=dev)
        p = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        self._c_args = (int(self.scheme), _IN[in_dtype], self.rows, self.cols, g,
                        float(spec.z_threshold), self.k_cap, p(self.codes), p(self.scales),
                        p(self.offsets), p(self.idx), p(self.val),
                        None if self.idx is None else self.k_status.data_ptr() + 4,
                        self.status.data_ptr(), p(self.ws), self.ws_bytes)
        out_code = _lib.U8 if self.scheme is Scheme.BIT_MASK else _IN[self.out_dtype]
        self._d_args = (int(self.scheme), p(self.codes), p(self.scales), p(self.offsets),
                        p(self.idx), p(self.val),
                        None if self.idx is None else self.k_status.data_ptr() + 4,
                        self.k_cap, self.rows, self.cols, g)
        self._out_code = out_code
        self._compress = _lib.lib().adc_compress
        self._decompress = _lib.lib().adc_decompress

    # -- raw launches --------------------------------------------------------
    def compress_ptr(self, x_ptr: int, stream: int) -> None:
        a = self._c_args
        st = self._compress(a[0], x_ptr, *a[1:], stream)
        if st:
            _lib.check(st, "compress")

    def decompress_ptr(self, y_ptr: int, stream: int) -> None:
        st = self._decompress(*self._d_args, y_ptr, self._out_code, stream)
        if st:
            _lib.check(st, "decompress")

    # -- tensor conveniences -------------------------------------------------
    def compress(self, x: torch.Tensor) -> None:
        assert x.is_contiguous() and x.numel() == self.rows * self.cols and x.dtype == self.in_dtype
        self.compress_ptr(x.data_ptr(), torch.cuda.current_stream(x.device).cuda_stream)

    def decompress(self, out: torch.Tensor | None = None) -> torch.Tensor:
        if out is None:
            out = torch.empty((self.rows, self.cols), dtype=self.out_dtype, device=self.device)
        self.decompress_ptr(out.data_ptr(), torch.cuda.current_stream(out.device).cuda_stream)
        return out

    # -- accounting ----------------------------------------------------------
    @property
    def device_bytes(self) -> int:
        """HBM the slot holds for the payload (incl. unused outlier capacity)."""
        return sum(t.numel() * t.element_size() for t in (self.codes, self.scales, self.offsets, self.idx, self.val)
                   if t is not None)

    def payload_bytes(self, k: int = 0) -> int:
        return _layout(int(self.scheme), self.rows, self.cols, self.group, k)[2]

    @property
    def elem_in(self) -> int:
        return torch.empty((), dtype=self.in_dtype).element_size()

    @property
    def elem_out(self) -> int:
        return torch.empty((), dtype=self.out_dtype).element_size()

    def algorithmic_bytes(self, k: int = 0) -> tuple[int, int]:
        """(compress, decompress) bytes: N*s_in + payload, payload + N*s_out."""
        n = self.rows * self.cols
        pay = self.payload_bytes(k)
        return n * self.elem_in + pay, pay + n * self.elem_out

    def record(self) -> CompressedTensor:
        """A CompressedTensor view of the slot's current contents (k from the device)."""
        return CompressedTensor(self.scheme, self.rows, self.cols, self.group, self.scales,
                                self.offsets, None if self.scheme is Scheme.BIT_MASK else self.codes,
                                outlier_indices=self.idx, outlier_values=self.val,
                                mask_bits=self.codes if self.scheme is Scheme.BIT_MASK else None,
                                k_dev=self.k_status, k_cap=self.k_cap)


class Int8Slot:
    """Preallocated int8 group codes + float32 scales (the EXTENSION codec,
    ``adc_compress_int8``; no reference counterpart): the same launch-path
    interface as :class:`CodecSlot`, for kinds a caller moves to 8-bit codes
    (``ActivationPolicy(codec_overrides=...)``)."""

    k_cap = 0

    def __init__(self, rows: int, cols: int, group: int, in_dtype: torch.dtype,
                 out_dtype: torch.dtype | None = None, *, device=None, status: torch.Tensor | None = None):
        self.rows, self.cols, self.group = int(rows), int(cols), int(group)
        self.in_dtype = in_dtype
        self.out_dtype = out_dtype or in_dtype
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        n = self.rows * self.cols
        self.codes = torch.empty(n, dtype=torch.int8, device=dev)
        self.scales = torch.empty(-(-n // self.group), dtype=torch.float32, device=dev)
        self.status = status if status is not None else torch.zeros(2, dtype=torch.int32, device=dev)
        self._compress = _lib.lib().adc_compress_int8
        self._decompress = _lib.lib().adc_decompress_int8
        self._c = (_IN[in_dtype], self.rows, self.cols, self.group, self.codes.data_ptr(),
                   self.scales.data_ptr(), self.status.data_ptr())
        self._d = (self.codes.data_ptr(), self.scales.data_ptr(), self.rows, self.cols, self.group)
        self._out_code = _IN[self.out_dtype]

    def compress_ptr(self, x_ptr: int, stream: int) -> None:
        st = self._compress(x_ptr, *self._c, stream)
        if st:
            _lib.check(st, "compress_int8")

    def decompress_ptr(self, y_ptr: int, stream: int) -> None:
        st = self._decompress(*self._d, y_ptr, self._out_code, stream)
        if st:
            _lib.check(st, "decompress_int8")

    @property
    def device_bytes(self) -> int:
        return self.codes.numel() + 4 * self.scales.numel()
