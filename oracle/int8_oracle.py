"""CPU restatement of the int8 EXTENSION codec -- TEST INFRASTRUCTURE ONLY.

Parity UNPINNED: the reference (``actplan`` 0.1.0) has no int8 codec
(its SPEC.md:240 lists "no FP8/INT8 variants" as a non-goal),
so there is nothing upstream to pin against.  The semantics below are defined
by this project (include/adacc.h, adc_compress_int8) and this module restates
them in numpy float32 so the CUDA kernels (paper_2508_00806_b200/csrc/int8.cu)
can be checked bit-for-bit:

  h = float16(x)                    the reference's cast and non-finite rule (codec.py:156-171)
  groups of g row-major elements    as the reference's grouping (codec.py:183), tail unpadded
  s = f32(max|h| / 127)             IEEE float32 division
  code = clip(rint(f32(h / s')), -127, 127), s' = 1 if s == 0, ties to even
  dequant = f32(code * s)

and of the int4 / FLOAT32-SCALE extension (adc_compress_int4f32; the reference
rounds every scale to float16, codec.py:192-196):

  s = f32(max|h| / 8)               exact (power-of-two divisor)
  code = clip(rint(f32(h / s')), -8, 7), s' = 1 if s == 0, ties to even
  nibbles packed as the reference's _pack_nibbles (codec.py:199-203)
  dequant = f32(code * s)
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .codec_oracle import OracleError, nibble_pack, nibble_unpack, to_f16_matrix


@dataclass
class Int8CT:
    rows: int
    cols: int
    group: int
    codes: np.ndarray   # int8 (rows*cols,)
    scales: np.ndarray  # float32 (n_groups,)


def quantize_int8(x, group_size: int = 128) -> Int8CT:
    if group_size < 1:
        raise OracleError("ValidationError", f"group_size {group_size}")
    h = to_f16_matrix(x)
    rows, cols = h.shape
    v = h.ravel().astype(np.float32)
    n = v.size
    n_groups = -(-n // group_size)
    pad = n_groups * group_size - n
    vp = np.concatenate([v, np.zeros(pad, np.float32)]) if pad else v
    g = vp.reshape(n_groups, group_size)
    top = np.abs(g).max(axis=1).astype(np.float32)
    s = (top / np.float32(127)).astype(np.float32)
    sd = np.where(s == 0, np.float32(1), s).astype(np.float32)
    q = (g / sd[:, None]).astype(np.float32)
    codes = np.clip(np.rint(q), -127, 127).astype(np.int8).ravel()[:n]
    return Int8CT(rows, cols, group_size, codes, s)


def dequantize_int8(ct: Int8CT) -> np.ndarray:
    n = ct.rows * ct.cols
    s = np.repeat(ct.scales, ct.group)[:n]
    return (ct.codes.astype(np.float32) * s).astype(np.float32).reshape(ct.rows, ct.cols)


@dataclass
class Int4F32CT:
    rows: int
    cols: int
    group: int
    codes: np.ndarray   # uint8 (ceil(rows*cols/2),)
    scales: np.ndarray  # float32 (n_groups,)


def quantize_int4_f32(x, group_size: int = 128) -> Int4F32CT:
    if group_size < 1:
        raise OracleError("ValidationError", f"group_size {group_size}")
    h = to_f16_matrix(x)
    rows, cols = h.shape
    v = h.ravel().astype(np.float32)
    n = v.size
    n_groups = -(-n // group_size)
    pad = n_groups * group_size - n
    vp = np.concatenate([v, np.zeros(pad, np.float32)]) if pad else v
    g = vp.reshape(n_groups, group_size)
    top = np.abs(g).max(axis=1).astype(np.float32)
    s = (top / np.float32(8)).astype(np.float32)
    sd = np.where(s == 0, np.float32(1), s).astype(np.float32)
    q = (g / sd[:, None]).astype(np.float32)
    codes = np.clip(np.rint(q), -8, 7).astype(np.int8).ravel()[:n]
    return Int4F32CT(rows, cols, group_size, nibble_pack(codes), s)


def dequantize_int4_f32(ct: Int4F32CT) -> np.ndarray:
    n = ct.rows * ct.cols
    codes = nibble_unpack(ct.codes, n).astype(np.float32)
    s = np.repeat(ct.scales, ct.group)[:n]
    return (codes * s).astype(np.float32).reshape(ct.rows, ct.cols)

