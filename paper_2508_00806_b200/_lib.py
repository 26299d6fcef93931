"""ctypes binding of the C-ABI library ``_lib/libadacc.so`` (include/adacc.h).

The product path has no CPU fallback: if the library is missing this module
raises on first use instead of silently degrading.  Loading the library does
not touch the GPU, so the symbol table can be checked on a CPU-only host.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libadacc.so"

# enum mirrors of include/adacc.h
SYMMETRIC_GROUP, ASYMMETRIC_GROUP, OUTLIER_SEPARATED, BIT_MASK = 0, 1, 2, 3
PER_CHANNEL = 0
F32, BF16, F16, U8 = 0, 1, 2, 3
OK, EINVAL, ECUDA, EWORKSPACE = 0, -1, -2, -3

_i64, _vp, _sz = C.c_int64, C.c_void_p, C.c_size_t
_P64 = C.POINTER(C.c_int64)


class WireHeader(C.Structure):
    """adc_wire_header (include/adacc.h)."""
    _fields_ = [("scheme", C.c_int32), ("rows", C.c_uint32), ("cols", C.c_uint32),
                ("group_size", C.c_uint32), ("group_count", C.c_uint32), ("outlier_count", C.c_uint32),
                ("expected_groups", C.c_uint64), ("code_bytes", C.c_uint64), ("total_bytes", C.c_uint64)]


(WIRE_OK, WIRE_TRUNCATED, WIRE_BAD_MAGIC, WIRE_BAD_SCHEME, WIRE_BAD_SHAPE, WIRE_OUTLIERS_NOT_ALLOWED,
 WIRE_TOO_MANY_OUTLIERS, WIRE_BAD_GROUP_SIZE, WIRE_BAD_GROUP_COUNT, WIRE_SIZE_MISMATCH) = range(10)
ERR_BAD_SCALE, ERR_BAD_OFFSET, ERR_BAD_INDEX_RANGE, ERR_BAD_INDEX_ORDER = 16, 32, 64, 128

SIGNATURES = {
    "adc_version": (C.c_char_p, []),
    "adc_abi_version": (C.c_int, []),
    "adc_last_error": (C.c_char_p, []),
    "adc_kernel_launches": (C.c_ulonglong, []),
    "adc_set_option": (C.c_int, [C.c_char_p, C.c_int]),
    "adc_debug_trace_k4": (C.c_int, [_vp, C.c_int]),
    "adc_payload_bytes": (C.c_int, [C.c_int, _i64, _i64, _i64, _i64, _P64, _P64, _P64]),
    "adc_workspace_bytes": (_sz, [C.c_int, _i64, _i64, _i64]),
    "adc_compress": (C.c_int, [C.c_int, _vp, C.c_int, _i64, _i64, _i64, C.c_double, _i64,
                               _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "adc_decompress": (C.c_int, [C.c_int, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64,
                                 _i64, _vp, C.c_int, _vp]),
    "adc_compress_int8": (C.c_int, [_vp, C.c_int, _i64, _i64, _i64, _vp, _vp, _vp, _vp]),
    "adc_decompress_int8": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, C.c_int, _vp]),
    "adc_compress_int4f32": (C.c_int, [_vp, C.c_int, _i64, _i64, _i64, _vp, _vp, _vp, _vp]),
    "adc_decompress_int4f32": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, C.c_int, _vp]),
    "adc_serialize": (C.c_int, [C.c_int, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _vp, _sz,
                                _vp, _vp, _vp]),
    "adc_parse_header": (C.c_int, [C.c_char_p, C.c_uint64, C.POINTER(WireHeader)]),
    "adc_deserialize": (C.c_int, [_vp, C.POINTER(WireHeader), _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "adc_channel_abs_sums": (C.c_int, [_vp, C.c_int, _i64, _i64, _vp, _vp, _vp, _sz, _vp]),
    "adc_detect_outliers": (C.c_int, [_vp, C.c_int, _i64, _i64, C.c_double, _i64, _vp, _vp,
                                      _vp, _vp, _sz, _vp]),
}

_lock = threading.Lock()
_lib = None


class LibraryMissingError(RuntimeError):
    """libadacc.so is not built: there is deliberately no fallback path."""


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise LibraryMissingError(
                    f"{LIB_PATH} not found; build it with `python -m paper_2508_00806_b200.build` "
                    "(the compressor has no CPU fallback)")
            handle = C.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def set_option(key: str, value: int) -> None:
    check(lib().adc_set_option(key.encode(), int(value)), f"set_option({key})")


def last_error() -> str:
    return lib().adc_last_error().decode()


def check(status: int, what: str) -> None:
    if status == OK:
        return
    from .errors import CudaError, ValidationError
    msg = f"{what}: {last_error()}"
    if status == EINVAL:
        raise ValidationError(msg)
    raise CudaError(msg)
