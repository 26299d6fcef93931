"""The C-ABI library: loads without a GPU, exports the header, validates args.

No kernel is launched here (CPU-only); the numerics are in test_gpu_parity.py.
"""

import ctypes as C
import re
from pathlib import Path

import pytest

from oracle import codec_oracle as orc
from paper_2508_00806_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "adacc.h"


def declared_symbols():
    return sorted(set(re.findall(r"ADC_API\s+[\w\s\*]+?\b(adc_\w+)\s*\(", HEADER.read_text())))


def test_header_declares_entry_points():
    names = declared_symbols()
    assert {"adc_compress", "adc_decompress", "adc_payload_bytes", "adc_workspace_bytes",
            "adc_detect_outliers", "adc_channel_abs_sums"} <= set(names)


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(_lib.SIGNATURES) == set(declared_symbols())


def test_abi_version_and_name():
    lib = _lib.lib()
    assert lib.adc_abi_version() == 1
    assert b"sm_100a" in lib.adc_version()


@pytest.mark.parametrize("scheme", [0, 1, 2, 3])
@pytest.mark.parametrize("rows,cols,group,k", [(1, 1, 128, 0), (16, 256, 128, 0), (64, 512, 128, 2),
                                                (3, 2, 0, 0), (7, 129, 16, 3), (8192, 768, 128, 8)])
def test_payload_bytes_matches_oracle(scheme, rows, cols, group, k):
    lib = _lib.lib()
    g, cb, tot = C.c_int64(), C.c_int64(), C.c_int64()
    kk = k if scheme == 2 else 0
    assert lib.adc_payload_bytes(scheme, rows, cols, group, kk, C.byref(g), C.byref(cb), C.byref(tot)) == 0
    assert tot.value == orc.payload_bytes(scheme, rows, cols, group, kk)


def test_payload_bytes_rejects_bad_args():
    lib = _lib.lib()
    assert lib.adc_payload_bytes(7, 1, 1, 128, 0, None, None, None) == _lib.EINVAL
    assert lib.adc_payload_bytes(0, 0, 5, 128, 0, None, None, None) == _lib.EINVAL
    assert lib.adc_payload_bytes(0, 2, 5, -3, 0, None, None, None) == _lib.EINVAL


def test_workspace_bytes_grows_with_cols():
    lib = _lib.lib()
    assert lib.adc_workspace_bytes(2, 8, 768, 128) > 768 * 8
    assert lib.adc_workspace_bytes(2, 8, 11008, 128) > lib.adc_workspace_bytes(2, 8, 768, 128)


def test_compress_validation_happens_before_any_launch():
    """ValidationError-class failures return ADC_EINVAL synchronously (no GPU needed)."""
    lib = _lib.lib()
    fake = C.c_void_p(0x1000)
    # empty matrix (codec.py:165-166)
    assert lib.adc_compress(0, fake, 0, 0, 8, 128, 3.0, 0, fake, fake, None, None, None, None,
                            None, None, 0, None) == _lib.EINVAL
    # bad group size (codec.py:174-176)
    assert lib.adc_compress(0, fake, 0, 4, 8, -2, 3.0, 0, fake, fake, None, None, None, None,
                            None, None, 0, None) == _lib.EINVAL
    # unknown scheme / dtype
    assert lib.adc_compress(9, fake, 0, 4, 8, 128, 3.0, 0, fake, fake, None, None, None, None,
                            None, None, 0, None) == _lib.EINVAL
    assert lib.adc_compress(0, fake, 3, 4, 8, 128, 3.0, 0, fake, fake, None, None, None, None,
                            None, None, 0, None) == _lib.EINVAL
    # outlier scheme without workspace
    assert lib.adc_compress(2, fake, 0, 4, 8, 128, 3.0, 4, fake, fake, None, fake, fake, fake,
                            fake, None, 0, None) == _lib.EWORKSPACE
    assert "workspace" in _lib.last_error()


# ---------------------------------------------------------------- ADC1 header check (host C code)
_VERDICT_TEXT = {_lib.WIRE_TRUNCATED: "truncated", _lib.WIRE_BAD_MAGIC: "bad magic",
                 _lib.WIRE_BAD_SCHEME: "unknown scheme", _lib.WIRE_BAD_SHAPE: "invalid shape",
                 _lib.WIRE_OUTLIERS_NOT_ALLOWED: "cannot carry outliers",
                 _lib.WIRE_TOO_MANY_OUTLIERS: "exceeds half", _lib.WIRE_BAD_GROUP_COUNT: "group count",
                 _lib.WIRE_SIZE_MISMATCH: "size mismatch"}


def _blobs():
    import numpy as np
    rng = np.random.default_rng(11)
    x = rng.normal(size=(6, 256)).astype(np.float32)
    x[:, 5] *= 80
    out = []
    for scheme, group in ((0, 128), (0, 0), (0, 7), (1, 32), (2, 128), (3, 0)):
        data = (x > 0).astype(np.uint8) if scheme == 3 else x
        out.append(orc.serialize(orc.compress(data, scheme, group)))
    return out


def _header_verdict(blob):
    h = _lib.WireHeader()
    return _lib.lib().adc_parse_header(blob[:25], len(blob), C.byref(h)), h


def test_parse_header_accepts_every_scheme():
    for blob in _blobs():
        v, h = _header_verdict(blob)
        assert v == _lib.WIRE_OK
        assert h.total_bytes == len(blob)


def test_parse_header_matches_reference_validator(reference_codec):
    """Every single-byte corruption of every header byte (and truncations /
    extensions) gets the reference deserialize's verdict (codec.py:464-493)."""
    checked = 0
    for blob in _blobs():
        variants = [blob[:n] for n in (0, 10, 24, 25, len(blob) - 1)] + [blob + b"\0"]
        for at in range(25):
            for flip in (0x01, 0x80, 0xFF):
                b = bytearray(blob)
                b[at] ^= flip
                variants.append(bytes(b))
        for b in variants:
            v, _ = _header_verdict(b)
            try:
                reference_codec.deserialize(b)
                ref = None
            except reference_codec.CorruptPayloadError as e:
                ref = str(e)
            if v == _lib.WIRE_OK:
                # header accepted: the reference either accepts or rejects on CONTENT
                assert ref is None or not any(t in ref for t in _VERDICT_TEXT.values()), (b[:25], ref)
            else:
                assert ref is not None and _VERDICT_TEXT[v] in ref, (v, ref)
            checked += 1
    assert checked > 400
