"""int8 EXTENSION codec (no reference counterpart: parity unpinned).

The semantics are defined by include/adacc.h (adc_compress_int8) and restated
in oracle/int8_oracle.py; the CPU tests pin the restatement's properties, the
GPU tests check the CUDA kernels against it bit-for-bit.
"""

import numpy as np
import pytest

from oracle import int8_oracle as I8
from oracle.codec_oracle import OracleError


def test_oracle_properties():
    rng = np.random.default_rng(0)
    x = rng.normal(size=(64, 96)).astype(np.float32) * rng.uniform(0.01, 100)
    ct = I8.quantize_int8(x, 32)
    assert ct.codes.dtype == np.int8 and ct.scales.dtype == np.float32
    assert ct.codes.min() >= -127 and ct.codes.max() <= 127
    h = x.astype(np.float16).astype(np.float32)
    g = h.reshape(-1, 32)
    # the group maximum maps to +-127 exactly and the error is at most half a step
    assert np.all(np.abs(ct.codes.reshape(-1, 32)).max(axis=1) == 127)
    err = np.abs(I8.dequantize_int8(ct).reshape(-1, 32) - g)
    assert np.all(err <= ct.scales[:, None] * 0.5 * (1 + 2**-20) + 1e-30)


def test_oracle_zero_tail_and_errors():
    ct = I8.quantize_int8(np.zeros((3, 5), np.float32), 4)  # ragged tail group, all zero
    assert np.all(ct.codes == 0) and np.all(ct.scales == 0)
    with pytest.raises(OracleError):
        I8.quantize_int8(np.array([[1.0, np.inf]]), 2)
    with pytest.raises(OracleError):
        I8.quantize_int8(np.ones((2, 2)), 0)


def test_oracle_ties_to_even():
    # h / s exactly k + 1/2: s = 127/127 = 1 -> 2.5 -> 2, 3.5 -> 4, -0.5 -> -0
    x = np.array([[127.0, 2.5, 3.5, -0.5, 0.5, -1.5, 0.0, 1.0]], np.float32)
    ct = I8.quantize_int8(x, 8)
    assert ct.scales[0] == 1.0
    assert ct.codes.tolist() == [127, 2, 4, 0, 0, -2, 0, 1]


CASES = [((256, 768), 128, "float32"), ((8192, 1024), 128, "bfloat16"), ((1000, 40), 8, "float16"),
         ((333, 1024), 64, "bfloat16"), ((7, 13), 5, "float32"), ((64, 4096), 256, "float16"),
         ((3, 1), 1, "float32")]


@pytest.mark.gpu
@pytest.mark.parametrize("shape,group,dtype_name", CASES)
def test_int8_device_matches_oracle(shape, group, dtype_name):
    import torch
    import paper_2508_00806_b200 as adc
    rng = np.random.default_rng(shape[0] + group)
    x = rng.normal(size=shape).astype(np.float32) * 3
    x[:, :: max(1, shape[1] // 7)] *= 25
    x[0, : min(8, shape[1])] = 0.0  # a zero run
    xt = torch.from_numpy(x).to(getattr(torch, dtype_name))
    want = I8.quantize_int8(xt.to(torch.float32).numpy(), group)
    ct = adc.quantize_int8(xt.cuda(), group)
    np.testing.assert_array_equal(ct.codes.cpu().numpy(), want.codes)
    np.testing.assert_array_equal(ct.scales.cpu().numpy().view(np.uint32), want.scales.view(np.uint32))
    y = adc.dequantize_int8(ct).cpu().numpy()
    np.testing.assert_array_equal(y.view(np.uint32), I8.dequantize_int8(want).view(np.uint32))
    yb = adc.dequantize_int8(ct, torch.bfloat16).cpu()
    assert torch.equal(yb, torch.from_numpy(y).to(torch.bfloat16))
    n = shape[0] * shape[1]
    assert ct.compression_ratio == pytest.approx(2 * n / (n + 4 * -(-n // group)))


@pytest.mark.gpu
def test_int8_nonfinite_raises():
    import torch
    import paper_2508_00806_b200 as adc
    x = torch.ones(4, 256, device="cuda", dtype=torch.bfloat16)
    x[2, 7] = float("inf")
    with pytest.raises(adc.NonFiniteInputError):
        adc.quantize_int8(x)


# ---------------------------------------------------------------- int4 with float32 scales
def test_int4f32_oracle_equals_reference_when_scales_are_f16_exact(reference_codec):
    """Where max|h|/8 is exactly a float16 the float32-scale codec must write
    the reference's own int4 codes (only the scale's storage differs)."""
    rng = np.random.default_rng(5)
    x = rng.normal(size=(32, 256)).astype(np.float16).astype(np.float32)
    x.reshape(-1, 128)[:, 0] = 8.0  # group maxima 8 -> s = 1 (f16-exact)
    ct = I8.quantize_int4_f32(x, 128)
    ref = reference_codec.quantize_symmetric(x, 128)
    assert np.array_equal(ct.codes, np.frombuffer(ref.packed_codes, np.uint8))
    assert np.array_equal(ct.scales, ref.scales.astype(np.float32))


def test_int4f32_oracle_properties():
    rng = np.random.default_rng(1)
    x = rng.normal(size=(48, 80)).astype(np.float32) * 3e-3  # scales below the f16 normal range
    ct = I8.quantize_int4_f32(x, 16)
    h = x.astype(np.float16).astype(np.float32).reshape(-1, 16)
    top = np.abs(h).max(axis=1)
    assert np.array_equal(ct.scales, (top / 8).astype(np.float32))  # not rounded to f16
    err = np.abs(I8.dequantize_int4_f32(ct).reshape(-1, 16) - h)
    # half a step, except the +8 s quotient of a positive maximum, clipped to 7 (codec.py:231)
    bound = np.where(h >= 7.5 * ct.scales[:, None], ct.scales[:, None], 0.5 * ct.scales[:, None])
    assert np.all(err <= bound * (1 + 2**-20) + 1e-30)
    assert ct.codes.size == (48 * 80 + 1) // 2


CASES4 = [((256, 768), 128, "float32"), ((8192, 1024), 128, "bfloat16"), ((1000, 40), 8, "float16"),
          ((333, 1024), 64, "bfloat16"), ((7, 13), 5, "float32"), ((64, 4096), 256, "float16"),
          ((3, 1), 1, "float32"), ((5, 7), 3, "bfloat16")]


@pytest.mark.gpu
@pytest.mark.parametrize("shape,group,dtype_name", CASES4)
def test_int4f32_device_matches_oracle(shape, group, dtype_name):
    import torch
    import paper_2508_00806_b200 as adc
    rng = np.random.default_rng(shape[0] + 7 * group)
    x = rng.normal(size=shape).astype(np.float32) * 3
    x[:, :: max(1, shape[1] // 7)] *= 25
    x[0, : min(8, shape[1])] = 0.0
    xt = torch.from_numpy(x).to(getattr(torch, dtype_name))
    want = I8.quantize_int4_f32(xt.to(torch.float32).numpy(), group)
    ct = adc.quantize_int4_f32(xt.cuda(), group)
    np.testing.assert_array_equal(ct.codes.cpu().numpy(), want.codes)
    np.testing.assert_array_equal(ct.scales.cpu().numpy().view(np.uint32), want.scales.view(np.uint32))
    y = adc.dequantize_int4_f32(ct).cpu().numpy()
    np.testing.assert_array_equal(y.view(np.uint32), I8.dequantize_int4_f32(want).view(np.uint32))
    n = shape[0] * shape[1]
    assert ct.compressed_size_bytes == (n + 1) // 2 + 4 * -(-n // group)


def _tie_matrix(top: float, steps: float, rows: int = 64, cols: int = 1024, seed: int = 7):
    """Groups of 128 whose maximum is `top` and whose other elements sit on or
    next to half-integer multiples of the scale (exact and near ties: the
    division-free fast path must hand these to the IEEE division)."""
    rng = np.random.default_rng(seed)
    s = np.float32(top) / np.float32(steps)
    k = rng.integers(-int(steps), int(steps), size=(rows, cols)).astype(np.float32)
    x = ((k + np.float32(0.5)) * s).astype(np.float16).astype(np.float32)
    # nudge a third of them by one f16 ulp either way
    nudge = rng.integers(-1, 2, size=(rows, cols))
    xb = x.astype(np.float16).view(np.uint16).astype(np.int32) + nudge
    x = np.where(rng.random((rows, cols)) < 0.33, xb.astype(np.uint16).view(np.float16).astype(np.float32), x)
    x[:, ::128] = top  # every group's abs-max
    return x


@pytest.mark.gpu
@pytest.mark.parametrize("top", [127.0, 63.5, 1.7, 3000.0, 0.011])
def test_int8_ties_device_matches_oracle(top):
    import torch
    import paper_2508_00806_b200 as adc
    x = _tie_matrix(top, 127.0)
    want = I8.quantize_int8(x, 128)
    ct = adc.quantize_int8(torch.from_numpy(x).cuda(), 128)
    np.testing.assert_array_equal(ct.codes.cpu().numpy(), want.codes)
    y = adc.dequantize_int8(ct).cpu().numpy()
    np.testing.assert_array_equal(y.view(np.uint32), I8.dequantize_int8(want).view(np.uint32))


@pytest.mark.gpu
@pytest.mark.parametrize("top", [8.0, 4.0, 1.7, 3000.0, 0.011])
def test_int4f32_ties_device_matches_oracle(top):
    import torch
    import paper_2508_00806_b200 as adc
    x = _tie_matrix(top, 8.0)
    want = I8.quantize_int4_f32(x, 128)
    ct = adc.quantize_int4_f32(torch.from_numpy(x).cuda(), 128)
    np.testing.assert_array_equal(ct.codes.cpu().numpy(), want.codes)
    y = adc.dequantize_int4_f32(ct).cpu().numpy()
    np.testing.assert_array_equal(y.view(np.uint32), I8.dequantize_int4_f32(want).view(np.uint32))


@pytest.mark.gpu
def test_int8_scale_division_exhaustive():
    """The device computes RN32(top / 127) without a division: every finite
    f16 group maximum (both signs) gives the IEEE quotient's scale and codes."""
    import torch
    import paper_2508_00806_b200 as adc
    tops = np.arange(0, 0x7C00, dtype=np.uint16).view(np.float16).astype(np.float32)
    x = np.zeros((2 * tops.size, 128), dtype=np.float32)
    x[: tops.size, 0] = tops
    x[tops.size:, 5] = -tops
    x[:, 64] = x[:, 0] * 0.37 - x[:, 5] * 0.61  # one more element per group
    want = I8.quantize_int8(x, 128)
    ct = adc.quantize_int8(torch.from_numpy(x).cuda(), 128)
    np.testing.assert_array_equal(ct.scales.cpu().numpy().view(np.uint32), want.scales.view(np.uint32))
    np.testing.assert_array_equal(ct.codes.cpu().numpy(), want.codes)
