"""The reference's own codec API tests, restated against the device API.

Each test cites the reference test it restates (/root/reference/pkg/tests):
scheme mapping (test_codec.py:224-251), size formula / ratio (:254-275),
wire format incl. every CorruptPayloadError path (:278-337,
test_codec_properties.py:161-187), measure_codec report fields (:340-349).
Arrays come back as device tensors; comparisons are on their bytes.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def adc():
    import torch
    torch.cuda.init()
    import paper_2508_00806_b200 as m
    return m


def _np(t):
    return t.detach().cpu().numpy()


# ---------------------------------------------------------------- scheme mapping
KIND_SCHEME = [("linear", "OUTLIER_SEPARATED"), ("layer_norm", "OUTLIER_SEPARATED"),
               ("gelu", "OUTLIER_SEPARATED"), ("qkv_matrix", "SYMMETRIC_GROUP"),
               ("softmax", "ASYMMETRIC_GROUP"), ("score", "ASYMMETRIC_GROUP"),
               ("dropout_mask", "BIT_MASK"), ("other", "SYMMETRIC_GROUP")]


@pytest.mark.parametrize("kind,scheme", KIND_SCHEME)
def test_kind_to_scheme(adc, kind, scheme):  # test_codec.py:225-238
    assert adc.scheme_for(adc.LayerKind(kind)).scheme is adc.Scheme[scheme]


def test_qkv_is_per_channel(adc):  # test_codec.py:240-241
    assert adc.scheme_for(adc.LayerKind.QKV_MATRIX).group_size == adc.PER_CHANNEL


def test_compress_dispatches(adc):  # test_codec.py:243-251
    rng = np.random.default_rng(4)
    x = rng.normal(size=(8, 128)).astype(np.float32)
    for kind in adc.LayerKind:
        spec = adc.scheme_for(kind)
        data = (x > 0).astype(np.float32) if spec.scheme is adc.Scheme.BIT_MASK else x
        ct = adc.compress(data, spec)
        assert ct.scheme is spec.scheme
        assert tuple(adc.decompress(ct).shape) == (8, 128)


# ---------------------------------------------------------------- sizes / ratios
def test_symmetric_formula(adc):  # test_codec.py:255-260
    ct = adc.quantize_symmetric(np.ones((16, 256), dtype=np.float32))
    expected = adc.packed_payload_bytes(adc.Scheme.SYMMETRIC_GROUP, 16, 256, adc.DEFAULT_GROUP_SIZE)
    assert ct.compressed_size_bytes == expected == 2048 + 64
    assert ct.original_bytes == 16 * 256 * 2
    assert ct.compression_ratio == ct.original_bytes / expected


def test_asymmetric_adds_offsets(adc):  # test_codec.py:262-265
    sym = adc.packed_payload_bytes(adc.Scheme.SYMMETRIC_GROUP, 16, 256, 128)
    asym = adc.packed_payload_bytes(adc.Scheme.ASYMMETRIC_GROUP, 16, 256, 128)
    assert asym == sym + 32 * 2


def test_outlier_cost_per_channel(adc):  # test_codec.py:267-270
    base = adc.packed_payload_bytes(adc.Scheme.OUTLIER_SEPARATED, 64, 512, 128, 0)
    with_two = adc.packed_payload_bytes(adc.Scheme.OUTLIER_SEPARATED, 64, 512, 128, 2)
    assert with_two == base + 2 * (4 + 2 * 64)


def test_rate_helper_matches_ratio(adc):  # test_codec.py:272-275
    rate = adc.outlier_separated_rate(64, 512, 3, 128)
    size = adc.packed_payload_bytes(adc.Scheme.OUTLIER_SEPARATED, 64, 512, 128, 3)
    assert rate == size / (64 * 512 * 2)


@pytest.mark.parametrize("scheme,group", [(0, 128), (0, 0), (1, 32), (2, 128), (3, 0)])
def test_record_sizes_match_formula(adc, scheme, group):  # test_codec_properties.py:150-158
    rng = np.random.default_rng(scheme * 7 + group)
    x = rng.normal(size=(24, 320)).astype(np.float32)
    x[:, 11] *= 80.0
    if scheme == 3:
        x = (x > 0).astype(np.uint8)
    ct = adc.compress(x, adc.SchemeSpec(adc.Scheme(scheme), group))
    assert ct.compressed_size_bytes == adc.packed_payload_bytes(ct.scheme, ct.rows, ct.cols, ct.group_size,
                                                                ct.outlier_count)
    assert ct.original_bytes == 24 * 320 * (1 if scheme == 3 else 2)
    assert ct.compression_ratio == pytest.approx(ct.original_bytes / ct.compressed_size_bytes)
    if scheme == 2:
        assert ct.outlier_count >= 1 and 11 in _np(ct.outlier_indices).tolist()


# ---------------------------------------------------------------- wire format
SPECS = [(0, 128), (0, 0), (1, 32), (2, 128), (3, 0)]


def _spec_input(adc, scheme):
    rng = np.random.default_rng(6)
    x = rng.normal(size=(16, 256)).astype(np.float32)
    if scheme == 3:
        x = (x > 0).astype(np.float32)
    if scheme == 2:
        x[:, 17] *= 90.0
    return x


@pytest.mark.parametrize("scheme,group", SPECS)
def test_wire_round_trip(adc, scheme, group):  # test_codec.py:279-297
    ct = adc.compress(_spec_input(adc, scheme), adc.SchemeSpec(adc.Scheme(scheme), group))
    blob = adc.serialize(ct)
    back = adc.deserialize(blob)
    assert adc.serialize(back) == blob
    assert np.array_equal(_np(adc.decompress(back)).view(np.uint8), _np(adc.decompress(ct)).view(np.uint8))


@pytest.mark.parametrize("scheme,group", SPECS)
def test_device_deserialize_round_trip(adc, scheme, group):
    """The same round trip with the payload already in HBM (device validator)."""
    import torch
    ct = adc.compress(_spec_input(adc, scheme), adc.SchemeSpec(adc.Scheme(scheme), group))
    blob = adc.serialize(ct)
    dev = torch.frombuffer(bytearray(blob), dtype=torch.uint8).cuda()
    back = adc.deserialize(dev)
    assert adc.serialize(back) == blob
    assert np.array_equal(_np(adc.decompress(back)).view(np.uint8), _np(adc.decompress(ct)).view(np.uint8))


def test_header_size(adc):  # test_codec.py:299-302
    ct = adc.quantize_symmetric(np.ones(8, dtype=np.float32))
    assert len(adc.serialize(ct)) == adc.SERIALIZED_HEADER_BYTES + ct.compressed_size_bytes


def _blob(adc):
    return adc.serialize(adc.quantize_symmetric(np.ones(8, dtype=np.float32)))


def _both(adc, blob):
    """Feed a payload to deserialize as host bytes and as a device tensor."""
    import torch
    yield bytes(blob)
    yield torch.frombuffer(bytearray(blob), dtype=torch.uint8).cuda() if len(blob) else \
        torch.empty(0, dtype=torch.uint8, device="cuda")


def _rejects(adc, blob, match=None):
    for b in _both(adc, blob):
        with pytest.raises(adc.CorruptPayloadError, match=match):
            adc.deserialize(b)


def test_bad_magic(adc):  # test_codec.py:304-307
    blob = _blob(adc)
    _rejects(adc, b"XXXX" + blob[4:], "bad magic")


def test_truncated(adc):  # test_codec.py:309-312
    _rejects(adc, _blob(adc)[:-1], "size mismatch")
    _rejects(adc, _blob(adc)[:10], "truncated")


def test_trailing_garbage(adc):  # test_codec.py:314-317
    _rejects(adc, _blob(adc) + b"\x00", "size mismatch")


def test_bad_scheme_byte(adc):  # test_codec.py:319-323
    blob = bytearray(_blob(adc))
    blob[4] = 200
    _rejects(adc, bytes(blob), "unknown scheme")


def _outlier_blob(adc):
    rng = np.random.default_rng(7)
    x = rng.normal(size=(8, 256)).astype(np.float32)
    x[:, 3] *= 90.0
    x[:, 9] *= 95.0
    ct = adc.compress_outlier_separated(x)
    return bytearray(adc.serialize(ct)), ct


def test_unsorted_outlier_indices(adc):  # test_codec.py:325-337
    blob, ct = _outlier_blob(adc)
    assert _np(ct.outlier_indices).tolist() == [3, 9]
    idx_off = len(blob) - ct.outlier_values.numel() * 2 - ct.outlier_count * 4
    blob[idx_off:idx_off + 8] = blob[idx_off + 4:idx_off + 8] + blob[idx_off:idx_off + 4]
    _rejects(adc, bytes(blob), "strictly increasing")


def test_outlier_index_out_of_range(adc):  # codec.py:530-531
    blob, ct = _outlier_blob(adc)
    idx_off = len(blob) - ct.outlier_values.numel() * 2 - ct.outlier_count * 4
    blob[idx_off + 4:idx_off + 8] = (256).to_bytes(4, "little")
    _rejects(adc, bytes(blob), "out of range")


def test_bad_scales_and_offsets(adc):  # codec.py:512-518
    import struct
    ct = adc.quantize_symmetric(np.arange(16, dtype=np.float32), 8)
    blob = bytearray(adc.serialize(ct))
    for bad in (np.float16(-1.0), np.float16(np.inf), np.float16(np.nan)):
        b = bytearray(blob)
        b[25:27] = struct.pack("<e", bad)
        _rejects(adc, bytes(b), "scales must be finite and non-negative")
    ca = adc.quantize_asymmetric(np.arange(16, dtype=np.float32), 8)
    blob = bytearray(adc.serialize(ca))
    b = bytearray(blob)
    b[27:29] = struct.pack("<e", np.float16(np.inf))  # first offset
    _rejects(adc, bytes(b), "offsets must be finite")


def test_header_field_checks(adc):  # codec.py:474-505
    import struct
    hdr = struct.Struct("<4sBIIIII")
    good = _blob(adc)
    _, s, r, c, g, gc, k = hdr.unpack_from(good)
    body = good[hdr.size:]
    _rejects(adc, hdr.pack(b"ADC1", s, 0, c, g, gc, k) + body, "invalid shape")
    _rejects(adc, hdr.pack(b"ADC1", s, r, c, g, gc, 1) + body, "cannot carry outliers")
    _rejects(adc, hdr.pack(b"ADC1", s, r, c, g, gc + 1, k) + body, "group count")
    blob, ct = _outlier_blob(adc)
    _, s, r, c, g, gc, k = hdr.unpack_from(blob)
    _rejects(adc, hdr.pack(b"ADC1", s, r, c, g, gc, c) + bytes(blob[hdr.size:]), "exceeds half")


@pytest.mark.parametrize("flip_at", [0, 4, 5, 9, 13, 24])
def test_header_corruption_detected_or_harmless(adc, flip_at):  # test_codec_properties.py:177-187
    x = np.arange(64, dtype=np.float32).reshape(4, 16)
    blob = bytearray(adc.serialize(adc.quantize_symmetric(x, 8)))
    blob[flip_at] ^= 0xFF
    for b in _both(adc, blob):
        try:
            back = adc.deserialize(b)
        except adc.CorruptPayloadError:
            continue
        assert adc.serialize(back) == bytes(blob)


@pytest.mark.parametrize("group", [8, 16, 0])
def test_wire_round_trip_bytes_random(adc, group):  # test_codec_properties.py:161-168
    rng = np.random.default_rng(group + 100)
    for _ in range(40):
        rows, cols = int(rng.integers(1, 5)), int(rng.integers(1, 33))
        x = (rng.normal(size=(rows, cols)) * 10 ** rng.uniform(-3, 3)).astype(np.float32)
        for q in (adc.quantize_symmetric, adc.quantize_asymmetric):
            blob = adc.serialize(q(x, group))
            assert adc.serialize(adc.deserialize(blob)) == blob


def test_values_survive_wire(adc):  # test_codec_properties.py:170-174
    rng = np.random.default_rng(5)
    for _ in range(30):
        x = rng.normal(size=(int(rng.integers(1, 5)), int(rng.integers(1, 17)))).astype(np.float32)
        ct = adc.quantize_symmetric(x, 8)
        a = _np(adc.dequantize(adc.deserialize(adc.serialize(ct))))
        assert np.array_equal(a.view(np.uint32), _np(adc.dequantize(ct)).view(np.uint32))


# ---------------------------------------------------------------- measure_codec
def test_measure_report_fields(adc):  # test_codec.py:340-349
    rng = np.random.default_rng(8)
    x = rng.normal(size=(32, 512)).astype(np.float32)
    report = adc.measure_codec(x, adc.SchemeSpec(adc.Scheme.SYMMETRIC_GROUP))
    assert report.scheme is adc.Scheme.SYMMETRIC_GROUP
    assert report.compress_ms >= 0.0
    assert report.decompress_ms >= 0.0
    assert report.original_bytes == 32 * 512 * 2
    assert report.ratio == pytest.approx(report.original_bytes / report.compressed_bytes)


@pytest.mark.parametrize("scheme,group", SPECS)
def test_measure_every_scheme(adc, scheme, group):
    x = _spec_input(adc, scheme)
    r = adc.measure_codec(x, adc.SchemeSpec(adc.Scheme(scheme), group))
    ct = adc.compress(x, adc.SchemeSpec(adc.Scheme(scheme), group))
    assert r.compressed_bytes == ct.compressed_size_bytes
    assert 0 < r.compress_ms < 1000 and 0 < r.decompress_ms < 1000


# ---------------------------------------------------------------- float64 input rounding
def test_float64_input_rounds_once_like_numpy(adc):
    """np.asarray(x, dtype=float16) rounds float64 once (codec.py:158); values just
    past f16 midpoints expose a double rounding through float32."""
    import torch
    from oracle import codec_oracle as orc
    base = np.array([1 + 2 ** -11 + 2 ** -40, 2049.0000001, -(1 + 2 ** -11 + 2 ** -40), 3.0] * 64)
    rng = np.random.default_rng(3)
    x = np.concatenate([base, rng.normal(size=768) * 100]).reshape(8, 128)
    for inp in (x, torch.from_numpy(x), torch.from_numpy(x).cuda(), x.tolist()):
        ct = adc.compress_outlier_separated(inp)
        ref = orc.compress(x, orc.OUTLIER_SEPARATED, 128, 3.0)
        assert np.array_equal(_np(ct.packed_codes), ref.codes)
        assert np.array_equal(_np(ct.scales).view(np.uint16), ref.scales.view(np.uint16))
        got = _np(adc.decompress(ct))
        assert np.array_equal(got.view(np.uint32), orc.decompress(ref).view(np.uint32))
