"""Pin the CPU oracle (oracle/codec_oracle.py) to the reference.

Runs without a GPU.  Three layers of evidence:
  1. golden vectors produced by the reference itself (tests/golden/);
  2. the reference's own worked examples restated (tests/test_codec.py);
  3. when /root/reference is present, a live diff on fresh random inputs.
"""

import numpy as np
import pytest

import cases
from _harness import (assert_matches_golden, load_digests, load_small, oracle_run,
                      small_inputs)
from oracle import codec_oracle as orc

SMALL = load_small()
INPUTS = small_inputs()


@pytest.mark.parametrize("name", sorted(SMALL))
def test_oracle_small_golden(name):
    x, s, g, t = INPUTS[name]
    norm, deq = oracle_run(x, s, g, t)
    assert_matches_golden(name, SMALL[name], norm, deq)


def test_asym_tie_kat_value():
    # offset -13, scale 2, code of 2^-24 is 7 (naive f32 gives 6)
    ct = orc.quantize(np.array([3.0, -29.0, 2.0 ** -24] + [0.0] * 13, np.float32), 16, asym=True)
    assert float(ct.offsets[0]) == -13.0 and float(ct.scales[0]) == 2.0
    assert orc.nibble_unpack(ct.codes, 16)[2] == 7


def test_worked_examples():
    # reference tests/test_codec.py:54-75, 95-99, 118-124
    ct = orc.quantize(np.array([-2.0, -1.0, 0.0, 1.0, 2.0], np.float32))
    assert float(ct.scales[0]) == 0.25
    assert orc.nibble_unpack(ct.codes, 5).tolist() == [-8, -4, 0, 4, 7]
    assert orc.dequantize(ct).ravel().tolist() == [-2.0, -1.0, 0.0, 1.0, 1.75]
    ct = orc.quantize(np.array([0.5, 1.5, 2.5, 3.5, -0.5, -2.5, 8.0, -8.0], np.float32))
    assert orc.nibble_unpack(ct.codes, 8).tolist() == [0, 2, 2, 4, 0, -2, 7, -8]
    ct = orc.quantize(np.array([1.0, 2.0, 3.0], np.float32), asym=True)
    assert (float(ct.offsets[0]), float(ct.scales[0])) == (2.0, 0.125)
    assert orc.dequantize(ct).ravel().tolist() == [1.0, 2.0, 2.875]
    ct = orc.quantize(np.array([[1.0, 10.0], [2.0, 20.0], [-4.0, -40.0]], np.float32), orc.PER_CHANNEL)
    assert ct.scales.tolist() == [0.5, 5.0]


def test_payload_formula():
    # reference tests/test_codec.py:254-275
    assert orc.payload_bytes(orc.SYMMETRIC_GROUP, 16, 256, 128) == 2048 + 64
    assert orc.payload_bytes(orc.ASYMMETRIC_GROUP, 16, 256, 128) == 2048 + 128
    assert (orc.payload_bytes(orc.OUTLIER_SEPARATED, 64, 512, 128, 2)
            == orc.payload_bytes(orc.OUTLIER_SEPARATED, 64, 512, 128, 0) + 2 * (4 + 128))
    assert orc.payload_bytes(orc.BIT_MASK, 8, 128, 0) == 128


@pytest.mark.parametrize("n", list(range(1, 300)) + [768, 1000, 1024, 3072, 4096, 11008, 20000])
def test_pairwise_sum_matches_numpy(n):
    """The device stats kernel follows this tree; it must equal ndarray.sum bitwise."""
    rng = np.random.default_rng(n)
    a = rng.normal(size=n) * 10.0 ** rng.integers(-3, 8, size=n)
    assert orc.pairwise_sum(a) == a.sum()
    assert orc.pairwise_sum(a) / n == a.mean()


DIGESTS = load_digests()


@pytest.mark.parametrize("key", sorted(k for k in DIGESTS if k.startswith("config1/")))
def test_oracle_config1_digest(key):
    _, s, g, seed = key.split("/")
    scheme, group, seed = int(s[1:]), int(g[1:]), int(seed[4:])
    x = cases.config1_input(scheme, seed)
    norm, deq = oracle_run(x, scheme, group, 3.0)
    assert cases.norm_digest(norm, deq) == DIGESTS[key]


def test_oracle_llama_digest():
    x = cases.llama_input(0)
    norm, deq = oracle_run(x, cases.OUTL, 128, 3.0)
    assert norm["idx"].size == DIGESTS["llama4096/outl/seed0/k"]
    assert cases.norm_digest(norm, deq) == DIGESTS["llama4096/outl/seed0"]


def test_oracle_gate2_digests():
    parts = {"sym16": [], "asym16": [], "pc": [], "outl16": [], "mask": []}
    for x, hot, mask in cases.gate2_inputs():
        for key, (arr, s, g) in {
            "sym16": (x, cases.SYM, 16), "asym16": (x, cases.ASYM, 16),
            "pc": (x, cases.SYM, cases.PER_CHANNEL), "outl16": (hot, cases.OUTL, 16),
            "mask": (mask, cases.MASK, 0),
        }.items():
            norm, deq = oracle_run(arr, s, g, 3.0)
            parts[key].append(cases.norm_digest(norm, deq))
    for key, lst in parts.items():
        assert cases.digest(np.array(lst)) == DIGESTS[f"gate2/{key}"], key


def test_oracle_gate9_digest():
    flagged = [",".join(str(i) for i in orc.outlier_channels(x).tolist())
               for x in cases.gate9_inputs()]
    assert cases.digest(np.array(flagged)) == DIGESTS["gate9/flagged"]


def test_oracle_vs_live_reference(reference_codec):
    """Fresh random inputs, diffed against the live reference (build container only)."""
    ref = reference_codec
    rng = np.random.default_rng(4242)
    for i in range(150):
        rows, cols = int(rng.integers(1, 40)), int(rng.integers(1, 300))
        x = (rng.normal(size=(rows, cols)) * 10.0 ** rng.uniform(-5, 3)).astype(np.float32)
        if cols > 4:
            x[:, int(rng.integers(0, cols))] *= 60.0
        for s, g in ((0, 128), (0, 0), (1, 128), (1, 16), (2, 128), (2, 8)):
            try:
                rct = ref.compress(x, ref.SchemeSpec(ref.Scheme(s), g, 3.0))
                want = (cases.normalized(rct.scales, rct.offsets, rct.packed_codes,
                                         rct.outlier_indices, rct.outlier_values, None),
                        ref.decompress(rct))
            except Exception as exc:  # reference error type by name
                want = (type(exc).__name__, None)
            got = oracle_run(x, s, g, 3.0)
            if isinstance(want[0], str):
                assert got[0] == want[0]
                continue
            assert cases.norm_digest(*got) == cases.norm_digest(*want), (i, s, g)
