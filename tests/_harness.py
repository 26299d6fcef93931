"""Helpers shared by the parity tests: run the oracle / load golden vectors."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

import cases
from oracle import codec_oracle as orc

GOLDEN = Path(__file__).resolve().parent / "golden"


def oracle_run(x, scheme, group, thr):
    """Oracle compress+decompress -> (normalized dict, dequant) or error name."""
    try:
        ct = orc.compress(x, scheme, group, thr)
    except orc.OracleError as exc:
        return exc.kind, None
    deq = orc.decompress(ct)
    norm = cases.normalized(
        None if scheme == cases.MASK else ct.scales, ct.offsets,
        None if scheme == cases.MASK else ct.codes,
        ct.outlier_idx, ct.outlier_val, ct.mask_bits)
    return norm, deq


def load_small():
    """{name: {"error": str} | {key: array, "dequant": array}} from small_golden.npz."""
    z = np.load(GOLDEN / "small_golden.npz")
    out = {str(n): {} for n in z["__names__"]}
    for key in z.files:
        if key == "__names__":
            continue
        name, field = key.split("/", 1)
        out[name][field] = z[key]
    for name, d in out.items():
        if "error" in d:
            d["error"] = str(d["error"])
    return out


def load_digests():
    return json.loads((GOLDEN / "digests.json").read_text())


def small_inputs():
    return {name: (x, s, g, t) for name, x, s, g, t in
            cases.kat_cases() + cases.random_cases() + cases.tie_family_cases()}


def assert_matches_golden(name, golden, norm, deq):
    if "error" in golden:
        assert norm == golden["error"], f"{name}: expected {golden['error']}, got {norm!r}"
        return
    assert not isinstance(norm, str), f"{name}: unexpected error {norm}"
    for key in ("scales", "offsets", "codes", "idx", "vals", "mask"):
        want = golden.get(key)
        got = norm[key]
        if want is None:
            assert got is None or got.size == 0, f"{name}/{key}: expected none"
        else:
            assert got is not None, f"{name}/{key}: missing"
            np.testing.assert_array_equal(np.asarray(got), want, err_msg=f"{name}/{key}")
    want = np.ascontiguousarray(golden["dequant"])
    got = np.ascontiguousarray(np.asarray(deq))
    assert got.shape == want.shape and got.dtype == want.dtype, f"{name}/dequant: {got.shape}/{got.dtype}"
    # bitwise, so -0.0 vs +0.0 would be caught too
    np.testing.assert_array_equal(got.view(np.uint8), want.view(np.uint8), err_msg=f"{name}/dequant")


def device_run(x, scheme, group, thr, *, in_dtype=None):
    """CUDA path (through the C-ABI) -> (normalized dict, dequant f32) or error name."""
    import torch
    import paper_2508_00806_b200 as adc
    from paper_2508_00806_b200 import errors as E
    t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(x))
    if in_dtype is not None:
        t = t.to(in_dtype)
    try:
        ct = adc.compress(t, adc.SchemeSpec(adc.Scheme(scheme), group, thr))
    except E.ActplanError as exc:
        return type(exc).__name__, None
    deq = adc.decompress(ct).cpu().numpy()
    if scheme == cases.MASK:
        norm = cases.normalized(None, None, None, None, None, ct.mask_bits.cpu().numpy())
    else:
        norm = cases.normalized(
            ct.scales.cpu().numpy(),
            None if ct.offsets is None else ct.offsets.cpu().numpy(),
            ct.packed_codes.cpu().numpy(),
            None if ct.outlier_indices is None else ct.outlier_indices.cpu().numpy(),
            None if ct.outlier_values is None else ct.outlier_values.cpu().numpy(), None)
    return norm, deq
