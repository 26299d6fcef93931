"""Deterministic input generators shared by the golden-vector script and the tests.

Every input the parity suite uses is produced here from a seed, so the golden
fixtures only need to store reference *outputs* (or their digests) and the GPU
box can regenerate identical inputs without /root/reference.

Sources of the distributions:
  * worked examples / KATs: reference tests/test_codec.py:54-220;
  * asymmetric tie KAT: SURVEY.md section 0.2 item 3 / Appendix A.5;
  * config 1: BASELINE.json configs[0], SURVEY.md section 8(d) (normal, 8 channels x50;
    asym U[0,1) and per-channel normal*lognormal as in cli.py:253-268);
  * gate 2 / gate 9: reference tests/test_acceptance.py:68-92, 225-250.
"""

from __future__ import annotations

import hashlib

import numpy as np

SYM, ASYM, OUTL, MASK = 0, 1, 2, 3
PER_CHANNEL = 0


def kat_cases():
    """(name, x, scheme, group, threshold) for the reference worked examples."""
    f = np.float32
    out = [
        ("sym_worked", np.array([-2.0, -1.0, 0.0, 1.0, 2.0], f), SYM, 128, 3.0),
        ("sym_zero16", np.zeros(16, f), SYM, 128, 3.0),
        ("sym_ties", np.array([0.5, 1.5, 2.5, 3.5, -0.5, -2.5, 8.0, -8.0], f), SYM, 128, 3.0),
        ("sym_two_groups", np.concatenate([np.full(128, 1.0), np.full(128, 100.0)]).astype(f), SYM, 128, 3.0),
        ("sym_nonfinite", np.array([1.0, np.inf], f), SYM, 128, 3.0),
        ("sym_overflow", np.array([1.0, 70000.0], f), SYM, 128, 3.0),
        ("sym_tail129", np.arange(1, 130, dtype=f), SYM, 128, 3.0),
        ("sym_single", np.array([5.0], f), SYM, 128, 3.0),
        ("asym_worked", np.array([1.0, 2.0, 3.0], f), ASYM, 128, 3.0),
        ("asym_const", np.full(16, 3.5, f), ASYM, 128, 3.0),
        ("asym_linspace", np.linspace(0.0, 1.0, 128).astype(f), ASYM, 128, 3.0),
        ("asym_tie_kat", np.array([3.0, -29.0, 2.0 ** -24] + [0.0] * 13, f), ASYM, 16, 3.0),
        ("pc_scales", np.array([[1.0, 10.0], [2.0, 20.0], [-4.0, -40.0]], f), SYM, PER_CHANNEL, 3.0),
        ("mask_ones", np.ones((8, 128), f), MASK, 0, 3.0),
        ("mask_nonbinary", np.array([0.0, 0.5, 1.0], f), MASK, 0, 3.0),
        ("outl_too_many", np.array([[1000.0, 1000.0, 1.0]] * 4, f), OUTL, 128, 0.1),
        ("outl_const", np.ones((8, 16), f), OUTL, 128, 3.0),
    ]
    rng = np.random.default_rng(5)
    x = (rng.normal(size=(64, 16)) * rng.lognormal(sigma=2.0, size=16)).astype(f)
    out.append(("pc_bound", x, SYM, PER_CHANNEL, 3.0))
    rng = np.random.default_rng(1)
    x = rng.normal(size=(64, 32)).astype(f)
    x[:, 7] *= 50.0
    out.append(("outl_col7", x, OUTL, 128, 3.0))
    rng = np.random.default_rng(2)
    x = rng.normal(size=(32, 256)).astype(f)
    x[:, 100] *= 80.0
    x[:, 200] *= 60.0
    out.append(("outl_100_200", x, OUTL, 128, 3.0))
    rng = np.random.default_rng(3)
    x = rng.normal(size=(16, 128)).astype(f)
    out.append(("outl_none", x, OUTL, 128, 1000.0))
    rng = np.random.default_rng(0)
    out.append(("mask_rand200", (rng.random(200) < 0.5).astype(f), MASK, 0, 3.0))
    return out


def _value_scale(rng):
    return float(10.0 ** rng.uniform(-7, 4))


def random_cases(n: int = 240, seed: int = 1234):
    """Small ragged matrices over every scheme and many group sizes."""
    rng = np.random.default_rng(seed)
    groups = [1, 2, 3, 5, 7, 8, 16, 24, 32, 64, 100, 128, 256, PER_CHANNEL]
    out = []
    for i in range(n):
        rows = int(rng.integers(1, 10))
        cols = int(rng.integers(1, 72))
        kind = i % 4
        x = rng.normal(size=(rows, cols)) * _value_scale(rng)
        if i % 11 == 0:
            x = x + _value_scale(rng)          # one-sided offsets
        if i % 13 == 0:
            x[rng.random(size=x.shape) < 0.3] = 0.0
        if i % 17 == 0:                        # bf16-valued input
            x = _round_bf16(x)
        g = groups[int(rng.integers(0, len(groups)))]
        thr = 3.0
        if kind == OUTL:
            if g == PER_CHANNEL:
                g = 8
            if cols > 1:
                hot = rng.choice(cols, size=min(cols // 3 + 1, int(rng.integers(1, 4))), replace=False)
                x[:, hot] *= float(rng.choice([5.0, 50.0, 500.0]))
            thr = float(rng.choice([3.0, 1.5, 2.5]))
        if kind == MASK:
            x = (rng.random(size=(rows, cols)) < 0.5).astype(np.float64)
            g = 0
        out.append((f"rand{i:03d}", np.asarray(x, np.float32), kind, g, thr))
    return out


def tie_family_cases():
    """Adversarial asymmetric groups of 16: [hi, lo, tiny..., 0...] (Appendix A.5)."""
    rows = []
    for a in range(1, 40):
        for b in range(1, 40):
            for e in (-6, 0, 3):
                hi, lo = a * 2.0 ** e, -b * 2.0 ** e
                tiny = [2.0 ** -24, 2.0 ** -20, 3 * 2.0 ** -24, -(2.0 ** -24), 2.0 ** -14]
                grp = [hi, lo] + tiny + [0.0] * 9
                rows.append(grp)
    x = np.asarray(rows, np.float32)
    half = x.astype(np.float16).astype(np.float32)
    return [("asym_tie_family", half, ASYM, 16, 3.0),
            ("sym_tie_family", half, SYM, 16, 3.0)]


def _round_bf16(x):
    f = np.asarray(x, np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)


def round_bf16(x):
    """float32 -> bfloat16 (RNE) -> float32, as torch's ``.to(torch.bfloat16)``."""
    return _round_bf16(x)


# --------------------------------------------------------------------------
# configuration-sized inputs (digests only)
# --------------------------------------------------------------------------
def config1_input(scheme: int, seed: int, rows: int = 8192, cols: int = 768):
    """BASELINE configs[0]: [8,1024,768] fp32 viewed [8192,768]."""
    rng = np.random.default_rng(seed)
    if scheme == ASYM:
        return rng.random(size=(rows, cols)).astype(np.float32)
    if scheme == MASK:
        return (rng.random(size=(rows, cols)) < 0.9).astype(np.uint8)
    x = rng.normal(size=(rows, cols))
    if scheme == SYM and seed % 2 == 1:      # per-channel flavour (cli.py:256)
        x = x * rng.lognormal(sigma=1.0, size=cols)
    hot = rng.choice(cols, size=8, replace=False)
    x[:, hot] *= 50.0
    return x.astype(np.float32)


def llama_input(seed: int, rows: int = 4096, cols: int = 4096):
    """configs[2]-shaped activation: normal, 1% channels x50, bf16-valued."""
    rng = np.random.default_rng(seed)
    x = rng.normal(size=(rows, cols)).astype(np.float32)
    hot = rng.choice(cols, size=max(1, cols // 100), replace=False)
    x[:, hot] *= 50.0
    return round_bf16(x)


def gate2_inputs():
    """Yield the acceptance-gate-2 tensors in reference order (test_acceptance.py:68-92)."""
    rng = np.random.default_rng(20240811)
    for i in range(1000):
        rows = 1 + i % 8
        cols = 8 * (1 + i % 8)
        scale = 10.0 ** (i % 5 - 2)
        x = (rng.normal(size=(rows, cols)) * scale).astype(np.float32)
        hot = rng.normal(size=(6, 32)).astype(np.float32)
        hot[:, int(rng.integers(0, 32))] *= 500.0
        mask = rng.integers(0, 2, size=rows * cols).astype(np.uint8)
        yield x, hot, mask


def gate9_inputs():
    """Yield the acceptance-gate-9 matrices (test_acceptance.py:225-250)."""
    rng = np.random.default_rng(99)
    for i in range(10_000):
        rows = 1 + i % 8
        cols = 2 + i % 23
        if i % 7 == 0:
            x = np.full((rows, cols), float(i % 5), dtype=np.float32)
        else:
            x = rng.normal(size=(rows, cols)).astype(np.float32)
            if i % 3 == 0:
                x[:, int(rng.integers(0, cols))] *= 20.0
        yield x


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        if a is None:
            h.update(b"<none>")
            continue
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def normalized(scales, offsets, codes, idx, vals, mask_bits):
    """Canonical byte-level view of a compressed tensor for comparison/digests.

    scales/offsets -> float16 bit patterns (uint16); codes/mask -> uint8;
    outlier indices -> uint32; outlier values -> float16 bit patterns.
    Accepts reference (float32 f16-exact scales, ``bytes`` codes), oracle and
    device (float16) representations alike.
    """
    def f16bits(a):
        if a is None:
            return None
        return np.ascontiguousarray(np.asarray(a).astype(np.float16)).view(np.uint16)

    def u8(a):
        if a is None:
            return None
        if isinstance(a, (bytes, bytearray)):
            return np.frombuffer(bytes(a), np.uint8)
        return np.asarray(a, np.uint8).ravel()

    idx = None if idx is None or len(idx) == 0 else np.asarray(idx, np.uint32)
    vals = None if idx is None else f16bits(vals)
    off = f16bits(offsets)
    if off is not None:
        # An all-zero group's offset is (hi+lo)/2 of zeros; its SIGN is whatever
        # numpy's SIMD max/min returns for a tie between -0.0 and +0.0 (CPU
        # dependent).  Numerically identical; compared as +0.
        off = np.where(off == 0x8000, np.uint16(0), off).astype(np.uint16)
    return {
        "scales": f16bits(scales), "offsets": off, "codes": u8(codes),
        "idx": idx, "vals": vals, "mask": u8(mask_bits),
    }


def norm_digest(norm: dict, dequant=None) -> str:
    keys = ("scales", "offsets", "codes", "idx", "vals", "mask")
    return digest(*[norm[k] for k in keys], None if dequant is None else np.asarray(dequant))
