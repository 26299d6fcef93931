"""Generate golden vectors by running the REFERENCE codec (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Imports ``actplan`` from /root/reference/pkg/src (read-only, never copied),
feeds it the seeded inputs of ``cases.py`` and writes
  * ``small_golden.npz``  -- full outputs of every small case (KATs, ragged
    random matrices, adversarial tie families);
  * ``digests.json``      -- sha256 digests of the outputs of the large cases
    (config-1 shapes, Llama-shaped, acceptance gates 2 and 9).
The GPU box regenerates the inputs from the same seeds and compares its
outputs against these files; nothing there reads /root/reference.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

import cases  # noqa: E402
from actplan import codec as ref  # noqa: E402
from actplan import errors as ref_errors  # noqa: E402


def run_ref(x, scheme, group, thr):
    """Reference compress + decompress -> (normalized dict, dequant) or error name."""
    spec = ref.SchemeSpec(ref.Scheme(scheme), group, thr)
    try:
        ct = ref.compress(x, spec)
    except ref_errors.ActplanError as exc:
        return type(exc).__name__, None
    out = ref.decompress(ct)
    norm = cases.normalized(
        None if scheme == cases.MASK else ct.scales,
        ct.offsets,
        None if scheme == cases.MASK else ct.packed_codes,
        ct.outlier_indices, ct.outlier_values, ct.mask_bits)
    return norm, np.asarray(out)


def small():
    store = {}
    names = []
    for name, x, scheme, group, thr in (cases.kat_cases() + cases.random_cases()
                                         + cases.tie_family_cases()):
        norm, deq = run_ref(x, scheme, group, thr)
        names.append(name)
        if isinstance(norm, str):
            store[f"{name}/error"] = np.array(norm)
            continue
        for key, val in norm.items():
            if val is not None:
                store[f"{name}/{key}"] = val
        store[f"{name}/dequant"] = deq
    store["__names__"] = np.array(names)
    np.savez_compressed(HERE / "small_golden.npz", **store)
    print(f"small_golden.npz: {len(names)} cases")


def large():
    dig = {}
    for scheme in (cases.SYM, cases.ASYM, cases.OUTL, cases.MASK):
        for seed in range(5):
            x = cases.config1_input(scheme, seed)
            group = 128
            if scheme == cases.SYM and seed % 2 == 1:
                group = cases.PER_CHANNEL
            if scheme == cases.MASK:
                group = 0
            norm, deq = run_ref(x, scheme, group, 3.0)
            dig[f"config1/s{scheme}/g{group}/seed{seed}"] = cases.norm_digest(norm, deq)
    for seed in range(2):
        x = cases.llama_input(seed)
        norm, deq = run_ref(x, cases.OUTL, 128, 3.0)
        dig[f"llama4096/outl/seed{seed}"] = cases.norm_digest(norm, deq)
        dig[f"llama4096/outl/seed{seed}/k"] = int(0 if norm["idx"] is None else norm["idx"].size)
    # acceptance gate 2: one running digest per codec over all 1000 iterations
    parts = {"sym16": [], "asym16": [], "pc": [], "outl16": [], "mask": []}
    for x, hot, mask in cases.gate2_inputs():
        for key, (arr, s, g) in {
            "sym16": (x, cases.SYM, 16), "asym16": (x, cases.ASYM, 16),
            "pc": (x, cases.SYM, cases.PER_CHANNEL), "outl16": (hot, cases.OUTL, 16),
            "mask": (mask, cases.MASK, 0),
        }.items():
            norm, deq = run_ref(arr, s, g, 3.0)
            parts[key].append(cases.norm_digest(norm, deq))
    for key, lst in parts.items():
        dig[f"gate2/{key}"] = cases.digest(np.array(lst))
    flagged = []
    for x in cases.gate9_inputs():
        flagged.append(",".join(str(i) for i in ref.detect_outlier_channels(x).tolist()))
    dig["gate9/flagged"] = cases.digest(np.array(flagged))
    (HERE / "digests.json").write_text(json.dumps(dig, indent=1, sort_keys=True) + "\n")
    print(f"digests.json: {len(dig)} entries")


if __name__ == "__main__":
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    small()
    large()
