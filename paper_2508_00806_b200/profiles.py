"""Boundary types shared with the host planner.

``LayerKind`` selects the compressor (reference profiles.py:24-34 with
codec.py:72-82).  ``OperatorProfile`` / ``ModelProfile`` are the records the
GPU profiler emits; their JSON form is field-for-field the reference schema
(profiles.py:37-55, 202-223, unknown fields rejected as in :134-140) so the
reference's ``load_profile`` -> ``solve`` consumes our measured profiles
unchanged.  Only what the compressor path needs lives here; the planner,
simulator and CLI stay in the reference.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass
from enum import Enum
from pathlib import Path

from .errors import ParseError, ValidationError


class LayerKind(str, Enum):
    """Operator family that produced an activation (profiles.py:24-34)."""

    LINEAR = "linear"
    LAYER_NORM = "layer_norm"
    GELU = "gelu"
    QKV_MATRIX = "qkv_matrix"
    SOFTMAX = "softmax"
    SCORE = "score"
    DROPOUT_MASK = "dropout_mask"
    OTHER = "other"


OPERATOR_KEYS = (
    "id", "name", "kind", "mem_bytes", "compute_time_ms",
    "compress_time_ms", "decompress_time_ms", "compression_rate",
)
PROFILE_KEYS = (
    "n_layers", "static_mem_bytes", "mem_budget_bytes",
    "reference_batch", "base_step_time_ms", "operators",
)


def _check_keys(raw: dict, keys: tuple, what: str) -> None:
    missing = [k for k in keys if k not in raw]
    extra = [k for k in raw if k not in keys]
    if missing:
        raise ParseError(f"{what}: missing fields {missing}")
    if extra:
        raise ParseError(f"{what}: unknown fields {extra}")


@dataclass(frozen=True)
class OperatorProfile:
    """One activation tensor of the block (profiles.py:58-88)."""

    id: int
    name: str
    kind: LayerKind
    mem_bytes: int
    compute_time_ms: float
    compress_time_ms: float
    decompress_time_ms: float
    compression_rate: float

    def __post_init__(self) -> None:
        if isinstance(self.mem_bytes, bool) or not isinstance(self.mem_bytes, int) or self.mem_bytes <= 0:
            raise ValidationError(f"operator {self.id}: mem_bytes must be a positive integer")
        for key in ("compute_time_ms", "compress_time_ms", "decompress_time_ms"):
            v = getattr(self, key)
            if not math.isfinite(v) or v < 0:
                raise ValidationError(f"operator {self.id}: {key} must be finite and >= 0, got {v}")
        if not 0.0 < self.compression_rate <= 1.0:
            raise ValidationError(f"operator {self.id}: compression_rate must be in (0, 1]")

    def to_dict(self) -> dict:
        return {
            "id": self.id, "name": self.name, "kind": self.kind.value,
            "mem_bytes": self.mem_bytes, "compute_time_ms": self.compute_time_ms,
            "compress_time_ms": self.compress_time_ms,
            "decompress_time_ms": self.decompress_time_ms,
            "compression_rate": self.compression_rate,
        }

    @classmethod
    def from_dict(cls, raw: dict) -> "OperatorProfile":
        if not isinstance(raw, dict):
            raise ParseError("operator entry must be an object")
        _check_keys(raw, OPERATOR_KEYS, "operator")
        try:
            kind = LayerKind(raw["kind"])
        except ValueError:
            raise ParseError(f"operator {raw['id']}: unknown kind {raw['kind']!r}") from None
        return cls(int(raw["id"]), str(raw["name"]), kind, raw["mem_bytes"],
                   float(raw["compute_time_ms"]), float(raw["compress_time_ms"]),
                   float(raw["decompress_time_ms"]), float(raw["compression_rate"]))


@dataclass(frozen=True)
class ModelProfile:
    """A profiled block plus model-level context (profiles.py:91-131)."""

    operators: tuple
    n_layers: int
    static_mem_bytes: int
    mem_budget_bytes: int
    reference_batch: int
    base_step_time_ms: float

    def __post_init__(self) -> None:
        if not self.operators:
            raise ValidationError("operators must be non-empty")
        ids = [op.id for op in self.operators]
        if ids != list(range(1, len(ids) + 1)):
            raise ValidationError(f"operator ids must be contiguous 1..N in order, got {ids}")
        if self.mem_budget_bytes <= self.static_mem_bytes:
            raise ValidationError("mem_budget_bytes must exceed static_mem_bytes")
        if self.reference_batch < 1 or self.n_layers < 1 or self.base_step_time_ms <= 0:
            raise ValidationError("n_layers, reference_batch and base_step_time_ms must be positive")

    @property
    def n_operators(self) -> int:
        return len(self.operators)

    def to_dict(self) -> dict:
        return {
            "n_layers": self.n_layers, "static_mem_bytes": self.static_mem_bytes,
            "mem_budget_bytes": self.mem_budget_bytes,
            "reference_batch": self.reference_batch,
            "base_step_time_ms": self.base_step_time_ms,
            "operators": [op.to_dict() for op in self.operators],
        }

    @classmethod
    def from_dict(cls, raw: dict) -> "ModelProfile":
        if not isinstance(raw, dict):
            raise ParseError("profile must be an object")
        _check_keys(raw, PROFILE_KEYS, "profile")
        ops = tuple(OperatorProfile.from_dict(o) for o in raw["operators"])
        return cls(ops, raw["n_layers"], raw["static_mem_bytes"], raw["mem_budget_bytes"],
                   raw["reference_batch"], float(raw["base_step_time_ms"]))


def save_profile(profile: ModelProfile, path) -> None:
    Path(path).write_text(json.dumps(profile.to_dict(), indent=2) + "\n")


def load_profile(path) -> ModelProfile:
    try:
        raw = json.loads(Path(path).read_text())
    except (OSError, json.JSONDecodeError) as exc:
        raise ParseError(f"cannot read profile {path}: {exc}") from exc
    return ModelProfile.from_dict(raw)
