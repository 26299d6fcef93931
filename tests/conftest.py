"""Shared pytest configuration: the ``gpu`` marker and import paths.

``-m "not gpu"`` runs everywhere (oracle vs golden vectors, host logic, the
C-ABI library's exported symbols, gloo multi-process tests); ``-m gpu`` needs
a B200 and calls the CUDA path through the C-ABI.
"""

import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
for p in (ROOT, ROOT / "tests" / "golden", ROOT / "tests"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _has_cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


REFERENCE_SRC = Path("/root/reference/pkg/src")


@pytest.fixture(scope="session")
def reference_codec():
    """The live reference codec when /root/reference exists (build container only)."""
    if not REFERENCE_SRC.is_dir():
        pytest.skip("reference tree not present (GPU box)")
    sys.dont_write_bytecode = True
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.append(str(REFERENCE_SRC))
    from actplan import codec
    return codec
