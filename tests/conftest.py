"""Shared test setup: the `gpu` marker, repo import path, golden fixtures.

`-m "not gpu"` tests run on CPU only (oracle vs golden vectors, host logic,
C-ABI symbol table); `-m gpu` tests are the parity tests proper and call the
CUDA path through the C ABI.
"""
import json
import sys
from functools import lru_cache
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden" / "golden.json"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libpsim.so")


@lru_cache(maxsize=1)
def golden():
    return json.loads(GOLDEN.read_text())


def cuda_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def gold():
    return golden()
