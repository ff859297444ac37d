"""Shared test configuration.

Markers:
  gpu  -- needs a B200 (run by the driver with ``-m gpu`` on a GPU box).
Everything unmarked runs on CPU here (``-m "not gpu"``).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent
GOLDEN = REPO / "tests" / "golden"
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def digests():
    return json.loads((GOLDEN / "digests.json").read_text())


@pytest.fixture(scope="session")
def small_cases():
    raw = np.load(GOLDEN / "small_cases.npz")
    cases: dict = {}
    for key in raw.files:
        name, field = key.split("/", 1)
        cases.setdefault(name, {})[field] = raw[key]
    return cases


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as orc
    orc.build()
    return orc


def cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False
