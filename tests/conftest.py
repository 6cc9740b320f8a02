"""Shared test setup.

* registers the ``gpu`` marker (tests that need a B200 and libmehdg_b200.so);
* builds the C-ABI library in-tree if it is missing (nvcc cross-compiles on
  the CPU-only build box);
* helpers to load the golden fixtures written by tests/golden/make_golden.py.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))

_lib_path = ROOT / "paper_2302_10917_b200" / "libmehdg_b200.so"
if not _lib_path.exists():
    from paper_2302_10917_b200 import _build

    _build.build()


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the CUDA library")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


def golden(name: str):
    p = GOLDEN / name
    if not p.exists():
        pytest.skip(f"golden fixture {name} missing")
    return np.load(p, allow_pickle=False)


def has_gpu() -> bool:
    from paper_2302_10917_b200 import _lib

    return _lib.device_count() > 0


def rel(a, b) -> float:
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    den = max(np.linalg.norm(b), 1e-300)
    return float(np.linalg.norm(a - b) / den)


@pytest.fixture(scope="session")
def gpu():
    if not has_gpu():
        pytest.skip("no CUDA device")
    import torch

    torch.cuda.init()
    return 0


@pytest.fixture(params=["default", "cta", "pipe"])
def lu_kernel(request, monkeypatch):
    """The default batched LU, the CTA-resident one (csrc/lu_cta.cu, 32 < Q <= 168) and
    the pipelined one (csrc/lu_pipe.cu, 32 < Q <= 224; blocks that need row exchanges
    come back through the default kernel), chosen by MEHDG_LU when a system is
    factorized."""
    if request.param != "default":
        monkeypatch.setenv("MEHDG_LU", request.param)
    return request.param
