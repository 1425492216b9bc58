"""Shared test setup.

`-m gpu` tests need a B200 and the built CUDA library; everything else runs on
CPU (oracle vs golden vectors, host protocol logic, C-ABI symbol table, gloo
multi-process tests).
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libpetals_b200.so")
    config.addinivalue_line("markers", "slow: long-running (large shapes)")


def load_golden(name: str):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False)


@pytest.fixture(scope="session")
def golden():
    return load_golden


def has_cuda() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False


def pytest_collection_modifyitems(config, items):
    # a gpu-marked test on a box without CUDA is an error, not a skip: the
    # driver runs `-m gpu` only on B200 boxes, and a silent skip would hide a
    # missing device.
    pass
