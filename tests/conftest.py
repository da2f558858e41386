"""Test configuration: the `gpu` marker and shared fixtures.

`-m "not gpu"` runs here on CPU (oracle vs golden vectors, host logic, ABI
symbol checks, gloo world-2 tests); `-m gpu` runs on a B200 and calls the
CUDA library through its C-ABI."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLD = os.path.join(ROOT, "tests", "golden")
DATA = os.path.join(ROOT, "paper_2210_02023_b200", "data")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")


@pytest.fixture(scope="session")
def pools():
    with open(os.path.join(DATA, "pools.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def ckpt_path():
    return os.path.join(DATA, "dreamshard_m50_d4.dshd")


@pytest.fixture(scope="session")
def ckpt_path_d8():
    return os.path.join(DATA, "dreamshard_m100_d8.dshd")


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
