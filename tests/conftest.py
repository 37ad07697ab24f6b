"""Test configuration: the `gpu` marker and shared golden-fixture loaders.

`pytest -m "not gpu"` runs here (no GPU): oracle-vs-golden pinning, host
planning logic, workspace format, the C ABI's exported symbols.
`pytest -m gpu` runs on a B200: every device result is compared with the
oracle / golden vectors produced by the reference (tests/golden/make_golden.py).
"""

import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (runs on the B200 box)")
    config.addinivalue_line("markers", "slow: long-running (large configs)")


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch
