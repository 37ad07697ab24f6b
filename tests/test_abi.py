"""The C ABI library loads and exports every symbol include/polydet_b200.h
declares (CPU only: no compute calls)."""

import ctypes
import re

from helpers import ROOT
from paper_2010_12117_b200 import native


def _declared():
    text = (ROOT / "include" / "polydet_b200.h").read_text()
    return sorted(set(re.findall(r"\b(pdb_\w+)\s*\(", text)))


def test_header_and_binding_agree():
    assert _declared() == native.exported_symbols()


def test_library_exports_every_declared_symbol():
    lib = native.load_library()
    for name in _declared():
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr), name
    assert lib.pdb_version() == 1
    assert lib.pdb_crt_limbs(23) == (31 * 23 + 31) // 32 + 1
    assert lib.pdb_det_scratch_bytes(40, 1024) > 1024 * 8


def test_no_cpu_fallback_without_gpu():
    import pytest
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2010_12117_b200 import DeviceError, det_grid, find_fourier_primes
    import numpy as np

    spec = find_fourier_primes(4, 1, start=97, min_count=1)[0]
    with pytest.raises(DeviceError):
        det_grid([np.array([1, 2])], 1, spec)
