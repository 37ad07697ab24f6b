"""The native host module (_pdb_host, csrc/host_ints.cpp) that turns the GPU
CRT's limb rows into Python ints: the direct-PyLong path (CPython 3.12/3.13)
and the portable public-API path (any other interpreter) must agree with
int.from_bytes on every magnitude and sign (CPU test)."""

import random

import numpy as np
import pytest

from paper_2010_12117_b200 import native


@pytest.mark.parametrize("width", [1, 2, 3, 15, 24, 80])
@pytest.mark.parametrize("ordered", [True, False])
def test_both_paths_equal_int_from_bytes(width, ordered):
    host = native.host_module()
    rng = random.Random(width)
    n = 2000
    idx = sorted(rng.sample(range(n), 500))
    if not ordered:
        rng.shuffle(idx)
    bits = [rng.choice([0, 1, 29, 30, 31, 32, 59, 60, 61, 63, 64, 65, 32 * width]) for _ in idx]
    vals = [rng.getrandbits(min(b, 32 * width)) for b in bits]
    limbs = np.frombuffer(b"".join(v.to_bytes(4 * width, "little") for v in vals), dtype="<u4").reshape(-1, width)
    neg = np.array([rng.random() < 0.5 for _ in idx], dtype=np.uint8)
    ix = np.array(idx, dtype=np.int64)
    want = [0] * n
    for i, v, s in zip(idx, vals, neg):
        want[i] = -v if s else v
    assert host.ints_from_limbs(limbs, ix, neg, n, width) == tuple(want)
    assert host.ints_from_limbs_portable(limbs, ix, neg, n, width) == tuple(want)


def test_rejects_inconsistent_buffers():
    host = native.host_module()
    limbs = np.zeros((3, 2), dtype=np.uint32)
    with pytest.raises(ValueError):
        host.ints_from_limbs(limbs, np.arange(2, dtype=np.int64), np.zeros(2, dtype=np.uint8), 5, 2)
    with pytest.raises(IndexError):
        host.ints_from_limbs(limbs, np.array([0, 1, 9], dtype=np.int64), np.zeros(3, dtype=np.uint8), 5, 2)


def test_formatter_portable_build_agrees(tmp_path):
    """format_terms built without the direct-PyLong code (the path on other
    CPython ABIs) prints the same text as the direct build and the oracle,
    including coefficients beyond the direct path's 2400-bit fast case."""
    import importlib.util
    import shutil
    import subprocess
    import sysconfig

    from helpers import ROOT
    from oracle import polydet_oracle as O

    if not shutil.which("g++"):
        pytest.skip("no g++")
    out = tmp_path / ("_pdb_host" + sysconfig.get_config_var("EXT_SUFFIX"))
    subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-DPDB_NO_DIRECT_LONG",
                    "-I" + sysconfig.get_paths()["include"], "-o", str(out),
                    str(ROOT / "paper_2010_12117_b200" / "csrc" / "host_ints.cpp")], check=True)
    spec = importlib.util.spec_from_file_location("_pdb_host", out)
    portable = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(portable)
    assert portable.direct_path() is False
    rng = random.Random(3)
    terms = {(rng.randint(0, 5), rng.randint(0, 5)): rng.choice([1, -1, 0, rng.randint(-2**3000, 2**3000),
                                                                 rng.randint(-99, 99)]) for _ in range(3000)}
    want = O.format_polynomial(terms, ("x", "y"))
    assert portable.format_terms(terms, ("x", "y"), 4) == want
    assert native.host_module().format_terms(terms, ("x", "y"), 4) == want
    dense = [0] * 36
    for (a, b), c in terms.items():
        dense[a * 6 + b] = c
    for mod in (portable, native.host_module()):
        assert mod.format_dense(tuple(dense), (6, 6), ("x", "y"), 4) == want


def test_ints_from_digits_matches_limb_path():
    """The digit-row constructor (rows re-cut on the device by
    pdb_limbs_to_digits30; here cut in Python) builds the same ints as the
    limb-row one."""
    host = native.host_module()
    if not host.direct_path():
        pytest.skip("direct PyLong layout only")
    rng = random.Random(30)
    n, width = 5000, 17
    idx = sorted(rng.sample(range(n), 1200))
    vals = [rng.getrandbits(rng.choice([1, 30, 31, 60, 61, 62, 200, 32 * width])) for _ in idx]
    neg = np.array([rng.random() < 0.5 for _ in idx], dtype=np.uint8)
    D = (32 * width + 29) // 30
    digits = np.array([[(v >> (30 * k)) & ((1 << 30) - 1) for k in range(D)] for v in vals], dtype=np.uint32)
    nd = np.array([(v.bit_length() + 29) // 30 for v in vals], dtype=np.uint8)
    ix = np.array(idx, dtype=np.int64)
    limbs = np.frombuffer(b"".join(v.to_bytes(4 * width, "little") for v in vals), dtype="<u4").reshape(-1, width)
    want = host.ints_from_limbs(limbs, ix, neg, n, width)
    assert host.ints_from_digits(digits, nd, ix, neg, n, D) == want
    with pytest.raises(IndexError):
        host.ints_from_digits(digits, nd, ix[::-1].copy(), neg, n, D)
    # the threaded builder: same tuple for any thread count, canonical small ints,
    # objects that behave (arithmetic, hashing, text) and free cleanly
    for threads in (1, 3, 8):
        got = host.ints_from_digits_mt(digits, nd, ix, neg, n, D, threads)
        assert got == want
    assert all(got[i] is want[i] for i, v in zip(idx, vals) if v.bit_length() <= 60 and -5 <= want[i] <= 256)
    assert {hash(x) for x in got} == {hash(x) for x in want}
    assert [str(got[i]) for i in idx] == [str(want[i]) for i in idx]
    assert sum(got) == sum(want) and sum(x * x for x in got) == sum(x * x for x in want)
    del got
    import gc
    gc.collect()
    with pytest.raises(IndexError):
        host.ints_from_digits_mt(digits, nd, ix[::-1].copy(), neg, n, D, 4)
