"""Host-side logic (CPU): planning decisions and digests, prime selection,
tensor layout, workspace format, matrix builders.  The planner must reproduce
the reference's Plan digests bit for bit (they key checkpoints and fix every
evaluation point)."""

import math
import random

import numpy as np
import pytest

from helpers import golden
import naive
from paper_2010_12117_b200 import (
    CoeffTensor,
    CorruptWorkspaceError,
    PipelineConfig,
    PlanningError,
    PrimeSpec,
    StaleWorkspaceError,
    Workspace,
    build_basis,
    census,
    coefficient_bound,
    decode_array,
    degree_bound,
    digest_of,
    encode,
    encode_array,
    find_fourier_primes,
    find_root_of_order,
    horner_lift,
    is_prime,
    pad_shape,
    pad_to,
    plan,
    poly_matrix,
    reduce_mod,
    signed_lift,
    sylvester,
    tensor_from_terms,
)


def test_plan_digests_match_reference_configs():
    from paper_2010_12117_b200 import workloads

    gold = golden("plans.json")
    builders = {"C1": workloads.c1, "C2": workloads.c2, "C2w": lambda: workloads.c2(True),
                "C3": workloads.c3, "C5": workloads.c5,
                "C4_3src_T5T7_m": lambda: workloads.harmonic(3, (5, 7), True),
                "C4_4src_T5T11_m": lambda: workloads.harmonic(4, (5, 11), True)}
    for name, build in builders.items():
        m, cfg = build()
        pl = plan(m, cfg)
        assert pl.digest() == gold[name]["digest"], name
        assert pl.to_dict() == gold[name]["plan"], name
        assert digest_of(m.to_dict()) == gold[name]["input_digest"], name


def test_prime_search_known_answers():
    g = golden("primes.json")
    assert find_root_of_order(17, 16) == g["root_17_16"] == 3
    assert find_root_of_order(2013265921, 2**27) == g["root_2013265921_2^27"]
    quad = lambda specs: [[s.p, s.c, s.q, s.omega] for s in specs]
    assert quad(find_fourier_primes(6, 1, 10**9, min_count=3)) == g["q6_first3"]
    assert quad(find_fourier_primes(8, 1, 10**9, min_count=3)) == g["q8_first3"]
    assert [s.p for s in find_fourier_primes(0, 1, 2, min_count=2)] == g["q0_small"] == [2, 3]
    assert [s.p for s in find_fourier_primes(0, 1, 10**9, min_count=2)] == g["q0_big"]
    assert [s.p for s in find_fourier_primes(30, 1, 2, min_count=1)] == g["q30"] == [3221225473]
    assert quad(find_fourier_primes(27, 1, 2 * 10**9, min_count=1)) == g["q27_2e9"]
    assert quad(find_fourier_primes(26, 1, 1800000000, min_count=1)) == g["q26_start"]
    got = census((64, 128, 256, 512, 4096, 8192, 65536), 2000).counts
    assert {str(k): v for k, v in got.items()} == g["census"]


def test_primality_against_trial_division():
    def trial(n):
        return n >= 2 and all(n % d for d in range(2, int(n ** 0.5) + 1))

    assert [n for n in range(3000) if is_prime(n)] == [n for n in range(3000) if trial(n)]
    assert not is_prime(561) and not is_prime(3215031751)
    assert is_prime(2**61 - 1)


def test_prime_spec_validation():
    PrimeSpec(97, 3, 5, find_root_of_order(97, 32))
    with pytest.raises(ValueError):
        PrimeSpec(97, 3, 5, 1)
    with pytest.raises(ValueError):
        PrimeSpec(91, 45, 1, 90)
    with pytest.raises(PlanningError, match="insufficient primes"):
        find_fourier_primes(20, 10**100, 10**9, scan_limit=5)


def test_tensor_layout_known_answers():
    t = encode({(0, 0): 1, (0, 2): 5, (1, 0): 2, (1, 1): 3, (2, 0): 4}, (3, 3), ("x", "y"))
    assert list(t.coeffs) == [1, 0, 5, 2, 3, 0, 4, 0, 0]
    assert pad_shape((16, 8, 10)) == ((16, 8, 16), 4)
    assert pad_shape((15, 7, 9)) == ((16, 8, 16), 4)
    z = tensor_from_terms({}, ("x", "y"))
    assert z.shape == (1, 1) and z.coeffs == (0,)
    assert pad_to(tensor_from_terms({(1,): 3}, ("x",)), (4,)).coeffs == (0, 3, 0, 0)
    with pytest.raises(ValueError, match="degree overflow"):
        encode({(3,): 1}, (2,), ("x",))
    spec = find_fourier_primes(4, 1, start=97, min_count=1)[0]
    assert reduce_mod(CoeffTensor((3,), (-1, 98, 5), ("x",)), spec).residues.tolist() == [96, 1, 5]


def test_poly_matrix_dedup_and_bounds():
    a = {(1,): 1, (0,): 1}
    m = poly_matrix([[a, dict(a)], [{}, {(3,): 2}]], ("x",))
    assert m.k == 3 and m.entry_ids == (0, 0, 1, 2)
    assert degree_bound(m) == (4,)
    assert coefficient_bound(m) == 2 * 2 * 2
    rng = random.Random(5)
    for _ in range(15):
        rows = naive.random_poly_matrix(rng, 3, 2, 2, 9, 4)
        mm = poly_matrix(rows, ("x", "y"))
        det = naive.symbolic_det(rows, 2)
        assert coefficient_bound(mm) >= max((abs(c) for c in det.values()), default=0)
        assert all(all(e <= b for e, b in zip(ex, degree_bound(mm))) for ex in det)


def test_sylvester_structure():
    m = sylvester({(2,): 1, (0,): 1}, {(1,): 1, (0,): 1}, ("x",), "x")
    assert m.r == 3 and m.variables == ()
    with pytest.raises(ValueError, match="no eliminand"):
        sylvester({(0, 1): 1}, {(0, 2): 1}, ("x", "y"), "x")
    f = {(4, 0, 0): 1, (1, 1, 0): 1, (0, 0, 1): 1}
    g = {(4, 0, 0): 1, (2, 0, 1): 1, (0, 1, 0): 1}
    m = sylvester(f, g, ("x", "u", "v"), "x")
    assert m.r == 8 and m.k < 64


def test_artifact_codec_and_workspace_format(tmp_path):
    blob = encode_array([1, 2, 3, 2**61], (2, 2))
    vals, shape = decode_array(blob)
    assert vals.tolist() == [1, 2, 3, 2**61] and shape == (2, 2)
    with pytest.raises(CorruptWorkspaceError, match="bad artifact magic"):
        decode_array(b"NOTMAGIC" + blob[8:])
    with pytest.raises(CorruptWorkspaceError, match="truncated"):
        decode_array(blob[:-1])
    ws = Workspace(tmp_path / "w")
    ws.create({"input_sha256": "a", "plan_sha256": "b"})
    ws.store_array("p0/det", [5, 6], (2,))
    ws.store_residues("p0/ifft", np.array([7, 8], dtype=np.uint32), (2,))
    ws.store_json("crt", {"coeffs": [1]})
    assert (tmp_path / "w" / "p0_det.bin").read_bytes() == encode_array([5, 6], (2,))
    assert (tmp_path / "w" / "p0_ifft.bin").read_bytes() == encode_array([7, 8], (2,))
    with open(tmp_path / "w" / "manifest", "ab") as fh:
        fh.write(b'{"kind": "done", "unit": "p1/det", "artif')     # torn append
    again = Workspace(tmp_path / "w")
    assert again.open() == {"input_sha256": "a", "plan_sha256": "b"}
    again.verify()
    assert again.has("crt") and not again.has("p1/det")
    (tmp_path / "w" / "p0_det.bin").write_bytes(b"POLYDET\x00" + b"\x00" * 30)
    with pytest.raises(CorruptWorkspaceError, match="checkpoint invalid"):
        again.verify()
    with pytest.raises(StaleWorkspaceError, match="stale workspace"):
        Workspace(tmp_path / "missing").open()


def test_workspace_bytes_match_reference_run():
    """Named files and manifest lines the reference wrote for a small run:
    the planner/layout must regenerate the same input/plan JSON bytes."""
    from paper_2010_12117_b200 import PolyMatrix, stable_json
    import hashlib

    g = golden("workspace.json")
    m = PolyMatrix.from_dict(g["input"])
    pl = plan(m)
    assert hashlib.sha256(stable_json(m.to_dict())).hexdigest() == g["files"]["input.json"]
    assert hashlib.sha256(stable_json(pl.to_dict())).hexdigest() == g["files"]["plan.json"]
    header = {"kind": "header", "input_sha256": digest_of(m.to_dict()), "plan_sha256": pl.digest()}
    assert stable_json(header).decode() == g["manifest"][0]


def test_crt_host_helpers():
    basis = build_basis([3, 5, 7])
    assert basis.weights == (1, 3, 15) and basis.inverses[1] == 2 and basis.inverses[2] == 1
    assert horner_lift([2, 2, 1], basis) == 2 + 2 * 3 + 15 == 23
    assert naive.exhaustive_crt([2, 3, 2], [3, 5, 7]) == 23
    assert signed_lift(104, 105) == -1 and signed_lift(52, 105) == 52 and signed_lift(53, 105) == -52
    with pytest.raises(ValueError):
        signed_lift(105, 105)
    with pytest.raises(ValueError, match="duplicate"):
        build_basis([3, 5, 3])


def test_native_ints_from_limbs_matches_python_path():
    """_pdb_host (csrc/host_ints.cpp) builds the same Python ints as the
    reference-style per-coefficient from_bytes path, for any limb width."""
    from paper_2010_12117_b200 import native
    from paper_2010_12117_b200.crt import limbs_to_ints
    h = native.host_module()
    rng = np.random.default_rng(7)
    n = 5000
    for L in (1, 2, 3, 9, 74, 75):   # <= 74 limbs: direct digit fill; wider: from_bytes fallback
        limbs = np.zeros((n, L), dtype=np.uint32)
        nz = np.sort(rng.choice(n, 1700, replace=False))
        for i in nz:
            w = int(rng.integers(1, L + 1))
            limbs[i, :w] = rng.integers(0, 2**32, w, dtype=np.uint32)
        limbs[nz[:3]] = 0xFFFFFFFF                     # widest magnitudes
        neg = rng.integers(0, 2, n).astype(np.uint8)
        want = limbs_to_ints(limbs, neg)
        keep = np.flatnonzero(limbs.any(axis=1))
        got = h.ints_from_limbs(limbs[keep].tobytes(), keep.astype(np.int64).tobytes(), neg[keep].tobytes(), n, L)
        assert type(got) is tuple and list(got) == want
        shuffled = rng.permutation(keep)                 # unsorted indices take the second loop
        got2 = h.ints_from_limbs(limbs[shuffled].tobytes(), shuffled.astype(np.int64).tobytes(),
                                 neg[shuffled].tobytes(), n, L)
        assert got2 == got
        assert all(type(v) is int for v in got)
        zero = 0
        assert all(v is zero for v in got if v == 0)   # small ints stay the shared singletons
    with pytest.raises(ValueError):
        h.ints_from_limbs(b"\0" * 8, np.zeros(1, np.int64).tobytes(), b"\0", 4, 1)
    with pytest.raises(IndexError):
        h.ints_from_limbs(b"\1\0\0\0", np.array([9], np.int64).tobytes(), b"\0", 4, 1)


def test_predicted_total_reference_arithmetic():
    """Reference test_pipeline.py:205-209 and acceptance criterion 2 (2088.96)."""
    from paper_2010_12117_b200 import predicted_total
    assert predicted_total(6, 16, 256, 1.36) == 2088.96
    assert predicted_total(3, 4, 1, 0.5) == 1.5
    assert predicted_total(2, 2, 4, 1.005) == pytest.approx(2 * 4 * 1.01)
    with pytest.raises(ValueError):
        predicted_total(1, 2, 5, 1.0)


REFERENCE_IMPORTS = {   # every name the reference's own tests import from each submodule
    "pipeline": ["PipelineConfig", "coefficient_bound", "degree_bound", "plan", "predict", "predicted_total",
                 "resume", "run", "run_report"],
    "tensor": ["CoeffTensor", "DegreeVector", "ModTensor", "PolyMatrix", "axis_rotate", "encode", "normalize_terms",
               "pad_shape", "pad_to", "poly_matrix", "reduce_mod", "tensor_from_terms"],
    "modular": ["MODULUS_LIMIT", "PrimeSpec", "add_mod", "census", "find_fourier_primes", "find_root_of_order",
                "inv_mod", "is_prime", "mul_mod", "pow_mod", "sub_mod"],
    "workspace": ["Workspace", "decode_array", "encode_array"],
    "transform": ["TwiddleTable", "ntt_forward_1d", "ntt_forward_multi", "ntt_inverse_1d", "ntt_inverse_multi"],
    "determinant": ["ModMatrix", "condense", "det_grid", "det_mod"],
    "crt": ["build_basis", "combine_tensor", "horner_lift", "mrc_digits", "signed_lift"],
    "resultant": ["sylvester"],
    "errors": ["CorruptWorkspaceError", "ParseError", "PlanningError", "StaleWorkspaceError"],
}


def test_reference_module_names_resolve():
    """`polydet.<module>.<name>` imports of the reference's tests resolve here too."""
    import importlib
    for mod, names in REFERENCE_IMPORTS.items():
        m = importlib.import_module("paper_2010_12117_b200." + mod)
        missing = [n for n in names if not hasattr(m, n)]
        assert not missing, (mod, missing)


def test_reference_error_messages_before_any_device_work():
    """The reference's tests match these message substrings (test_determinant.py:188-192,
    test_crt.py:155-161, test_tensor.py:182-185, test_modular.py:59, 105-107); here they
    are raised by host-side validation, before any kernel runs."""
    from paper_2010_12117_b200 import (ModTensor, combine_tensor, det_grid, find_fourier_primes,
                                       find_root_of_order, inv_mod, poly_matrix)
    spec = find_fourier_primes(5, 1, start=97, min_count=1)[0]
    a, b = np.zeros(4, dtype=np.int64), np.zeros(5, dtype=np.int64)
    with pytest.raises(ValueError, match="share one shape"):
        det_grid([a, b, a, b], 2, spec)
    with pytest.raises(ValueError, match="need 4 entry ids"):
        det_grid([a, a], 2, spec, entry_ids=[0, 1, 1])
    with pytest.raises(ValueError, match="missing grid"):
        det_grid([a, a], 2, spec, entry_ids=[0, 1, 2, 0])
    s1, s2 = find_fourier_primes(3, 2, start=10**9, min_count=2)
    t1 = ModTensor((2,), np.array([1, 2], dtype=np.int64), s1, ("x",))
    t2 = ModTensor((4,), np.array([1, 2, 3, 4], dtype=np.int64), s2, ("x",))
    with pytest.raises(ValueError, match="share one shape"):
        combine_tensor([t1, t2])
    with pytest.raises(ValueError, match="at least one residue tensor"):
        combine_tensor([])
    with pytest.raises(ValueError, match="square"):
        poly_matrix([[{}, {}], [{}]], ("x",))
    with pytest.raises(ValueError, match="no inverse"):
        inv_mod(0, 97)
    with pytest.raises(ValueError, match="order unavailable"):
        find_root_of_order(97, 64)
