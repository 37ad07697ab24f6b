"""Synthetic inputs for the five BASELINE.json configurations (host side).

Recipes follow SURVEY.md §8(d) (one fresh `random.Random(seed)` per matrix;
dense entries draw every monomial with per-variable exponent <= d in
`itertools.product` order; rows are generated row-major).  The plan digests
these produce are pinned against the reference in tests/golden.

* C1: 4x4, bivariate, degree <= 2, coeffs U[-7,7], seed 1, one 31-bit prime
      (PipelineConfig(prime_start=2**30, min_primes=1)).
* C2: Sylvester matrix (w.r.t. x) of two random bivariate polynomials of total
      degree 8, coeffs U[-100,100] (or U[-2^31,2^31]), seed 2.
* C3: 16x16, 3 variables, degree <= 3, coeffs U[-2^32,2^32], seed 3.
* C4: harmonic-elimination resultants, deterministic.
* C5: 40x40, 3 variables, degree <= 4, coeffs U[-100,100], seed 5.
"""

from __future__ import annotations

import itertools
import random

from .layout import poly_matrix
from .planner import PipelineConfig
from .resultant import sylvester

NAMES = ("x", "y", "z", "w")


def dense_matrix(r: int, vn: int, d: int, lo: int, hi: int, seed: int):
    """r x r matrix of dense polynomials (every monomial with exponents <= d)."""
    rng = random.Random(seed)
    monomials = list(itertools.product(range(d + 1), repeat=vn))

    def entry():
        return {e: rng.randint(lo, hi) for e in monomials}

    rows = [[entry() for _ in range(r)] for _ in range(r)]
    return poly_matrix(rows, NAMES[:vn])


def c1():
    return dense_matrix(4, 2, 2, -7, 7, 1), PipelineConfig(prime_start=2**30, min_primes=1)


def c2(wide: bool = False):
    bound = 2**31 if wide else 100
    rng = random.Random(2)

    def poly():
        return {(i, j): rng.randint(-bound, bound) for i in range(9) for j in range(9 - i)}

    f, g = poly(), poly()
    for h in (f, g):
        while h[(8, 0)] == 0:
            h[(8, 0)] = rng.randint(-bound, bound)
    return sylvester(f, g, ("x", "y"), "x"), PipelineConfig()


def c3():
    return dense_matrix(16, 3, 3, -2**32, 2**32, 3), PipelineConfig()


def c5(min_primes: int = 2):
    return dense_matrix(40, 3, 4, -100, 100, 5), PipelineConfig(min_primes=min_primes)


# -- harmonic elimination (C4) -------------------------------------------------

def _padd(a, b):
    out = dict(a)
    for e, c in b.items():
        out[e] = out.get(e, 0) + c
    return {e: c for e, c in out.items() if c}


def _pscale(a, s):
    return {e: c * s for e, c in a.items() if c * s}


def _pmul(a, b):
    out: dict = {}
    for ea, ca in a.items():
        for eb, cb in b.items():
            e = tuple(x + y for x, y in zip(ea, eb))
            out[e] = out.get(e, 0) + ca * cb
    return {e: c for e, c in out.items() if c}


def _chebyshev(k: int, x: dict, nv: int):
    """T_k(x) for a polynomial x: T0 = 1, T1 = x, T_{n+1} = 2x T_n - T_{n-1}."""
    one = {(0,) * nv: 1}
    prev, cur = one, x
    if k == 0:
        return one
    for _ in range(k - 1):
        prev, cur = cur, _padd(_pscale(_pmul(x, cur), 2), _pscale(prev, -1))
    return cur


def harmonic(sources: int, pair=(5, 7), symbolic_m: bool = True):
    """Res_{x_{s-1}}(E_k1, E_k2) of the selective-harmonic-elimination system.

    Variables x_1..x_{s-1} (+ m when symbolic); x_s is eliminated through the
    k = 1 equation, x_s = (-1)^(s+1) (m - sum_i (-1)^(i+1) x_i); then
    E_k = sum_i (-1)^(i+1) T_k(x_i) + (-1)^(s+1) T_k(x_s) for k in `pair`.
    """
    s = sources
    names = tuple("x%d" % i for i in range(1, s)) + (("m",) if symbolic_m else ())
    nv = len(names)

    def var(i):
        e = [0] * nv
        e[i] = 1
        return {tuple(e): 1}

    ell: dict = {}
    for i in range(1, s):
        ell = _padd(ell, _pscale(var(i - 1), (-1) ** (i + 1)))
    m_poly = var(nv - 1) if symbolic_m else {(0,) * nv: 1}
    x_last = _pscale(_padd(m_poly, _pscale(ell, -1)), (-1) ** (s + 1))

    def equation(k):
        acc: dict = {}
        for i in range(1, s):
            acc = _padd(acc, _pscale(_chebyshev(k, var(i - 1), nv), (-1) ** (i + 1)))
        return _padd(acc, _pscale(_chebyshev(k, x_last, nv), (-1) ** (s + 1)))

    return sylvester(equation(pair[0]), equation(pair[1]), names, "x%d" % (s - 1)), PipelineConfig()
