"""Independent naive checkers for the tests (no shared code with the package
or the oracle): O(N^2) DFTs, cofactor determinants, term-dict polynomial
algebra with a symbolic determinant, exhaustive CRT."""

from __future__ import annotations

import math
import random
from functools import lru_cache


def dft(vec, w, p):
    n = len(vec)
    return [sum(v * pow(w, j * k, p) for j, v in enumerate(vec)) % p for k in range(n)]


def idft(vec, w, p):
    n = len(vec)
    wi, ni = pow(w, -1, p), pow(n, -1, p)
    return [sum(v * pow(wi, j * k, p) for j, v in enumerate(vec)) * ni % p for k in range(n)]


def cofactor_det(rows, p=None):
    n = len(rows)
    if n == 0:
        return 1
    total = 0
    for j, a in enumerate(rows[0]):
        if a:
            minor = [row[:j] + row[j + 1:] for row in rows[1:]]
            total += (-1) ** j * a * cofactor_det(minor)
    return total % p if p is not None else total


def poly_add(a, b, sign=1):
    out = dict(a)
    for e, c in b.items():
        out[e] = out.get(e, 0) + sign * c
    return {e: c for e, c in out.items() if c}


def poly_mul(a, b):
    out = {}
    for ea, ca in a.items():
        for eb, cb in b.items():
            e = tuple(x + y for x, y in zip(ea, eb))
            out[e] = out.get(e, 0) + ca * cb
    return {e: c for e, c in out.items() if c}


def poly_eval(terms, point, p):
    """sum_terms c * prod x_i^e_i mod p (power tables per coordinate)."""
    if not terms:
        return 0
    tops = [max(e[i] for e in terms) for i in range(len(point))]
    tables = []
    for x, top in zip(point, tops):
        row = [1 % p] * (top + 1)
        for k in range(1, top + 1):
            row[k] = row[k - 1] * x % p
        tables.append(row)
    total = 0
    for exps, c in terms.items():
        v = c % p
        for t, e in zip(tables, exps):
            v = v * t[e] % p
        total += v
    return total % p


def symbolic_det(entries, nvars):
    """Laplace expansion along rows, memoised on the set of remaining columns."""
    r = len(entries)
    one = {(0,) * nvars: 1}

    @lru_cache(maxsize=None)
    def minor(row, cols):
        if row == r:
            return tuple(one.items())
        acc, sign = {}, 1
        for j in range(r):
            if cols >> j & 1:
                cell = entries[row][j]
                if cell:
                    sub = dict(minor(row + 1, cols & ~(1 << j)))
                    acc = poly_add(acc, poly_mul(cell, sub), sign)
                sign = -sign
        return tuple(acc.items())

    return dict(minor(0, (1 << r) - 1))


def exhaustive_crt(residues, primes):
    P = math.prod(primes)
    return next(x for x in range(P) if all(x % p == r for r, p in zip(residues, primes)))


def random_poly(rng: random.Random, vn, deg, bound, terms):
    out = {}
    for _ in range(rng.randint(0, terms)):
        e = tuple(rng.randint(0, deg) for _ in range(vn))
        out[e] = out.get(e, 0) + rng.randint(-bound, bound)
    return {e: c for e, c in out.items() if c}


def random_poly_matrix(rng, r, vn, deg, bound, terms, dup=0.2):
    made, rows = [], []
    for _ in range(r):
        row = []
        for _ in range(r):
            if made and rng.random() < dup:
                row.append(dict(rng.choice(made)))
            else:
                cell = random_poly(rng, vn, deg, bound, terms)
                made.append(cell)
                row.append(cell)
        rows.append(row)
    return rows
