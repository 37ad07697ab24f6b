"""Sylvester matrices (host-side matrix builder, reference `resultant.py:15-58`).

Not a kernel: it produces the polynomial matrices of configs C2 and C4,
whose shifted-row structure de-duplicates to k << r^2 unique entries.
"""

from __future__ import annotations

from .layout import normalize_terms, poly_matrix


def _coefficients_in(terms: dict, axis: int) -> dict:
    """{power of the eliminated variable: polynomial in the other variables}."""
    parts: dict = {}
    for exps, c in terms.items():
        rest = exps[:axis] + exps[axis + 1:]
        bucket = parts.setdefault(exps[axis], {})
        bucket[rest] = bucket.get(rest, 0) + c
    cleaned = {j: normalize_terms(b) for j, b in parts.items()}
    return {j: b for j, b in cleaned.items() if b}


def sylvester(f, g, variables, var: str):
    """(m+n) x (m+n) Sylvester matrix of f (degree m in var) and g (degree n)."""
    variables = tuple(variables)
    if var not in variables:
        raise ValueError("unknown variable %r" % (var,))
    axis = variables.index(var)
    fc = _coefficients_in(normalize_terms(f), axis)
    gc = _coefficients_in(normalize_terms(g), axis)
    m = max(fc, default=0)
    n = max(gc, default=0)
    if m == 0 and n == 0:
        raise ValueError("no eliminand: neither polynomial involves %r" % (var,))
    size = m + n

    def band(coeffs, degree, shifts):
        out = []
        for shift in range(shifts):
            row = [{} for _ in range(size)]
            for t in range(degree + 1):
                row[shift + t] = coeffs.get(degree - t, {})
            out.append(row)
        return out

    rows = band(fc, m, n) + band(gc, n, m)
    return poly_matrix(rows, variables[:axis] + variables[axis + 1:])
