"""CPU oracle for the modular-determinant hot path -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference algorithm (arXiv 2010.12117 reference
package `polydet`, read-only at /root/reference/pkg/src/polydet), used as the
checker by `tests/`, by `__graft_entry__.smoke()` and as the CPU baseline
("port") by `bench.py`.  The product (`paper_2010_12117_b200`) never imports
this module.

Parity pinning: every function here is checked against golden vectors that
were produced by importing the reference itself (`tests/golden/make_golden.py`
-> `tests/golden/*.json|npz`, see `tests/test_oracle_golden.py`).

Each function names the reference code it restates:

* `twiddle_row`        transform.py:19-72   (TwiddleTable rows, 1/N scale)
* `ntt_rows`           transform.py:75-92   (batched radix-2 Stockham pass loop)
* `ntt_multi`          transform.py:119-159 (vn rounds: last axis + rotation)
* `det_batch`          determinant.py:136-169 (division-free condensation)
* `det_grid`           determinant.py:92-133  (entry-id gather, chunked, threaded)
* `condense_trail`     determinant.py:57-84   (one matrix: determinant + pivot trail)
* `crt_combine`        crt.py:94-130        (mixed radix digits + Horner + signed lift)
* `reduce_entry`       tensor.py:214-237    (reduce_mod + pad_to of one entry)
* `run_pipeline`       pipeline.py:323-404  (per prime FFT -> DET -> IFFT, then CRT)
* `format_polynomial`  parsing.py:197-225   (canonical result text; tensor.py:25-32 normalisation)

All arithmetic is int64 with p <= 3037000499 (p^2 < 2^63), as on the
reference's fast path (`modular.py:15-19`, `tensor.py:152-154`).
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np

INT64_SAFE = 3037000499


def _check_prime(p):
    if p > INT64_SAFE:
        raise ValueError("oracle handles the int64 path only (p <= 3037000499)")


def root_of_length(p, omega, q, n):
    """omega_N = omega^(2^(q - log2 N))  (transform.py:41-44)."""
    return pow(omega, 1 << (q - (n.bit_length() - 1)), p)


def twiddle_row(p, omega, q, n, inverse=False):
    """(1, w, ..., w^(N/2-1)) for w = omega_N (or its inverse)."""
    w = root_of_length(p, omega, q, n)
    if inverse:
        w = pow(w, -1, p)
    out = np.ones(max(n // 2, 1), dtype=np.int64)
    acc = 1
    for i in range(1, n // 2):
        acc = acc * w % p
        out[i] = acc
    return out


def ntt_rows(rows, powers, p):
    """Natural-order NTT of every row of a (B, N) int64 array.

    Stockham formulation: pass with span s views x as (B, 2, N/(2s), s),
    scales the second half by w^(j * N/(2s)) and writes (a+b, a-b) into the
    (B, N/(2s), 2, s) layout of the next buffer.
    """
    b, n = rows.shape
    x = rows.copy()
    span = 1
    while span < n:
        half = n // (2 * span)
        view = x.reshape(b, 2, half, span)
        tw = powers[0: n // 2: half]
        t = view[:, 1] * tw % p
        y = np.empty((b, half, 2, span), dtype=np.int64)
        y[:, :, 0, :] = (view[:, 0] + t) % p
        y[:, :, 1, :] = (view[:, 0] - t) % p
        x = y.reshape(b, n)
        span *= 2
    return x


def ntt_multi(values, shape, p, omega, q, inverse=False):
    """Multivariate transform of a flat row-major tensor, natural order."""
    _check_prime(p)
    arr = np.asarray(values, dtype=np.int64).reshape(-1).copy()
    shape = tuple(shape)
    if not shape:
        return arr
    cur = shape
    for _ in range(len(shape)):
        n = cur[-1]
        rows = arr.reshape(-1, n)
        rows = ntt_rows(rows, twiddle_row(p, omega, q, n, inverse), p)
        if inverse and n > 1:
            rows = rows * pow(n, -1, p) % p
        arr = np.ascontiguousarray(np.moveaxis(rows.reshape(cur), -1, 0)).reshape(-1)
        cur = (cur[-1],) + cur[:-1]
    return arr


def det_batch(mats, p):
    """Determinant of every matrix in a (count, r, r) int64 stack.

    Step i takes the first nonzero entry z of row i as the pivot, replaces
    every lower row by z*row - t*pivot_row, and finally divides out the
    inflation prod z_i^(r-1-i) and applies the pivot-column permutation sign.
    A node whose row i is all zero gets det 0.
    """
    _check_prime(p)
    work = np.array(mats, dtype=np.int64, copy=True)
    count, r, _ = work.shape
    live = np.ones(count, dtype=bool)
    prod_z = np.ones(count, dtype=np.int64)
    infl = np.ones(count, dtype=np.int64)
    cols = np.zeros((count, r), dtype=np.int64)
    idx = np.arange(count)
    for i in range(r):
        row = work[:, i, :]
        nz = row != 0
        live &= nz.any(axis=1)
        c = np.argmax(nz, axis=1)
        z = np.where(live, row[idx, c], 1)
        cols[:, i] = c
        prod_z = prod_z * z % p
        for _ in range(r - 1 - i):
            infl = infl * z % p
        if i + 1 < r:
            lower = work[:, i + 1:, :]
            t = np.take_along_axis(lower, c[:, None, None], axis=2)
            work[:, i + 1:, :] = (z[:, None, None] * lower % p - t * row[:, None, :] % p) % p
    inv = np.array([pow(int(v), -1, p) for v in infl], dtype=np.int64)
    det = prod_z * inv % p
    swaps = np.zeros(count, dtype=np.int64)
    for a in range(r):
        for b in range(a + 1, r):
            swaps += cols[:, a] > cols[:, b]
    det = np.where(swaps % 2 == 1, (p - det) % p, det)
    return np.where(live, det, 0)


def condense_trail(rows, p):
    """(det, [(step, pivot value, pivot column, flips_sign)]) of one matrix,
    the reference's condensation with its pivot trail (pure Python ints; the
    trail stops at the first all-zero row, det 0)."""
    r = len(rows)
    work = [[int(v) % p for v in row] for row in rows]
    records, columns = [], []
    for i in range(r):
        row = work[i]
        col = next((j for j, v in enumerate(row) if v), None)
        if col is None:
            return 0, records
        z = row[col]
        flips = sum(1 for c in columns if c > col) % 2 == 1
        records.append((i, z, col, flips))
        columns.append(col)
        for jj in range(i + 1, r):
            t = work[jj][col]
            work[jj] = [(z * a - t * b) % p for a, b in zip(work[jj], row)]
    scale, infl = 1, 1
    for i, (_, z, _, _) in enumerate(records):
        scale = scale * z % p
        infl = infl * pow(z, r - 1 - i, p) % p
    det = scale * pow(infl, -1, p) % p
    if sum(f for *_, f in records) % 2:
        det = (p - det) % p
    return det, records


def det_grid(grids, r, p, entry_ids=None, chunk=4096, workers=1):
    """Per-node determinants of the matrices gathered through entry_ids."""
    if entry_ids is None:
        entry_ids = list(range(r * r))
    stack = np.stack([np.asarray(g, dtype=np.int64).reshape(-1) for g in grids])
    nodes = stack.shape[1]
    ids = np.asarray(entry_ids, dtype=np.int64).reshape(r, r)

    def piece(lo):
        hi = min(lo + chunk, nodes)
        block = np.ascontiguousarray(np.moveaxis(stack[:, lo:hi][ids], 2, 0))
        return det_batch(block, p)

    starts = list(range(0, nodes, chunk))
    if workers > 1 and len(starts) > 1:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            parts = list(pool.map(piece, starts))
    else:
        parts = [piece(lo) for lo in starts]
    return np.concatenate(parts) if parts else np.zeros(0, dtype=np.int64)


def crt_combine(residues, primes):
    """Exact signed integers from one residue vector per prime.

    Mixed radix: a_0 = x_0, a_i = (x_i - a_0) c_i - sum_{0<j<i} a_j (m_j mod p_i) c_i
    with m_j = p_0...p_{j-1} and c_i = m_i^-1 mod p_i; X = Horner over the
    digits; result X if 2X <= P else X - P.
    """
    primes = [int(p) for p in primes]
    for p in primes:
        _check_prime(p)
    xs = [np.asarray(x, dtype=np.int64).reshape(-1) for x in residues]
    weights = [1]
    for p in primes[:-1]:
        weights.append(weights[-1] * p)
    total = weights[-1] * primes[-1]
    digits = [xs[0] % primes[0]]
    for i in range(1, len(primes)):
        p = primes[i]
        c = pow(weights[i] % p, -1, p)
        acc = (xs[i] - digits[0]) * c % p
        for j in range(1, i):
            acc = (acc - digits[j] * (weights[j] % p) % p * c) % p
        digits.append(acc)
    out = []
    cols = [d.tolist() for d in digits]
    n = xs[0].size
    for pos in range(n):
        v = cols[-1][pos]
        for i in range(len(primes) - 2, -1, -1):
            v = v * primes[i] + cols[i][pos]
        out.append(v if 2 * v <= total else v - total)
    return out


def reduce_entry(terms, shape, p):
    """Dense residues (flat, padded to `shape`) of one term dict mod p."""
    grid = np.zeros(max(math.prod(shape), 1), dtype=np.int64)
    for exps, c in terms.items():
        pos = 0
        for e, n in zip(exps, shape):
            pos = pos * n + e
        grid[pos] = int(c) % p
    return grid


def run_pipeline(unique_terms, entry_ids, r, shape, primes, workers=1):
    """End-to-end exact determinant coefficients (flat, padded shape).

    `primes` is a list of (p, omega, q).  Returns (coeffs, per-prime residues).
    """
    residues = []
    for p, omega, q in primes:
        if workers > 1:   # the reference's forward stage maps entries over its worker pool (pipeline.py:364)
            from concurrent.futures import ThreadPoolExecutor
            with ThreadPoolExecutor(workers) as ex:
                grids = list(ex.map(lambda t: ntt_multi(reduce_entry(t, shape, p), shape, p, omega, q),
                                    unique_terms))
        else:
            grids = [ntt_multi(reduce_entry(t, shape, p), shape, p, omega, q) for t in unique_terms]
        values = det_grid(grids, r, p, entry_ids, workers=workers)
        residues.append(ntt_multi(values, shape, p, omega, q, inverse=True))
    return crt_combine(residues, [p for p, _, _ in primes]), residues


def format_polynomial(terms, variables):
    """parsing.py:197-225: graded lexicographic order (total degree, then the
    exponent tuple), highest first; tensor.py:25-32 combines like monomials
    and drops zeros first."""
    pairs = terms.items() if hasattr(terms, "items") else terms
    acc = {}
    for exps, coeff in pairs:
        e = tuple(int(x) for x in exps)
        acc[e] = acc.get(e, 0) + int(coeff)
    norm = {e: c for e, c in acc.items() if c}
    if not norm:
        return "0"
    variables = tuple(variables)
    out = []
    for i, (exps, coeff) in enumerate(sorted(norm.items(), key=lambda it: (sum(it[0]), it[0]), reverse=True)):
        parts = []
        for var, e in zip(variables, exps):
            if e == 1:
                parts.append(var)
            elif e > 1:
                parts.append("%s^%d" % (var, e))
        mag = abs(coeff)
        text = str(mag) if not parts else ("*".join(parts) if mag == 1 else "%d*%s" % (mag, "*".join(parts)))
        if i == 0:
            out.append("-" + text if coeff < 0 else text)
        else:
            out.append(("- " if coeff < 0 else "+ ") + text)
    return " ".join(out)
