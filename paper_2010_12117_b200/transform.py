"""Multivariate NTT evaluation / interpolation -- drop-in for the reference's
`transform.py` (reference lines 19-159), computed by `pdb_ntt_multi_u32`.

`TwiddleTable` keeps the reference's host API (check_length, root_of_length,
powers, inv_powers, scale) -- these are small host-side queries -- and owns
the device context whose twiddle tables the kernels use.  The transforms
themselves always run on the GPU; there is no host implementation.
"""

from __future__ import annotations

import numpy as np

from . import native
from .fields import PrimeSpec, inv_mod
from .layout import ModTensor, residue_dtype


class TwiddleTable:
    """Root-of-unity tables of one prime (device-resident for the kernels)."""

    def __init__(self, prime: PrimeSpec):
        self.prime = prime
        self._host: dict = {}

    def check_length(self, n: int):
        if n < 1 or n & (n - 1):
            raise ValueError("unsupported length: %d is not a power of two" % n)
        if n > 1 << self.prime.q:
            raise ValueError("unsupported length: %d exceeds 2^%d for p=%d"
                             % (n, self.prime.q, self.prime.p))

    def root_of_length(self, n: int) -> int:
        """w_N = omega^(2^(q - log2 N))  (reference transform.py:41-44)."""
        self.check_length(n)
        return pow(self.prime.omega, 1 << (self.prime.q - (n.bit_length() - 1)), self.prime.p)

    def _row(self, key, w: int, n: int) -> np.ndarray:
        if key not in self._host:
            p = self.prime.p
            vals = [1] * max(n // 2, 1)
            for i in range(1, n // 2):
                vals[i] = vals[i - 1] * w % p
            arr = np.array(vals, dtype=residue_dtype(self.prime))
            arr.setflags(write=False)
            self._host[key] = arr
        return self._host[key]

    def powers(self, n: int) -> np.ndarray:
        return self._row(("f", n), self.root_of_length(n), n)

    def inv_powers(self, n: int) -> np.ndarray:
        return self._row(("i", n), inv_mod(self.root_of_length(n), self.prime.p), n)

    def scale(self, n: int) -> int:
        self.check_length(n)
        return inv_mod(n, self.prime.p)

    def device(self) -> native.PrimeContext:
        return native.prime_context(self.prime)


def _device_transform(values: np.ndarray, shape: tuple, table: TwiddleTable, inverse: bool) -> np.ndarray:
    for n in shape:
        table.check_length(n)
    if not shape:
        return np.array(values, copy=True)
    ctx = table.device()
    data = native.to_device_words(values, ctx.wide)
    native.ntt_multi(ctx, data, 1, shape, None, range(len(shape)), inverse)
    return native.to_host_words(data, ctx.wide).astype(residue_dtype(table.prime))


def _as_row(data, table: TwiddleTable) -> np.ndarray:
    arr = np.array(list(data), dtype=residue_dtype(table.prime))
    if arr.ndim != 1:
        raise ValueError("expected a flat residue vector")
    return arr


def ntt_forward_1d(data, table: TwiddleTable) -> np.ndarray:
    """out[k] = sum_j data[j] w^(jk) mod p  (reference transform.py:102-107)."""
    row = _as_row(data, table)
    table.check_length(row.size)
    return _device_transform(row, (row.size,), table, False)


def ntt_inverse_1d(data, table: TwiddleTable) -> np.ndarray:
    """Inverse of ntt_forward_1d, including the 1/N factor (transform.py:110-116)."""
    row = _as_row(data, table)
    table.check_length(row.size)
    return _device_transform(row, (row.size,), table, True)


def _multi(t: ModTensor, table: TwiddleTable, inverse: bool) -> ModTensor:
    if t.prime != table.prime:
        raise ValueError("tensor and twiddle table use different primes")
    out = _device_transform(t.residues, tuple(t.shape), table, inverse)
    return ModTensor(tuple(t.shape), out, t.prime, tuple(t.axis_vars))


def ntt_forward_multi(t: ModTensor, table: TwiddleTable) -> ModTensor:
    """Values on the full root grid: position (a_0..a_{vn-1}) holds
    f(w_{N_0}^a_0, ..., w_{N_vn-1}^a_vn-1)  (reference transform.py:146-154)."""
    return _multi(t, table, False)


def ntt_inverse_multi(t: ModTensor, table: TwiddleTable) -> ModTensor:
    """The unique coefficient tensor interpolating an evaluation grid."""
    return _multi(t, table, True)
