"""Determinants mod p -- drop-in for the reference's `determinant.py`
(reference lines 23-169), computed by `pdb_det_batch_u32` / `pdb_condense_u32` (and their
`_u64` twins for primes >= 2^31).

`det_grid` keeps the reference's signature and errors; `chunk_size` and
`workers` are accepted and ignored (the result never depended on them in the
reference either, determinant.py:101-104).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import native
from .fields import PrimeSpec
from .layout import residue_dtype


@dataclass(frozen=True)
class ModMatrix:
    """r x r residues mod one prime."""

    r: int
    entries: tuple
    prime: PrimeSpec

    def __post_init__(self):
        if self.r < 1:
            raise ValueError("matrix order must be positive")
        if len(self.entries) != self.r or any(len(row) != self.r for row in self.entries):
            raise ValueError("entries do not form a %dx%d matrix" % (self.r, self.r))
        p = self.prime.p
        if not all(0 <= v < p for row in self.entries for v in row):
            raise ValueError("entries must be canonical residues in [0, p)")

    @classmethod
    def from_rows(cls, rows, prime: PrimeSpec) -> "ModMatrix":
        p = prime.p
        return cls(len(rows), tuple(tuple(v % p for v in row) for row in rows), prime)


@dataclass(frozen=True)
class PivotRecord:
    """Pivot of elimination step `step`: value, column, and whether that
    column flips the running permutation sign."""

    step: int
    value: int
    column: int
    flips_sign: bool


def condense(m: ModMatrix):
    """Determinant plus the pivot trail of the reference's condensation
    (first nonzero entry of row i is the pivot; determinant.py:57-84)."""
    torch = native._torch()
    ctx = native.prime_context(m.prime)
    r = m.r
    wide = ctx.wide
    word = native.word_dtype(wide)
    mat = native.to_device_words(np.array([int(v) for row in m.entries for v in row], dtype=object), wide)
    vals = torch.zeros(r, dtype=word, device=mat.device)
    cols = torch.zeros(r, dtype=torch.int32, device=mat.device)
    det = torch.zeros(1, dtype=word, device=mat.device)
    nbytes = 4 * r * r + 256 + (native.det_scratch_bytes(r, 1, True) if wide else 512 * r * r + 256)
    scratch = native.scratch_tensor(nbytes)
    native.condense(ctx, mat, r, vals, cols, det, scratch)
    vals_h = native.to_host_words(vals, wide).tolist()
    cols_h = cols.cpu().numpy().tolist()
    records, used = [], []
    for i in range(r):
        c = cols_h[i]
        if c < 0:
            break
        flips = sum(1 for u in used if u > c) % 2 == 1
        records.append(PivotRecord(i, int(vals_h[i]), c, flips))
        used.append(c)
    return int(native.to_host_words(det, wide)[0]), records


def det_mod(m: ModMatrix) -> int:
    """Exact determinant of a residue matrix."""
    return condense(m)[0]


def det_grid(entry_grids, r: int, prime: PrimeSpec, *, entry_ids=None, chunk_size: int = 4096,
             workers: int = 1) -> np.ndarray:
    """Determinant at every node; entry (i, j) of node n's matrix is
    entry_grids[entry_ids[i*r + j]][n] (identity layout by default)."""
    if entry_ids is None:
        entry_ids = list(range(r * r))
    entry_ids = [int(e) for e in entry_ids]
    if len(entry_ids) != r * r:
        raise ValueError("need %d entry ids, got %d" % (r * r, len(entry_ids)))
    if any(not 0 <= e < len(entry_grids) for e in entry_ids):
        raise ValueError("entry id references a missing grid")
    grids = [np.asarray(g).reshape(-1) for g in entry_grids]
    nodes = grids[0].size
    if any(g.size != nodes for g in grids):
        raise ValueError("entry grids must share one shape")
    dtype = residue_dtype(prime)
    if nodes == 0:
        return np.empty(0, dtype=dtype)
    torch = native._torch()
    ctx = native.prime_context(prime)
    wide = ctx.wide
    p = prime.p
    stacked = np.stack(grids)
    stacked = np.array([int(v) % p for v in stacked.reshape(-1)], dtype=object).reshape(stacked.shape) \
        if stacked.dtype == object else stacked.astype(np.int64) % p
    dev = native.to_device_words(stacked, wide)
    ids = torch.tensor(entry_ids, dtype=torch.int32, device=dev.device)
    out = torch.empty(nodes, dtype=native.word_dtype(wide), device=dev.device)
    scratch = native.scratch_tensor(native.det_scratch_bytes(r, nodes, wide))
    native.det_batch(ctx, dev, nodes, ids, r, 0, nodes, out, scratch)
    return native.to_host_words(out, wide).astype(dtype)
