"""Chinese remaindering -- drop-in for the reference's `crt.py` (lines 20-130).

`combine_tensor` runs the whole mixed-radix lift on the GPU
(`pdb_crt_mrc_u32`: digits, multi-limb Horner and the signed lift) and the
host only turns the returned limbs into Python ints.  `build_basis`,
`horner_lift` and `signed_lift` are exact big-integer host helpers of the
scalar API; `mrc_digits` reads the digits off the device-lifted value.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np

from . import native
from .fields import inv_mod
from .layout import CoeffTensor


@dataclass(frozen=True)
class CrtBasis:
    """weights[j] = p_0...p_{j-1}; inverses[i] = weights[i]^-1 mod p_i;
    weight_residues[i][j] = weights[j] mod p_i; product = P."""

    primes: tuple
    weights: tuple
    inverses: tuple
    weight_residues: tuple
    product: int


def build_basis(primes) -> CrtBasis:
    primes = tuple(int(p) for p in primes)
    if not primes:
        raise ValueError("at least one prime is required")
    if len(set(primes)) < len(primes):
        raise ValueError("duplicate primes in %s" % (primes,))
    weights = [1]
    for p in primes[:-1]:
        weights.append(weights[-1] * p)
    inverses = [1] + [inv_mod(weights[i] % primes[i], primes[i]) for i in range(1, len(primes))]
    table = [()] + [tuple(w % primes[i] for w in weights[:i]) for i in range(1, len(primes))]
    return CrtBasis(primes, tuple(weights), tuple(inverses), tuple(table), weights[-1] * primes[-1])


def horner_lift(digits, basis: CrtBasis) -> int:
    """sum_j digits[j] * weights[j], folded from the top digit."""
    if len(digits) != len(basis.primes):
        raise ValueError("got %d digits for %d primes" % (len(digits), len(basis.primes)))
    value = int(digits[-1])
    for d, p in zip(reversed(digits[:-1]), reversed(basis.primes[:-1])):
        value = value * p + int(d)
    return value


def signed_lift(x: int, product: int) -> int:
    """[0, P) -> (-P/2, P/2]."""
    if not 0 <= x < product:
        raise ValueError("%d is not a canonical residue mod %d" % (x, product))
    return x - product if 2 * x > product else x


def limbs_to_ints(limbs: np.ndarray, neg: np.ndarray) -> list:
    """Device CRT output (|X| as LE u32 limbs + sign) -> Python ints."""
    n, L = limbs.shape
    out = [0] * n
    nonzero = np.flatnonzero(limbs.any(axis=1))
    if nonzero.size == 0:
        return out
    small = limbs[nonzero, 2:].any(axis=1) == 0 if L > 2 else np.ones(nonzero.size, dtype=bool)
    sidx = nonzero[small]
    if sidx.size:
        mag = limbs[sidx, 0].astype(np.int64) | (limbs[sidx, 1].astype(np.int64) << 32) if L > 1 \
            else limbs[sidx, 0].astype(np.int64)
        big2 = (limbs[sidx, 1] >> 31).astype(bool) if L > 1 else np.zeros(sidx.size, dtype=bool)
        vals = np.where(neg[sidx].astype(bool), -mag, mag)
        for i, v, b in zip(sidx.tolist(), vals.tolist(), big2.tolist()):
            out[i] = v
        # magnitudes >= 2^63 do not fit int64: redo those exactly
        for i in sidx[big2].tolist():
            v = int.from_bytes(limbs[i].tobytes(), "little")
            out[i] = -v if neg[i] else v
    bidx = nonzero[~small]
    if bidx.size:
        rows = limbs[bidx]
        raw = rows.tobytes()
        width = 4 * L
        negs = neg[bidx].tolist()
        for j, i in enumerate(bidx.tolist()):
            v = int.from_bytes(raw[j * width:(j + 1) * width], "little")
            out[i] = -v if negs[j] else v
    return out


def wide_primes(primes) -> bool:
    """True when the set needs the u64 kernels (some p >= 2^31); the whole set then
    shares u64 residues."""
    return any(native.needs_wide(int(p)) for p in primes)


def device_lift(residues_dev, primes, n: int, stride: int) -> list:
    """CRT of device residue rows [P][stride] -> list of n Python ints.

    The GPU writes |X| as u32 limbs + a sign byte per coefficient; only the
    nonzero coefficients, trimmed to the widest limb actually used, are copied
    back, and the native host module (_pdb_host, csrc/host_ints.cpp) builds the
    Python ints in one C loop (reference crt.py:122-130 materialises them with
    Python big-int Horner).
    """
    torch = native._torch()
    P = len(primes)
    wide = wide_primes(primes)
    if residues_dev.dtype != native.word_dtype(wide):
        raise ValueError("residue rows must be %s for this prime set" % native.word_dtype(wide))
    L = native.crt_limbs(P, wide)
    dev = residues_dev.device
    host = native.host_module()
    if not wide:
        # the library finds the nonzero coefficients (some residue != 0), lifts
        # only those into compact limb rows and reports the widest; only the used
        # limbs of the nonzero rows cross to the host
        idx = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        native.crt_nonzero(residues_dev, P, n, stride, idx, cnt)
        count = int(cnt.item())
        limbs = torch.empty((max(count, 1), L), dtype=torch.int32, device=dev)
        neg = torch.empty(max(count, 1), dtype=torch.uint8, device=dev)
        wbuf = torch.zeros(1, dtype=torch.int32, device=dev)
        native.crt_mrc_sel(residues_dev, P, stride, primes, idx, count, limbs, L, neg, wbuf)
        width = max(int(wbuf.item()), 1)
        idx_h = np.ascontiguousarray(idx[:count].cpu().numpy())
        neg_h = np.ascontiguousarray(neg[:count].cpu().numpy())
        return _build_ints(host, limbs, count, width, L, idx_h, neg_h, n)
    limbs = torch.empty((n, L), dtype=torch.int32, device=dev)
    neg = torch.empty(n, dtype=torch.uint8, device=dev)
    scratch = native.scratch_tensor(native.crt_scratch_bytes(P, wide), dev)
    native.crt_mrc(residues_dev, P, n, stride, primes, limbs, L, neg, scratch, wide=wide)
    used = limbs != 0
    idx = used.any(dim=1).nonzero().squeeze(1)
    cols = used.any(dim=0).nonzero()
    width = int(cols.max().item()) + 1 if cols.numel() else 1
    del used
    sel = limbs.index_select(0, idx)[:, :width].contiguous()
    sel_neg = neg.index_select(0, idx)
    idx_h = np.ascontiguousarray(idx.cpu().numpy())
    neg_h = np.ascontiguousarray(sel_neg.cpu().numpy())
    with _PIN_LOCK:   # the staging buffer is shared; the ints are built before it is reused
        return host.ints_from_limbs(_to_host(sel), idx_h, neg_h, int(n), int(width))


def sharded_lift(block, primes, n: int, lo: int, rank: int, size: int) -> tuple:
    """Multi-GPU CRT (shard.py): `block` holds every prime's residues [P][m] of
    this rank's coefficient range [lo, lo + m); each rank compacts and lifts its
    range, the compact limb rows are all-gathered, and every rank builds the
    same tuple of n Python ints (u32 prime sets)."""
    from . import shard

    torch = native._torch()
    P, m = block.shape
    dev = block.device
    block = block.contiguous()
    idx = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    native.crt_nonzero(block, P, m, m, idx, cnt)
    count = int(cnt.item())
    L = native.crt_limbs(P)
    limbs = torch.empty((max(count, 1), L), dtype=torch.int32, device=dev)
    neg = torch.empty(max(count, 1), dtype=torch.uint8, device=dev)
    wbuf = torch.zeros(1, dtype=torch.int32, device=dev)
    native.crt_mrc_sel(block, P, m, primes, idx, count, limbs, L, neg, wbuf)
    import torch.distributed as dist
    dist.all_reduce(wbuf, op=dist.ReduceOp.MAX)
    width = max(int(wbuf.item()), 1)
    idx[:count] += lo
    g_limbs, g_idx, g_neg = shard.gather_compact(count, limbs, idx, neg, width, rank, size)
    idx_h = np.ascontiguousarray(g_idx.cpu().numpy())
    neg_h = np.ascontiguousarray(g_neg.cpu().numpy())
    g_limbs = g_limbs.contiguous()
    return _build_ints(native.host_module(), g_limbs, g_limbs.shape[0], width, g_limbs.shape[1], idx_h, neg_h, n)


def _build_ints(host, limbs, count: int, width: int, stride: int, idx_h, neg_h, n: int) -> tuple:
    """Compact |X| limb rows on the device -> the tuple of n Python ints.  On
    CPython 3.12/3.13 the device re-cuts the rows into CPython's 30-bit digits
    (pdb_limbs_to_digits30) so the host only allocates and copies; elsewhere
    the limb rows go through the portable constructor."""
    torch = native._torch()
    if count and host.direct_path() and (count < 2 or bool(np.all(idx_h[1:] > idx_h[:-1]))):
        D = (32 * width + 29) // 30
        digits = torch.empty((count, D), dtype=torch.int32, device=limbs.device)
        nd = torch.empty(count, dtype=torch.uint8, device=limbs.device)
        native.limbs_to_digits30(limbs, count, width, stride, digits, D, nd)
        nd_h = np.ascontiguousarray(nd.cpu().numpy())
        with _PIN_LOCK:   # the staging buffer is shared; the ints are built before it is reused
            if count >= _MT_MIN and _mt_ok():
                return host.ints_from_digits_mt(_to_host(digits), nd_h, idx_h, neg_h, int(n), int(D), _mt_threads())
            return host.ints_from_digits(_to_host(digits), nd_h, idx_h, neg_h, int(n), int(D))
    with _PIN_LOCK:
        return host.ints_from_limbs(_to_host(limbs[:count, :width]), idx_h, neg_h, int(n), int(width))


#: results with at least this many nonzero coefficients build their ints on threads
_MT_MIN = 1 << 16


def _mt_ok() -> bool:
    """The threaded builder allocates int objects with the raw allocator (freed
    through PyObject_Free like any large object); only without allocation hooks."""
    import os
    import sys
    import tracemalloc
    return (hasattr(native.host_module(), "ints_from_digits_mt") and not tracemalloc.is_tracing()
            and not sys.flags.dev_mode
            and os.environ.get("PYTHONMALLOC", "") in ("", "pymalloc", "malloc")
            and not os.environ.get("PDB_HOST_SERIAL"))


def _mt_threads() -> int:
    import os
    return max(1, min(16, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count() or 1))


_PINNED = {}
_PIN_LOCK = threading.Lock()


def _to_host(t):
    """Device tensor -> numpy through a reused page-locked staging buffer (the
    limb block of a large run is hundreds of MB; pageable copies run at a
    fraction of the link rate).  Small tensors take the plain path."""
    torch = native._torch()
    nbytes = t.numel() * t.element_size()
    if nbytes < (8 << 20) or t.device.type != "cuda":
        return np.ascontiguousarray(t.contiguous().cpu().numpy())
    buf = _PINNED.get(t.device.index)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1 << 28), dtype=torch.uint8, pin_memory=True)
        _PINNED[t.device.index] = buf
    view = buf[:nbytes].view(t.dtype).view(t.shape)
    view.copy_(t.contiguous())
    return view.numpy()


def mrc_digits(residues, basis: CrtBasis) -> list:
    """Mixed-radix digits: X = sum digits[j] weights[j], 0 <= digits[j] < p_j."""
    if len(residues) != len(basis.primes):
        raise ValueError("got %d residues for %d primes" % (len(residues), len(basis.primes)))
    vals = np.array([[int(x) % p] for x, p in zip(residues, basis.primes)], dtype=object)
    value = device_lift(native.to_device_words(vals, wide_primes(basis.primes)), basis.primes, 1, 1)[0]
    if value < 0:
        value += basis.product
    digits = []
    for p in basis.primes:
        value, d = divmod(value, p)
        digits.append(d)
    return digits


def combine_tensor(residue_tensors) -> CoeffTensor:
    """Exact signed coefficients from one residue tensor per prime."""
    if not residue_tensors:
        raise ValueError("at least one residue tensor is required")
    shape = residue_tensors[0].shape
    names = residue_tensors[0].axis_vars
    if any(t.shape != shape or t.axis_vars != names for t in residue_tensors):
        raise ValueError("residue tensors must share one shape")
    basis = build_basis([t.prime.p for t in residue_tensors])
    n = residue_tensors[0].size
    stacked = np.stack([np.asarray(t.residues, dtype=object).astype(np.int64) for t in residue_tensors])
    coeffs = device_lift(native.to_device_words(stacked, wide_primes(basis.primes)), basis.primes, n, n)
    return CoeffTensor(tuple(shape), tuple(coeffs), tuple(names))
