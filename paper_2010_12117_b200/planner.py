"""Planning: grid shape, coefficient bound, prime list (host side).

Every decision reproduces the reference's (`pipeline.py:45-222`) so that
`Plan.to_dict()` and `Plan.digest()` are identical -- the digest keys the
checkpoint workspace, and the primes/roots fix every evaluation point:

* det degree bound  D_i = sum over rows of max over the row's entries of deg_i
  (`pipeline.py:184-196`); grid N_i = 2^ceil(log2(D_i + 1)) (`tensor.py:184-191`);
* coefficient bound B = r! * prod over rows of the largest entry 1-norm
  (`pipeline.py:168-181`);
* primes = the shortest ascending run of p = 1 (mod 2^q_max), p >= prime_start,
  with product >= 2B + 1 and at least min_primes of them (`pipeline.py:199-222`).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction
from typing import Callable, Optional

from .checkpoint import digest_of
from .fields import PrimeSpec, find_fourier_primes
from .layout import PolyMatrix, pad_shape


@dataclass
class PipelineConfig:
    """Planning and scheduling knobs (reference `pipeline.py:45-63`).

    `workers` and `chunk_size` are accepted for drop-in compatibility; like in
    the reference they never change results, and on the GPU they are not
    used (the device kernels size their own launches).  Multi-GPU runs shard
    primes across the processes of a torch.distributed job (one per GPU; see
    executor.py and shard.py), not through this config.
    """

    prime_start: int = 10**9
    min_primes: int = 2
    scan_limit: int = 1_000_000
    workers: int = 1
    chunk_size: int = 4096
    progress: Optional[Callable[[str], None]] = None

    def _notify(self, unit: str):
        if self.progress is not None:
            self.progress(unit)


@dataclass(frozen=True)
class Plan:
    """Sizes, bound and primes fixed before any arithmetic runs."""

    r: int
    variables: tuple
    entry_degrees: tuple
    det_degrees: tuple
    shape: tuple
    q_max: int
    boundary: int
    primes: tuple
    unique_count: int

    def __post_init__(self):
        if any(n & (n - 1) for n in self.shape):
            raise ValueError("node shape %s is not power-of-two padded" % (self.shape,))
        for spec in self.primes:
            if spec.q < self.q_max:
                raise ValueError("prime %s cannot host length 2^%s" % (spec.p, self.q_max))
        if self.prime_product <= 2 * self.boundary:
            raise ValueError("prime product does not cover the signed coefficient range")
        if not 0 < self.unique_count <= self.r * self.r:
            raise ValueError("unique entry count %s out of range" % self.unique_count)

    @property
    def node_count(self) -> int:
        return math.prod(self.shape)

    @property
    def prime_count(self) -> int:
        return len(self.primes)

    @property
    def prime_product(self) -> int:
        return math.prod(s.p for s in self.primes)

    @property
    def mu(self) -> Fraction:
        return Fraction(self.unique_count, self.r * self.r)

    def to_dict(self) -> dict:
        return {
            "r": self.r,
            "variables": list(self.variables),
            "entry_degrees": list(self.entry_degrees),
            "det_degrees": list(self.det_degrees),
            "shape": list(self.shape),
            "q_max": self.q_max,
            "boundary": self.boundary,
            "primes": [[s.p, s.c, s.q, s.omega] for s in self.primes],
            "unique_count": self.unique_count,
        }

    @classmethod
    def from_dict(cls, data: dict) -> "Plan":
        return cls(
            r=int(data["r"]),
            variables=tuple(data["variables"]),
            entry_degrees=tuple(data["entry_degrees"]),
            det_degrees=tuple(data["det_degrees"]),
            shape=tuple(data["shape"]),
            q_max=int(data["q_max"]),
            boundary=int(data["boundary"]),
            primes=tuple(PrimeSpec(*quad) for quad in data["primes"]),
            unique_count=int(data["unique_count"]),
        )

    def digest(self) -> str:
        return digest_of(self.to_dict())


@dataclass
class StageTimings:
    """Seconds per stage, summed over primes.  On the GPU path these are
    CUDA-event times of the stage's kernels (host work excluded)."""

    fft: float = 0.0
    det: float = 0.0
    ifft: float = 0.0
    crt: float = 0.0

    def as_dict(self) -> dict:
        return {"fft": self.fft, "det": self.det, "ifft": self.ifft, "crt": self.crt}


def _one_norms(m: PolyMatrix):
    return [sum(abs(c) for c in t.coeffs) for t in m.unique_entries]


def coefficient_bound(m: PolyMatrix) -> int:
    """r! * prod_i max_j ||M_ij||_1: dominates every coefficient of det(M)."""
    norms = _one_norms(m)
    ids = m.entry_ids
    bound = math.factorial(m.r)
    for i in range(m.r):
        bound *= max(norms[e] for e in ids[i * m.r:(i + 1) * m.r])
    return bound


def degree_bound(m: PolyMatrix) -> tuple:
    """Per variable: sum over rows of the row's largest entry degree."""
    degs = [t.degrees() for t in m.unique_entries]
    vn = len(m.variables)
    ids = m.entry_ids
    total = [0] * vn
    for i in range(m.r):
        row = [degs[e] for e in ids[i * m.r:(i + 1) * m.r]]
        for v in range(vn):
            total[v] += max(d[v] for d in row)
    return tuple(total)


def plan(m: PolyMatrix, config: Optional[PipelineConfig] = None) -> Plan:
    """Choose the evaluation grid and the primes for an exact run."""
    cfg = config or PipelineConfig()
    det_degrees = degree_bound(m)
    shape, q_max = pad_shape([d + 1 for d in det_degrees])
    boundary = coefficient_bound(m)
    primes = find_fourier_primes(q_max, 2 * boundary + 1, cfg.prime_start,
                                 min_count=cfg.min_primes, scan_limit=cfg.scan_limit)
    return Plan(r=m.r, variables=m.variables, entry_degrees=m.max_degrees(),
                det_degrees=det_degrees, shape=shape, q_max=q_max, boundary=boundary,
                primes=tuple(primes), unique_count=m.k)
