"""Runtime forecast (reference pipeline.py:156-264, the paper's Section 5 model).

`predicted_total` is the reference's exact decimal formula
    T = C_p * r^2 * round(mean, 2) * (k / r^2) = C_p * k * round(mean, 2)
(order^2 and the replication factor cancel, so the product stays in exact
decimals: 6 primes, order 16, k = 256, mean 1.36 s -> 2088.96).

`predict` samples the per-unique-entry forward transform under the plan's
first prime, exactly as the reference does (reduce + pad + ntt_forward_multi
per sampled entry, wall-clock per call), except that the transform runs on the
GPU; the forecast therefore describes this package's transform-dominated
model, not the reference's CPU.
"""

from __future__ import annotations

import time
from dataclasses import dataclass
from decimal import ROUND_HALF_UP, Decimal
from fractions import Fraction

from .layout import PolyMatrix, pad_to, reduce_mod
from .planner import Plan
from .transform import TwiddleTable, ntt_forward_multi


@dataclass(frozen=True)
class Prediction:
    """Runtime forecast from sampled per-entry transform times."""

    prime_count: int
    order: int
    unique_count: int
    replication: Fraction
    sample_seconds: tuple
    mean_rounded: Decimal
    total_seconds: float


def _cents(x: float) -> Decimal:
    """x rounded half-up to 0.01, from its shortest decimal repr (the reference's rounding)."""
    return Decimal(repr(float(x))).quantize(Decimal("0.01"), rounding=ROUND_HALF_UP)


def predicted_total(prime_count: int, order: int, unique_count: int, mean_seconds) -> float:
    """Total-seconds forecast C_p * r^2 * round(T_e, 2) * mu with mu = k / r^2.

    r^2 cancels against mu, so the value is C_p * k * round(T_e, 2), computed in
    exact decimals before the final float conversion."""
    if order < 1 or unique_count < 1 or unique_count > order * order:
        raise ValueError(f"unique_count {unique_count} out of range for order {order}")
    return float(_cents(mean_seconds) * prime_count * unique_count)


def _entry_transform_seconds(m: PolyMatrix, pl: Plan, index: int, table: TwiddleTable) -> float:
    """Wall seconds of one unique entry's forward transform on the plan grid
    (reduction and padding are outside the timed call, as in the reference)."""
    grid = pad_to(reduce_mod(m.unique_entries[index % m.k], table.prime), pl.shape)
    t0 = time.perf_counter()
    ntt_forward_multi(grid, table)
    return time.perf_counter() - t0


def predict(m: PolyMatrix, pl: Plan, sample_size: int = 3) -> Prediction:
    """Forecast the run time from `sample_size` timed entry transforms under the
    plan's first prime (entries taken cyclically)."""
    if sample_size < 1:
        raise ValueError("sample_size must be positive")
    table = TwiddleTable(pl.primes[0])
    times = tuple(_entry_transform_seconds(m, pl, i, table) for i in range(sample_size))
    mean = sum(times) / sample_size
    return Prediction(prime_count=pl.prime_count, order=pl.r, unique_count=pl.unique_count,
                      replication=pl.mu, sample_seconds=times, mean_rounded=_cents(mean),
                      total_seconds=predicted_total(pl.prime_count, pl.r, pl.unique_count, mean))
