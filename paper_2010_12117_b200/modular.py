"""Reference module name `polydet.modular` (modular.py): word-size prime fields,
re-exported from this package's fields module."""

from .fields import (  # noqa: F401
    INT64_SAFE_MODULUS,
    MODULUS_LIMIT,
    CensusResult,
    PrimeSpec,
    add_mod,
    census,
    find_fourier_primes,
    find_root_of_order,
    inv_mod,
    is_prime,
    mul_mod,
    pow_mod,
    sub_mod,
)
