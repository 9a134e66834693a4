"""Prime-field descriptor F_p (odd p < 2^31) — host side.

Mirrors the reference ``FieldModulus`` (``pkg/src/fpgb/fp.py:80-128``): the
same precomputed constants (Barrett mu = floor(2^62/p), Montgomery p' with
p*p' = -1 mod 2^32, R^2 mod p, lazy window k) and the same validation.  All
hot arithmetic runs on the device (``csrc/fp.cuh``), which keeps residues in
u32 registers and multiplies with Montgomery (R = 2^32) or 32-bit Barrett;
the backend choice never changes a result, exactly as in the reference where
the three backends must agree (``tests/test_sparselin.py:213-221``).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

from .errors import NonInvertibleError, PreconditionError


class Backend(enum.Enum):
    NAIVE = "naive"
    BARRETT = "barrett"
    MONTGOMERY = "montgomery"


class Domain(enum.Enum):
    STANDARD = "standard"
    MONTGOMERY = "montgomery"


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin (witness set valid far beyond 2^64)."""
    if n < 2:
        return False
    small = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)
    for q in small:
        if n % q == 0:
            return n == q
    odd, twos = n - 1, 0
    while not odd & 1:
        odd >>= 1
        twos += 1
    for a in small:
        y = pow(a, odd, n)
        if y == 1 or y == n - 1:
            continue
        for _ in range(twos - 1):
            y = y * y % n
            if y == n - 1:
                break
        else:
            return False
    return True


def _inverse_mod_2k(p: int, k: int) -> int:
    # Hensel lifting: x <- x (2 - p x) doubles the number of correct bits.
    x, mask = 1, (1 << k) - 1
    for _ in range(k.bit_length() + 1):
        x = (x * (2 - p * x)) & mask
    return x


class FieldModulus:
    """Immutable F_p descriptor, shareable across threads and devices."""

    __slots__ = ("p", "backend", "barrett_mu", "mont_r_bits", "mont_pprime",
                 "mont_r2", "lazy_window_k")

    def __init__(self, p: int, backend: "Backend | str" = Backend.NAIVE):
        backend = Backend(backend) if isinstance(backend, str) else backend
        if not 2 < p < (1 << 31):
            raise PreconditionError(f"modulus must satisfy 2 < p < 2^31, got {p}")
        if p % 2 == 0 or not is_prime(p):
            raise PreconditionError(f"modulus must be an odd prime, got {p}")
        object.__setattr__(self, "p", int(p))
        object.__setattr__(self, "backend", backend)
        object.__setattr__(self, "barrett_mu", (1 << 62) // p)
        object.__setattr__(self, "mont_r_bits", 32)
        object.__setattr__(self, "mont_pprime", (-_inverse_mod_2k(p, 32)) % (1 << 32))
        object.__setattr__(self, "mont_r2", (1 << 64) % p)
        object.__setattr__(self, "lazy_window_k", min(16, (1 << 64) // ((p - 1) ** 2)))

    def __setattr__(self, name, value):
        raise AttributeError("FieldModulus is immutable")

    def __eq__(self, other):
        return isinstance(other, FieldModulus) and (self.p, self.backend) == (other.p, other.backend)

    def __hash__(self):
        return hash((self.p, self.backend))

    def __repr__(self):
        return f"FieldModulus(p={self.p}, backend={self.backend.value})"

    def inv(self, a: int) -> int:
        a %= self.p
        if a == 0:
            raise NonInvertibleError("zero is not invertible")
        return pow(a, self.p - 2, self.p)


@dataclass(frozen=True)
class FpElem:
    """A residue tagged with its representation domain."""

    value: int
    domain: Domain = Domain.STANDARD
