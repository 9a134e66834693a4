"""Monomials, term orders and packed keys (host side).

Two key encodings exist:

* the **reference key** — big-endian uint64 words, a 32-bit degree lane then
  one 16-bit lane per variable, grevlex tie lanes holding ``0xFFFF - e`` in
  reversed variable order (``pkg/src/fpgb/monomials.py:67-75, 137-154``,
  Assumption 11.1 at ``PAPER.md:1112-1116``).  It is the wire format of
  ``LayoutPlan.dict_keys`` and of ``Ring.sort_key``;
* the **device key** (:class:`DeviceKeyFormat`) — an order-isomorphic,
  injective re-packing with ``b = bits(max batch degree)`` bits per lane and
  the implied variable dropped, 1/2/4/8 uint64 words.  ``key(t*m) = key(m) +
  (key(t) - key(1))`` holds for both encodings, so the device shift-multiply
  is a multiword add of one per-row delta.
"""

from __future__ import annotations

import math

import numpy as np

from .errors import ArityMismatchError, CorruptKeyError, DivisionError, LaneOverflowError

ORDERS = ("grevlex", "deglex", "lex")
MAX_VARS = 32
_LANE = 16
_LANE_MAX = (1 << _LANE) - 1
_DEG_LANE = 32

Monomial = tuple
MonKey = tuple

ORDER_CODE = {"grevlex": 0, "deglex": 1, "lex": 2}


class Ring:
    """Variables, term order and coefficient field of a polynomial ring."""

    __slots__ = ("var_names", "order", "modulus", "n_vars", "n_key_words", "graded",
                 "_shifts", "_cache")

    def __init__(self, var_names, order: str, modulus):
        names = tuple(var_names)
        if not 1 <= len(names) <= MAX_VARS:
            raise ValueError(f"need 1..{MAX_VARS} variables, got {len(names)}")
        if len(set(names)) != len(names):
            raise ValueError("variable names must be distinct")
        if order not in ORDERS:
            raise ValueError(f"unknown order {order!r}; expected one of {ORDERS}")
        self.var_names = names
        self.order = order
        self.modulus = modulus
        self.n_vars = len(names)
        self.graded = order != "lex"
        head = _DEG_LANE if self.graded else 0
        self.n_key_words = (head + _LANE * self.n_vars + 63) // 64
        # bit offset (from the most significant end of the key) of each lane
        self._shifts = head
        self._cache: dict = {}

    # -- scalar reference keys ------------------------------------------------
    def sort_key(self, u: Monomial) -> MonKey:
        k = self._cache.get(u)
        if k is None:
            k = mon_key_pack(u, self)
            self._cache[u] = k
        return k

    def one(self) -> Monomial:
        return (0,) * self.n_vars

    def var(self, i: int) -> Monomial:
        return tuple(1 if j == i else 0 for j in range(self.n_vars))

    def __repr__(self):
        return f"Ring(vars={self.var_names}, order={self.order}, p={self.modulus.p})"


def _arity(u, ring):
    if len(u) != ring.n_vars:
        raise ArityMismatchError(f"expected {ring.n_vars} exponents, got {len(u)}")


def _lanes_of(u, ring):
    """Lane values in significance order (without the degree lane)."""
    if ring.order == "grevlex":
        return [_LANE_MAX - e for e in reversed(u)]
    return list(u)


def mon_key_pack(u: Monomial, ring: Ring) -> MonKey:
    """Reference key of one monomial as a tuple of W python ints."""
    _arity(u, ring)
    big = 0
    nbits = 0
    if ring.graded:
        d = 0
        for e in u:
            if not 0 <= e <= _LANE_MAX:
                raise LaneOverflowError(f"exponent {e} does not fit a 16-bit lane")
            d += e
        if d >> _DEG_LANE:
            raise LaneOverflowError("total degree does not fit the 32-bit degree lane")
        big, nbits = d, _DEG_LANE
    else:
        for e in u:
            if not 0 <= e <= _LANE_MAX:
                raise LaneOverflowError(f"exponent {e} does not fit a 16-bit lane")
    for lane in _lanes_of(u, ring):
        big = (big << _LANE) | lane
        nbits += _LANE
    W = ring.n_key_words
    big <<= 64 * W - nbits
    return tuple((big >> (64 * (W - 1 - w))) & 0xFFFFFFFFFFFFFFFF for w in range(W))


def mon_key_unpack(k: MonKey, ring: Ring) -> Monomial:
    return tuple(int(x) for x in key_unpack_vec(np.asarray([k], dtype=np.uint64), ring)[0])


def _lane_positions(ring: Ring):
    head = _DEG_LANE if ring.graded else 0
    pos = []
    for i in range(ring.n_vars):
        off = head + _LANE * i  # from the most significant bit
        pos.append((off // 64, 64 - (off % 64) - _LANE))
    return pos


def key_pack_vec(exps: np.ndarray, ring: Ring) -> np.ndarray:
    """(K, n) exponents -> (K, W) uint64 reference keys."""
    exps = np.asarray(exps)
    if exps.ndim != 2 or exps.shape[1] != ring.n_vars:
        raise ArityMismatchError(f"expected shape (K, {ring.n_vars}), got {exps.shape}")
    if len(exps) >= 4096 and exps.dtype == np.int64 and exps.flags.c_contiguous:
        # large blocks (the host basis copy): one pass in csrc/hostglue.cpp
        from .hostglue import native

        out = np.empty((exps.shape[0], ring.n_key_words), dtype=np.uint64)
        code = native().pack_keys(exps, exps.shape[0], ring.n_vars, int(ring.graded), int(ring.order == "grevlex"),
                                  ring.n_key_words, out)
        if code == 1:
            raise LaneOverflowError("exponent does not fit a 16-bit lane")
        if code == 2:
            raise LaneOverflowError("total degree does not fit the 32-bit degree lane")
        return out
    if exps.size and (exps.min() < 0 or exps.max() > _LANE_MAX):
        raise LaneOverflowError("exponent does not fit a 16-bit lane")
    e = exps.astype(np.uint64)
    out = np.zeros((e.shape[0], ring.n_key_words), dtype=np.uint64)
    if ring.graded:
        deg = e.sum(axis=1, dtype=np.uint64)
        if deg.size and int(deg.max()) >> _DEG_LANE:
            raise LaneOverflowError("total degree does not fit the 32-bit degree lane")
        out[:, 0] |= deg << np.uint64(32)
    lanes = (np.uint64(_LANE_MAX) - e[:, ::-1]) if ring.order == "grevlex" else e
    for i, (w, sh) in enumerate(_lane_positions(ring)):
        out[:, w] |= lanes[:, i] << np.uint64(sh)
    return out


def key_unpack_vec(keys: np.ndarray, ring: Ring) -> np.ndarray:
    """(K, W) reference keys -> (K, n) int64 exponents, rejecting corrupt keys."""
    keys = np.asarray(keys, dtype=np.uint64)
    if keys.ndim != 2 or keys.shape[1] != ring.n_key_words:
        raise CorruptKeyError(f"expected shape (K, {ring.n_key_words}), got {keys.shape}")
    lanes = np.empty((keys.shape[0], ring.n_vars), dtype=np.uint64)
    for i, (w, sh) in enumerate(_lane_positions(ring)):
        lanes[:, i] = (keys[:, w] >> np.uint64(sh)) & np.uint64(_LANE_MAX)
    exps = (np.uint64(_LANE_MAX) - lanes)[:, ::-1] if ring.order == "grevlex" else lanes
    if keys.size and not np.array_equal(key_pack_vec(exps, ring), keys):
        raise CorruptKeyError("key lanes are internally inconsistent")
    return exps.astype(np.int64)


def key_cmp_rows(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Row-wise lexicographic compare of key-word matrices: -1 / 0 / +1."""
    a = np.asarray(a, dtype=np.uint64)
    b = np.asarray(b, dtype=np.uint64)
    res = np.zeros(a.shape[0], dtype=np.int8)
    for w in reversed(range(a.shape[1])):
        aw, bw = a[:, w], b[:, w]
        res = np.where(aw < bw, np.int8(-1), np.where(aw > bw, np.int8(1), res))
    return res


def mon_degree(u: Monomial) -> int:
    return sum(u)


def mon_compare(u: Monomial, v: Monomial, ring: Ring) -> int:
    """Direct term-order comparison (not through keys): -1, 0 or +1."""
    _arity(u, ring)
    _arity(v, ring)
    if ring.graded and sum(u) != sum(v):
        return -1 if sum(u) < sum(v) else 1
    if ring.order == "grevlex":
        for a, b in zip(reversed(u), reversed(v)):
            if a != b:
                return 1 if a < b else -1
        return 0
    for a, b in zip(u, v):
        if a != b:
            return -1 if a < b else 1
    return 0


def mon_mul(u: Monomial, v: Monomial) -> Monomial:
    if len(u) != len(v):
        raise ArityMismatchError("arity mismatch in monomial product")
    w = tuple(a + b for a, b in zip(u, v))
    if (w and max(w) > _LANE_MAX) or sum(w) >> _DEG_LANE:
        raise LaneOverflowError("monomial product overflows key lanes")
    return w


def mon_lcm(u: Monomial, v: Monomial) -> Monomial:
    if len(u) != len(v):
        raise ArityMismatchError("arity mismatch in lcm")
    return tuple(a if a > b else b for a, b in zip(u, v))


def mon_divides(u: Monomial, v: Monomial) -> bool:
    """True iff u | v."""
    if len(u) != len(v):
        raise ArityMismatchError("arity mismatch in divisibility test")
    for a, b in zip(u, v):
        if a > b:
            return False
    return True


def mon_div(u: Monomial, v: Monomial) -> Monomial:
    """u / v, which must be exact."""
    if len(u) != len(v):
        raise ArityMismatchError("arity mismatch in monomial division")
    q = tuple(a - b for a, b in zip(u, v))
    if q and min(q) < 0:
        raise DivisionError(f"{v} does not divide {u}")
    return q


def count_monomials(n: int, d: int) -> int:
    if n < 1 or d < 0:
        raise ValueError("need n >= 1 and d >= 0")
    return math.comb(n + d, d)


def mon_format(u: Monomial, ring: Ring) -> str:
    parts = []
    for name, e in zip(ring.var_names, u):
        if e:
            parts.append(name if e == 1 else f"{name}^{e}")
    return "*".join(parts) if parts else "1"


# ---------------------------------------------------------------------------
# Device key format
# ---------------------------------------------------------------------------


class DeviceKeyFormat:
    """Compact order-isomorphic key used inside the CUDA engine.

    Graded orders: lane width ``b = max(1, bits(D))`` for a batch whose
    monomials all have degree <= D; lanes (most significant first) are the
    degree, then for grevlex ``(2^b-1) - e_{n-1}, ..., (2^b-1) - e_1`` and for
    deglex ``e_0, ..., e_{n-2}`` (the dropped variable is implied by the
    degree).  Lex keeps 16-bit lanes ``e_0..e_{n-1}``.  The key is an
    unsigned integer of ``64 * words`` bits, stored most significant word
    first; ``words`` is padded to 1, 2, 4 or 8.
    """

    __slots__ = ("order", "n_vars", "lane_bits", "n_lanes", "words", "max_degree")

    def __init__(self, ring: Ring, max_degree: int):
        self.order = ring.order
        self.n_vars = ring.n_vars
        self.max_degree = int(max_degree)
        if ring.graded:
            self.lane_bits = max(1, int(max_degree).bit_length())
            self.n_lanes = ring.n_vars  # degree lane + (n - 1) variable lanes
        else:
            self.lane_bits = _LANE
            self.n_lanes = ring.n_vars
        bits = self.lane_bits * self.n_lanes
        w = 1
        while 64 * w < bits:
            w *= 2
        if w > 8:
            raise LaneOverflowError(f"batch degree {max_degree} too large for the device key")
        self.words = w

    def lanes(self, exps: np.ndarray) -> np.ndarray:
        """(K, n) exponents -> (K, n_lanes) lane values, significance order."""
        e = np.asarray(exps, dtype=np.int64)
        full = (1 << self.lane_bits) - 1
        if self.order == "grevlex":
            return np.concatenate([e.sum(axis=1, keepdims=True), full - e[:, :0:-1]], axis=1)
        if self.order == "deglex":
            return np.concatenate([e.sum(axis=1, keepdims=True), e[:, :-1]], axis=1)
        return e

    def pack_int(self, u) -> int:
        """Device key of one monomial as a python int (for tests / deltas)."""
        v = 0
        for lane in self.lanes(np.asarray([u]))[0].tolist():
            v = (v << self.lane_bits) | int(lane)
        return v

    def as_tuple(self):
        return (ORDER_CODE[self.order], self.n_vars, self.lane_bits, self.words)
