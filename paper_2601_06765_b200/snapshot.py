"""Binary F4 state snapshots for replay and checkpoint.

The reference has no checkpoint format; its replay recipe is
text: ``format_system(ring, state.basis)`` (systems.py:125-132) plus the pair
list ``[(q.i, q.j)]``, re-parsed and re-paired with ``_make_pair``
(groebner.py:149-151).  This module stores the same information in a compact
binary container that loads without parsing polynomial text:

    b"F4BSNAP1" | u64 header_len | header (JSON, utf-8) |
    lengths i64[G] | exps u16[T][n] | coeffs u32[T] | pair_i i64[P] |
    pair_j i64[P] | sha256(everything before) (32 bytes)

Header: p, order, var names, G (basis size), T (terms), P (pairs),
zero_reductions, steps (BatchStats count).  Exponents are u16 (the device
lanes, monomials.py:142-147 caps them at 0xFFFF) and coefficients u32
(p < 2^31).  Loading rebuilds the pair queue with ``_make_pair`` and the
reference order ``Pair.sort_tuple`` (groebner.py:110-116), so a restored
state continues the F4 loop exactly as the saved one would.
"""

from __future__ import annotations

import hashlib
import json
import struct

import numpy as np

from .fp import FieldModulus
from .monomials import Ring
from .polynomials import Poly

MAGIC = b"F4BSNAP1"


def dumps_state(state) -> bytes:
    ring = state.ring
    basis = state.basis
    n = ring.n_vars
    lengths = np.asarray([len(f.terms) for f in basis], dtype=np.int64)
    T = int(lengths.sum())
    exps = np.zeros((T, n), dtype=np.uint16)
    coeffs = np.zeros(T, dtype=np.uint32)
    t = 0
    for f in basis:
        for e, c in f.terms:
            exps[t] = e
            coeffs[t] = c
            t += 1
    pi = np.asarray([q.i for q in state.pairs], dtype=np.int64)
    pj = np.asarray([q.j for q in state.pairs], dtype=np.int64)
    header = json.dumps({"p": ring.modulus.p, "order": ring.order, "vars": list(ring.var_names), "G": len(basis),
                         "T": T, "P": len(pi), "zero_reductions": int(state.zero_reductions),
                         "steps": len(state.stats)}).encode()
    body = b"".join([MAGIC, struct.pack("<Q", len(header)), header, lengths.tobytes(), exps.tobytes(),
                     coeffs.tobytes(), pi.tobytes(), pj.tobytes()])
    return body + hashlib.sha256(body).digest()


def loads_state(blob: bytes):
    from .groebner import GroebnerState, Pair, _make_pair

    if blob[:8] != MAGIC:
        raise ValueError("not an F4B state snapshot")
    body, digest = blob[:-32], blob[-32:]
    if hashlib.sha256(body).digest() != digest:
        raise ValueError("snapshot checksum mismatch")
    (hl,) = struct.unpack("<Q", body[8:16])
    hdr = json.loads(body[16:16 + hl].decode())
    ring = Ring(hdr["vars"], hdr["order"], FieldModulus(hdr["p"]))
    n, G, T, P = ring.n_vars, hdr["G"], hdr["T"], hdr["P"]
    off = 16 + hl

    def take(dtype, count, shape=None):
        nonlocal off
        a = np.frombuffer(body, dtype=dtype, count=count, offset=off)
        off += a.nbytes
        return a.reshape(shape) if shape else a

    lengths = take(np.int64, G)
    exps = take(np.uint16, T * n, (T, n))
    coeffs = take(np.uint32, T)
    pi, pj = take(np.int64, P), take(np.int64, P)
    st = GroebnerState(ring)
    t = 0
    ex_l, cf_l = exps.tolist(), coeffs.tolist()
    for L in lengths.tolist():
        st._push_basis(Poly(ring, tuple((tuple(ex_l[k]), cf_l[k]) for k in range(t, t + L))))
        t += L
    st.pairs = sorted([_make_pair(st, int(i), int(j)) for i, j in zip(pi, pj)], key=Pair.sort_tuple)
    st.zero_reductions = hdr["zero_reductions"]
    return st


def save_state(state, path: str) -> None:
    with open(path, "wb") as fh:
        fh.write(dumps_state(state))


def load_state(path: str):
    with open(path, "rb") as fh:
        return loads_state(fh.read())
