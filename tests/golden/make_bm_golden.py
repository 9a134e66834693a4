"""Golden Berlekamp–Massey vectors from the REAL reference (build container only).

Runs the reference's own ``fpgb.sparselin.berlekamp_massey`` (pkg/src/fpgb/
sparselin.py:377-413) on: the reference test's worked examples
(pkg/tests/test_sparselin.py:224-231), LFSR sequences, random sequences, and
Krylov projection sequences u^T A^k v of random sparse matrices (the shape
Block Wiedemann feeds it), over p in {31, 101, 32003, 65521, 2^31-1}.
Writes tests/golden/bm_golden.json.gz.  Usage: python tests/golden/make_bm_golden.py
"""
import gzip
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from fpgb.fp import FieldModulus  # noqa: E402
from fpgb.sparselin import berlekamp_massey  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def lfsr(rng, p, d, length):
    coeffs = [int(x) for x in rng.integers(0, p, d)]
    if coeffs[0] == 0:
        coeffs[0] = 1
    seq = [int(x) for x in rng.integers(0, p, d)]
    while len(seq) < length:
        k = len(seq)
        seq.append(sum(coeffs[i] * seq[k - 1 - i] for i in range(d)) % p)
    return seq


def krylov(rng, p, n, density, length):
    A = rng.integers(0, p, (n, n)) * (rng.random((n, n)) < density)
    u = rng.integers(0, p, n)
    v = rng.integers(0, p, n)
    out = []
    for _ in range(length):
        out.append(int(np.dot(u % p, v % p) % p))
        v = (A @ v) % p
    return out


def main():
    rng = np.random.default_rng(2026)
    cases = [(101, [5] * 8), (101, [1, 1, 2, 3, 5, 8, 13, 21]), (101, [3, 0, 0, 0, 0, 0]), (7, [0, 0, 0, 1]),
             (7, [0] * 5 + [2])]
    for p in (31, 101, 32003, 65521, 2147483647):
        for d in (1, 3, 17, 60):
            cases.append((p, lfsr(rng, p, d, 3 * d + 5)))
        for length in (1, 2, 9, 40, 257):
            cases.append((p, [int(x) for x in rng.integers(0, p, length)]))
        for n in (8, 40, 150):
            cases.append((p, krylov(rng, p, n, 0.1, 2 * n)))
    cases.append((31, lfsr(rng, 31, 300, 1200)))
    out = []
    for p, seq in cases:
        out.append({"p": p, "seq": seq, "poly": [int(c) for c in berlekamp_massey(seq, FieldModulus(p))]})
    with gzip.open(os.path.join(HERE, "bm_golden.json.gz"), "wt") as fh:
        json.dump({"source": "fpgb.sparselin.berlekamp_massey (reference)", "cases": out}, fh)
    print(len(out), "cases")


if __name__ == "__main__":
    main()
