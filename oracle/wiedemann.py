"""Berlekamp–Massey restated (reference pkg/src/fpgb/sparselin.py:377-413).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): the checker for the
device recurrence ``k_bm`` (paper_2601_06765_b200/csrc/bm.cu).  Pinned to the
real reference by tests/golden/bm_golden.json.gz (tests/golden/make_bm_golden.py
runs the reference's own ``berlekamp_massey`` on the recorded sequences).
"""


def berlekamp_massey(seq, p: int) -> list:
    """Minimal recurrence of ``seq`` over F_p as the ascending monic
    characteristic polynomial (reference sparselin.py:377-413: connection
    polynomial ``conn``, previous ``prev``, length ``L``, shift ``gap``, last
    nonzero discrepancy ``last_d``; update when ``2L <= n``)."""
    s = [int(x) % p for x in seq]
    if not s:
        raise ValueError("empty sequence")
    conn, prev = [1], [1]
    L, gap, last_d = 0, 1, 1
    for n, sn in enumerate(s):
        d = sn
        for i in range(1, L + 1):
            d = (d + conn[i] * s[n - i]) % p
        if d == 0:
            gap += 1
            continue
        scale = d * pow(last_d, p - 2, p) % p
        need = len(prev) + gap
        nxt = conn + [0] * max(0, need - len(conn))
        for i, b in enumerate(prev):
            nxt[i + gap] = (nxt[i + gap] - scale * b) % p
        if 2 * L <= n:
            prev, L, last_d, gap = conn, n + 1 - L, d, 1
        else:
            gap += 1
        conn = nxt
    conn = conn[:L + 1] + [0] * max(0, L + 1 - len(conn))
    return [c % p for c in reversed(conn)]
