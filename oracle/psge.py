"""Oracle restatement of panel-structured Gaussian elimination (``psge_reduce``).

TEST INFRASTRUCTURE ONLY.  Restates ``pkg/src/fpgb/sparselin.py``:

* ``_axpy``        — ``:267-278`` (a - c*b over sparse rows; fill count)
* ``psge_arrays``  — ``:281-369`` (column panels ascending; pivot = fewest
                     nonzeros then lowest index (:316); normalize; eliminate
                     the other rows leading at that column; full
                     back-reduction (:337-349); split rows by whether the
                     lead column was a lead of some input row (:351-360))
* ``rref_sha256``  — the RREF digest recipe of SURVEY.md Appendix A.

Arithmetic is the reference's NAIVE backend (standard residues, ``%``); the
reference requires all backends to agree byte for byte, so this pins them all.
"""

from __future__ import annotations

import hashlib

import numpy as np


def _axpy(ca, va, coef, cb, vb, p):
    cols = np.union1d(ca, cb)
    a = np.zeros(cols.size, dtype=np.uint64)
    a[np.searchsorted(cols, ca)] = va
    b = np.zeros(cols.size, dtype=np.uint64)
    b[np.searchsorted(cols, cb)] = vb
    out = (a + (np.uint64(p) - (b * np.uint64(coef)) % np.uint64(p))) % np.uint64(p)
    nz = out != 0
    return cols[nz], out[nz], int((nz & (a == 0)).sum())


def psge_arrays(n_rows, n_cols, row_ptr, col_ind, val, p, panel_width=256):
    if panel_width < 1:
        raise ValueError("PreconditionError: panel_width must be >= 1")
    rows = []
    leads_in = set()
    by_lead: dict = {}
    zero = 0
    for i in range(n_rows):
        s, e = int(row_ptr[i]), int(row_ptr[i + 1])
        if e == s:
            rows.append(None)
            zero += 1
            continue
        c = np.asarray(col_ind[s:e], dtype=np.int64).copy()
        rows.append([c, np.asarray(val[s:e], dtype=np.uint64).copy()])
        leads_in.add(int(c[0]))
        by_lead.setdefault(int(c[0]), []).append(i)
    piv: dict = {}
    fill = 0
    for start in range(0, max(n_cols, 1), panel_width):
        for col in range(start, min(n_cols, start + panel_width)):
            cand = by_lead.pop(col, None)
            if not cand:
                continue
            pv = min(sorted(cand), key=lambda i: (rows[i][0].size, i))
            inv = pow(int(rows[pv][1][0]), p - 2, p)
            rows[pv][1] = (rows[pv][1] * np.uint64(inv)) % np.uint64(p)
            piv[col] = pv
            for i in cand:
                if i == pv:
                    continue
                c, v, made = _axpy(rows[i][0], rows[i][1], int(rows[i][1][0]), rows[pv][0], rows[pv][1], p)
                fill += made
                if c.size == 0:
                    rows[i] = None
                    zero += 1
                else:
                    rows[i] = [c, v]
                    by_lead.setdefault(int(c[0]), []).append(i)
    for col in sorted(piv, reverse=True):
        pv = piv[col]
        for qcol, q in piv.items():
            if q == pv or qcol >= col:
                continue
            cq, vq = rows[q]
            at = int(np.searchsorted(cq, col))
            if at < cq.size and cq[at] == col:
                c, v, made = _axpy(cq, vq, int(vq[at]), rows[pv][0], rows[pv][1], p)
                fill += made
                rows[q] = [c, v]
    pivot_rows, nonpivot_rows = [], []
    for col in sorted(piv):
        c, v = rows[piv[col]]
        (pivot_rows if col in leads_in else nonpivot_rows).append((col, c, v))
    return dict(pivot_cols=sorted(piv), pivot_rows=pivot_rows, nonpivot_rows=nonpivot_rows,
                zero_row_count=n_rows - len(piv), rank=len(piv), fill_generated=fill)


def rref_sha256(pivot_rows, nonpivot_rows) -> str:
    h = hashlib.sha256()
    for lead, cols, vals in list(pivot_rows) + list(nonpivot_rows):
        h.update(f"{int(lead)}:{np.asarray(cols).tolist()}:{np.asarray(vals).tolist()};".encode())
    return h.hexdigest()
