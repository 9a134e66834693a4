"""Oracle restatement of FBSP symbolic preprocessing (reference ``compile_batch``).

Plain NumPy over arrays.  TEST INFRASTRUCTURE ONLY (see ``oracle/__init__``).

Reference map (all paths under ``/root/reference/pkg/src/fpgb``):

* ``ref_keys``             — ``monomials.py:137-154`` (key_pack_vec) and
                             ``:157-172`` (key_unpack_vec)
* ``_lsd_radix_sort``      — ``bulk.py:86-124`` (8*W stable byte passes,
                             least significant word/byte first)
* ``_unique``              — ``bulk.py:135-150``
* ``_lower_bound``         — ``bulk.py:169-184``
* ``_materialize``         — ``symbolic.py:204-225`` (count -> scan -> fill)
* ``_closure_round``       — ``symbolic.py:228-278`` (reducer preference
                             = (key(LM), index); rows in ascending key(m))
* ``_merge``               — ``symbolic.py:281-290``
* ``compile_batch_arrays`` — ``symbolic.py:293-388`` (loop, join, counters)
* ``plan_text``            — ``symbolic.py:438-466``
"""

from __future__ import annotations

import hashlib

import numpy as np

DICT_CAP = 10**6  # symbolic.py:46
_LANE_MAX = 0xFFFF


class OracleError(Exception):
    """Raised with the reference exception name in ``kind``."""

    def __init__(self, kind, msg):
        self.kind = kind
        super().__init__(f"{kind}: {msg}")


def key_words(n_vars: int, order: str) -> int:
    head = 0 if order == "lex" else 32
    return (head + 16 * n_vars + 63) // 64


def ref_keys(exps: np.ndarray, order: str) -> np.ndarray:
    """Exponent rows -> reference big-endian keys (K, W) uint64."""
    exps = np.asarray(exps, dtype=np.int64)
    K, n = exps.shape
    if exps.size and (exps.min() < 0 or exps.max() > _LANE_MAX):
        raise OracleError("LaneOverflowError", "exponent does not fit a 16-bit lane")
    W = key_words(n, order)
    out = np.zeros((K, W), dtype=np.uint64)
    head = 0
    if order != "lex":
        out[:, 0] = exps.sum(axis=1).astype(np.uint64) << np.uint64(32)
        head = 32
    lanes = (_LANE_MAX - exps[:, ::-1]) if order == "grevlex" else exps
    lanes = lanes.astype(np.uint64)
    for i in range(n):
        bit = head + 16 * i
        out[:, bit // 64] |= lanes[:, i] << np.uint64(48 - bit % 64)
    return out


def ref_unkeys(keys: np.ndarray, n: int, order: str) -> np.ndarray:
    keys = np.asarray(keys, dtype=np.uint64)
    head = 0 if order == "lex" else 32
    lanes = np.empty((keys.shape[0], n), dtype=np.int64)
    for i in range(n):
        bit = head + 16 * i
        lanes[:, i] = ((keys[:, bit // 64] >> np.uint64(48 - bit % 64)) & np.uint64(0xFFFF)).astype(np.int64)
    return (_LANE_MAX - lanes)[:, ::-1] if order == "grevlex" else lanes


def _cmp_lt(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Row-wise a < b for word matrices (most significant word first)."""
    lt = np.zeros(a.shape[0], dtype=bool)
    eq = np.ones(a.shape[0], dtype=bool)
    for w in range(a.shape[1]):
        lt |= eq & (a[:, w] < b[:, w])
        eq &= a[:, w] == b[:, w]
    return lt


def _lsd_radix_sort(keys: np.ndarray) -> np.ndarray:
    """Stable LSD radix sort of word rows, one byte per pass (8*W passes)."""
    perm = np.arange(keys.shape[0], dtype=np.int64)
    if keys.shape[0] <= 1:
        return keys.copy()
    for w in reversed(range(keys.shape[1])):
        col = keys[:, w]
        for byte in range(8):
            digit = (col[perm] >> np.uint64(8 * byte)) & np.uint64(0xFF)
            perm = perm[np.argsort(digit, kind="stable")]
    return keys[perm]


def _unique(sorted_keys: np.ndarray) -> np.ndarray:
    if sorted_keys.shape[0] == 0:
        return sorted_keys.copy()
    head = np.ones(sorted_keys.shape[0], dtype=bool)
    head[1:] = (sorted_keys[1:] != sorted_keys[:-1]).any(axis=1)
    return sorted_keys[head]


def _lower_bound(table: np.ndarray, q: np.ndarray) -> np.ndarray:
    lo = np.zeros(q.shape[0], dtype=np.int64)
    hi = np.full(q.shape[0], table.shape[0], dtype=np.int64)
    live = lo < hi
    while live.any():
        idx = np.flatnonzero(live)
        mid = (lo[idx] + hi[idx]) >> 1
        go_right = _cmp_lt(table[mid], q[idx])
        lo[idx[go_right]] = mid[go_right] + 1
        hi[idx[~go_right]] = mid[~go_right]
        live = lo < hi
    return lo


def _materialize(rows, basis, order):
    """Pass 1: lens/offsets.  Pass 2: gathered, shifted, packed keys + coeffs."""
    exps, coeff, offset, length = basis
    n = exps.shape[1]
    ks = np.fromiter((r[1] for r in rows), dtype=np.int64, count=len(rows))
    shifts = np.asarray([r[0] for r in rows], dtype=np.int64).reshape(len(rows), n)
    lens = length[ks]
    if (lens < 1).any():
        raise OracleError("PropertyViolationError", "zero polynomial referenced as a reducer")
    starts = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(lens, out=starts[1:])
    total = int(starts[-1])
    row_of = np.repeat(np.arange(len(rows)), lens)
    src = offset[ks][row_of] + (np.arange(total) - starts[:-1][row_of])
    keys = ref_keys(exps[src] + shifts[row_of], order)
    return lens, keys, coeff[src].astype(np.uint64), keys[starts[:-1]]


def _closure_round(dict_desc, done_desc, basis, order, candidates, round_id):
    exps, _, offset, length = basis
    n = exps.shape[1]
    todo = np.flatnonzero(~done_desc)
    if todo.size == 0:
        return []
    mons = ref_unkeys(dict_desc[todo], n, order)
    lms = exps[offset[np.asarray(candidates, dtype=np.int64)]]
    lm_keys = ref_keys(lms, order)
    pref = sorted(range(len(candidates)),
                  key=lambda c: (tuple(int(w) for w in lm_keys[c]), candidates[c]))
    red = np.full(todo.size, -1, dtype=np.int64)
    for c in pref:
        hit = (red < 0) & (mons >= lms[c]).all(axis=1)
        red[hit] = candidates[c]
    out = []
    for j in range(todo.size - 1, -1, -1):  # ascending key(m)
        k = int(red[j])
        if k >= 0:
            shift = tuple(int(x) for x in (mons[j] - exps[offset[k]]))
            out.append((shift, k, 1, round_id))
    return out


def _merge(dict_asc, done, new_unique):
    merged = _unique(_lsd_radix_sort(np.vstack([dict_asc, new_unique])))
    nd = np.zeros(merged.shape[0], dtype=bool)
    if dict_asc.shape[0]:
        nd[_lower_bound(merged, dict_asc)] = done
    return merged, nd


def compile_batch_arrays(rows, basis, order, closure=True, candidates=None, dict_cap=DICT_CAP):
    """rows: list of (shift tuple, basis_index, role, provenance), in order.
    basis: (exps (T,n) i64, coeff (T,) u64, offset (G+1,) i64, length (G,) i64).
    Returns a dict with row_ptr, col_ind, val, dict_keys (descending), row_meta,
    counters (reference field names)."""
    exps = basis[0]
    n = exps.shape[1]
    W = key_words(n, order)
    rows = list(rows)
    counters = dict(r=0, N=0, M=0, nnz=0, closure_rounds=0, keys_emitted=0, keys_generated_total=0)
    if not rows:
        return dict(row_ptr=np.zeros(1, np.int64), col_ind=np.zeros(0, np.int64),
                    val=np.zeros(0, np.uint64), dict_keys=np.zeros((0, W), np.uint64),
                    row_meta=[], counters=counters)
    if candidates is None:
        candidates = list(range(len(basis[3])))
    lens, keys, vals, leads = _materialize(rows, basis, order)
    parts = [(lens, keys, vals)]
    lead_list = [leads]
    counters["keys_emitted"] += keys.shape[0]
    counters["keys_generated_total"] += keys.shape[0]
    dict_asc = _unique(_lsd_radix_sort(keys))
    done = np.zeros(dict_asc.shape[0], dtype=bool)
    while closure:
        done[_lower_bound(dict_asc, np.vstack(lead_list))] = True
        new_rows = _closure_round(dict_asc[::-1], done[::-1].copy(), basis, order,
                                  candidates, counters["closure_rounds"] + 1)
        done[:] = True
        if not new_rows:
            break
        counters["closure_rounds"] += 1
        rows.extend(new_rows)
        nl, nk, nv, nlead = _materialize(new_rows, basis, order)
        counters["keys_emitted"] += nk.shape[0]
        counters["keys_generated_total"] += nk.shape[0]
        parts.append((nl, nk, nv))
        lead_list.append(nlead)
        dict_asc, done = _merge(dict_asc, done, _unique(_lsd_radix_sort(nk)))
        if dict_asc.shape[0] > dict_cap:
            raise OracleError("SizeCapError", f"dictionary exceeded {dict_cap} entries")
    all_lens = np.concatenate([p[0] for p in parts])
    flat = np.vstack([p[1] for p in parts])
    row_ptr = np.zeros(all_lens.size + 1, dtype=np.int64)
    np.cumsum(all_lens, out=row_ptr[1:])
    pos = _lower_bound(dict_asc, flat)
    N = dict_asc.shape[0]
    clipped = np.minimum(pos, N - 1)
    if ((pos >= N) | (dict_asc[clipped] != flat).any(axis=1)).any():
        raise OracleError("MissingKeyError", "row key absent from dictionary")
    counters.update(r=len(rows), N=N, M=int(row_ptr[-1]), nnz=int(row_ptr[-1]))
    return dict(row_ptr=row_ptr, col_ind=(N - 1) - pos,
                val=np.concatenate([p[2] for p in parts]),
                dict_keys=dict_asc[::-1].copy(), row_meta=rows, counters=counters)


def plan_text(plan, p, order, var_names) -> str:
    """Canonical dump, byte-identical to reference ``plan_to_text``."""
    c = plan["counters"]
    meta = " ".join(",".join([str(e) for e in sh] + [str(k), str(role), str(prov)])
                    for sh, k, role, prov in plan["row_meta"])
    lines = [
        "fpgb-plan v1", f"p {p}", f"order {order}", "vars " + " ".join(var_names),
        f"counters r={c['r']} N={c['N']} M={c['M']} nnz={c['nnz']} "
        f"closure_rounds={c['closure_rounds']} keys_emitted={c['keys_emitted']} "
        f"keys_generated_total={c['keys_generated_total']}",
        "row_ptr " + " ".join(map(str, plan["row_ptr"].tolist())),
        "col_ind " + " ".join(map(str, plan["col_ind"].tolist())),
        "val " + " ".join(map(str, plan["val"].tolist())),
        "dict_keys " + " ".join(map(str, plan["dict_keys"].ravel().tolist())),
        "row_meta " + meta,
    ]
    return "\n".join(lines) + "\n"


def plan_sha256(plan, p, order, var_names) -> str:
    return hashlib.sha256(plan_text(plan, p, order, var_names).encode()).hexdigest()
