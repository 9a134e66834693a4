"""Pin the CPU oracle to the REFERENCE (CPU suite).

Every F4 step of the committed reference snapshots is replayed through the
host pair logic (select_batch / select_rows) and the NumPy oracle; the plan
digest and RREF digest must equal the ones the real reference printed
(tests/golden/make_golden.py).  Also the reference's worked examples.
"""

import numpy as np
import pytest

import oracle
from conftest import load_golden, load_snapshots, state_from_snapshot
from paper_2601_06765_b200.fp import FieldModulus
from paper_2601_06765_b200.groebner import select_batch
from paper_2601_06765_b200.monomials import Ring, mon_key_pack
from paper_2601_06765_b200.polynomials import poly_parse, soa_pack
from paper_2601_06765_b200.symbolic import select_rows, BatchSpec, PairTarget

CONFIGS = ["cyclic5_p32003", "katsura5_p32003", "katsura6_p32003", "cyclic6_p32003"]


def _rows_arrays(rows):
    return [(r.shift, r.basis_index, r.role.value, r.provenance) for r in rows]


@pytest.mark.parametrize("name", CONFIGS)
def test_oracle_reproduces_reference_steps(name):
    gold = load_golden(name)
    snaps = load_snapshots(name)
    assert snaps, "snapshots missing"
    for k, snap in sorted(snaps.items()):
        ring, st = state_from_snapshot(snap)
        spec, degree = select_batch(st)
        assert degree == gold["steps"][k]["degree"]
        soa = st.soa()
        rows = select_rows(spec, soa)
        plan = oracle.compile_batch_arrays(_rows_arrays(rows), (soa.exps, soa.coeff, soa.offset, soa.length),
                                           ring.order)
        assert oracle.plan_sha256(plan, ring.modulus.p, ring.order, ring.var_names) == gold["steps"][k]["plan_sha256"]
        ech = oracle.psge_arrays(len(plan["row_ptr"]) - 1, plan["counters"]["N"], plan["row_ptr"], plan["col_ind"],
                                 plan["val"], ring.modulus.p)
        assert oracle.rref_sha256(ech["pivot_rows"], ech["nonpivot_rows"]) == gold["steps"][k]["rref_sha256"]
        assert ech["rank"] == gold["steps"][k]["rank"]


R2 = Ring(["x", "y"], "grevlex", FieldModulus(7))


def _two_poly_basis(extra=()):
    polys = [poly_parse("x^2 - y", R2), poly_parse("x*y - 1", R2)] + [poly_parse(t, R2) for t in extra]
    return soa_pack(polys, R2)


def _arrays(soa):
    return soa.exps, soa.coeff, soa.offset, soa.length


def test_oracle_worked_example_support_only():
    # reference tests/test_symbolic.py:71-85
    soa = _two_poly_basis()
    rows = select_rows(BatchSpec([PairTarget((2, 1), 0, 0, 1)], (0, 1)), soa)
    plan = oracle.compile_batch_arrays(_rows_arrays(rows), _arrays(soa), "grevlex", closure=False)
    assert [tuple(k) for k in plan["dict_keys"].tolist()] == [mon_key_pack(m, R2) for m in [(2, 1), (0, 2), (1, 0)]]
    assert plan["row_ptr"].tolist() == [0, 2, 4]
    assert plan["col_ind"].tolist() == [0, 1, 0, 2]
    assert plan["val"].tolist() == [1, 6, 1, 6]


def test_oracle_closure_chain():
    # reference tests/test_symbolic.py:122-139: x^3 -> x^2 -> x -> 1
    rx = Ring(["x"], "grevlex", FieldModulus(7))
    soa = soa_pack([poly_parse("x - 1", rx)], rx)
    plan = oracle.compile_batch_arrays([((2,), 0, 0, 0)], _arrays(soa), "grevlex")
    assert [m[0] for m in plan["row_meta"]] == [(2,), (1,), (0,)]
    assert plan["counters"]["closure_rounds"] == 2


def test_oracle_psge_worked_example():
    # reference tests/test_sparselin.py:133-142
    soa = _two_poly_basis()
    rows = select_rows(BatchSpec([PairTarget((2, 1), 0, 0, 1)], (0, 1)), soa)
    plan = oracle.compile_batch_arrays(_rows_arrays(rows), _arrays(soa), "grevlex", closure=False)
    e = oracle.psge_arrays(2, 3, plan["row_ptr"], plan["col_ind"], plan["val"], 7, panel_width=2)
    assert e["rank"] == 2 and e["pivot_cols"] == [0, 1]
    lead, cols, vals = e["nonpivot_rows"][0]
    assert lead == 1 and cols.tolist() == [1, 2] and vals.tolist() == [1, 6]


def test_oracle_psge_panel_width_invariance():
    rng = np.random.default_rng(860)
    p = 101
    mat = (rng.random((30, 25)) < 0.15) * rng.integers(1, p, (30, 25))
    rows, cols = np.nonzero(mat)
    rp = np.zeros(31, np.int64)
    np.cumsum(np.bincount(rows, minlength=30), out=rp[1:])
    digests = {oracle.rref_sha256(*(lambda e: (e["pivot_rows"], e["nonpivot_rows"]))(
        oracle.psge_arrays(30, 25, rp, cols, mat[rows, cols].astype(np.uint64), p, w))) for w in (1, 4, 64, 256)}
    assert len(digests) == 1


def test_oracle_berlekamp_massey_matches_reference_golden():
    """oracle.berlekamp_massey against the real reference's outputs
    (tests/golden/make_bm_golden.py: worked examples, LFSRs, random and
    Krylov-projection sequences over five primes)."""
    import gzip
    import json
    import os

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "bm_golden.json.gz")
    with gzip.open(path, "rt") as fh:
        cases = json.load(fh)["cases"]
    assert len(cases) > 60
    for c in cases:
        assert oracle.berlekamp_massey(c["seq"], c["p"]) == c["poly"]
