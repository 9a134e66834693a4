"""GPU parity: the CUDA path (through the Python API over the C ABI) against
the CPU oracle on seeded inputs and against the reference's golden digests.

Tolerance: none — everything is exact integer arithmetic mod p, so every
comparison is byte equality (plan_to_text / RREF digests / arrays)."""

import hashlib
import os

import numpy as np
import pytest

import oracle
from conftest import load_golden, load_snapshots, state_from_snapshot
from paper_2601_06765_b200 import errors
from paper_2601_06765_b200.fp import FieldModulus
from paper_2601_06765_b200.groebner import GroebnerState, f4_groebner, f4_step, select_batch, update_pairs
from paper_2601_06765_b200.monomials import Ring, mon_key_pack
from paper_2601_06765_b200.polynomials import poly_monic, poly_parse, soa_pack, poly_normalize
from paper_2601_06765_b200.sparselin import (CsrMatrix, KernelMode, csr_from_arrays, csr_from_dense, csr_from_plan,
                                             left_kernel, psge_reduce, spmm, spmv, wiedemann_solve)
from paper_2601_06765_b200.symbolic import (BatchSpec, Closure, PairTarget, Row, RowRole, compile_batch, plan_digest,
                                            plan_to_text, select_rows)
from paper_2601_06765_b200.systems import format_system, gen_cyclic, gen_katsura

pytestmark = pytest.mark.gpu

M7 = FieldModulus(7)
R2 = Ring(["x", "y"], "grevlex", M7)


def _oracle_plan(rows, soa, closure=True):
    return oracle.compile_batch_arrays([(r.shift, r.basis_index, r.role.value, r.provenance) for r in rows],
                                       (soa.exps, soa.coeff, soa.offset, soa.length), soa.ring.order, closure=closure)


def _check_plan(plan, rows, soa, closure=True):
    ring = soa.ring
    ref = _oracle_plan(rows, soa, closure)
    assert plan_to_text(plan) == oracle.plan_text(ref, ring.modulus.p, ring.order, ring.var_names)
    return ref


def _rref_digest(ech):
    return oracle.rref_sha256(ech.pivot_rows, ech.nonpivot_rows)


# ---------------------------------------------------------------------------
# compile_batch: worked examples and edge cases (reference tests/test_symbolic.py)
# ---------------------------------------------------------------------------
def test_compile_worked_example(cuda):
    soa = soa_pack([poly_parse("x^2 - y", R2), poly_parse("x*y - 1", R2)], R2)
    rows = select_rows(BatchSpec([PairTarget((2, 1), 0, 0, 1)], (0, 1)), soa)
    plan = compile_batch(rows, soa, Closure.SUPPORT_ONLY)
    assert [tuple(k) for k in plan.dict_keys.tolist()] == [mon_key_pack(m, R2) for m in [(2, 1), (0, 2), (1, 0)]]
    assert plan.row_ptr.tolist() == [0, 2, 4] and plan.col_ind.tolist() == [0, 1, 0, 2]
    assert plan.val.tolist() == [1, 6, 1, 6]
    plan.validate()
    ech = psge_reduce(csr_from_plan(plan, M7), panel_width=2)
    assert ech.rank == 2 and ech.pivot_cols == [0, 1]
    lead, cols, vals = ech.nonpivot_rows[0]
    assert lead == 1 and cols.tolist() == [1, 2] and vals.tolist() == [1, 6]


def test_compile_closure_examples(cuda):
    soa = soa_pack([poly_parse(t, R2) for t in ("x^2 - y", "x*y - 1", "y^2 - 1")], R2)
    rows = select_rows(BatchSpec([PairTarget((2, 1), 0, 0, 1)], (0, 1)), soa)
    plan = compile_batch(rows, soa, Closure.ONE_STEP_REDUCTION)
    assert [r.role for r in plan.row_meta] == [RowRole.SPOLY_HALF, RowRole.SPOLY_HALF, RowRole.REDUCER]
    assert plan.row_meta[2].shift == (0, 0) and plan.row_meta[2].basis_index == 2
    assert plan.counters.closure_rounds == 1
    _check_plan(plan, rows, soa)
    rx = Ring(["x"], "grevlex", M7)
    gb = soa_pack([poly_parse("x - 1", rx)], rx)
    seed = [Row((2,), 0, RowRole.SPOLY_HALF, 0)]
    plan = compile_batch(seed, gb, Closure.ONE_STEP_REDUCTION)
    assert [r.shift for r in plan.row_meta] == [(2,), (1,), (0,)]
    assert [tuple(k) for k in plan.dict_keys.tolist()] == [mon_key_pack((e,), rx) for e in (3, 2, 1, 0)]


def test_compile_edge_cases(cuda):
    soa = soa_pack([poly_parse("x^2 - y", R2), poly_parse("x*y - 1", R2)], R2)
    empty = compile_batch([], soa)
    assert empty.row_ptr.tolist() == [0] and empty.counters.N == 0 and empty.dict_keys.shape == (0, R2.n_key_words)
    with pytest.raises(errors.LaneOverflowError):
        compile_batch([Row((65535, 0), 0, RowRole.SPOLY_HALF, 0)], soa)
    zsoa = soa_pack([poly_parse("x - 1", R2), poly_parse("0", R2)], R2)
    with pytest.raises(errors.PropertyViolationError):
        compile_batch([Row((0, 1), 1, RowRole.SPOLY_HALF, 0)], zsoa)
    import paper_2601_06765_b200.symbolic as sym

    rx = Ring(["x"], "grevlex", M7)
    gb = soa_pack([poly_parse("x - 1", rx)], rx)
    old = sym.DICT_CAP
    sym.DICT_CAP = 10
    try:
        with pytest.raises(errors.SizeCapError):
            compile_batch([Row((50,), 0, RowRole.SPOLY_HALF, 0)], gb, Closure.ONE_STEP_REDUCTION)
    finally:
        sym.DICT_CAP = old


def _random_poly(rng, ring, max_exp, terms):
    ts = [(tuple(int(x) for x in rng.integers(0, max_exp + 1, ring.n_vars)), int(rng.integers(1, ring.modulus.p)))
          for _ in range(terms)]
    return poly_monic(poly_normalize(ts, ring))


@pytest.fixture(params=["rank", "sort", "multi"])
def dict_mode(request, force_option):
    """Every dictionary path: the rank bitmap in one cooperative k_fbsp
    (grevlex default), the same phases as separate launches (the sharded
    compile's building blocks) and the radix sort (lex / deglex default)."""
    if request.param == "sort":
        force_option("dict_sort", 1)
    elif request.param == "multi":
        force_option("fbsp", 1)
    return request.param


@pytest.mark.parametrize("order,n,max_exp,p", [("grevlex", 2, 3, 7), ("grevlex", 5, 4, 32003),
                                               ("deglex", 4, 3, 101), ("lex", 3, 3, 65521),
                                               ("lex", 6, 2, 101), ("grevlex", 9, 2, 2147483629),
                                               ("grevlex", 3, 40, 32003)])
def test_compile_random_against_oracle(cuda, dict_mode, order, n, max_exp, p):
    ring = Ring([f"v{i}" for i in range(n)], order, FieldModulus(p))
    rng = np.random.default_rng(n * 1000 + max_exp)
    for trial in range(6):
        polys = []
        while len(polys) < 5:
            f = _random_poly(rng, ring, max_exp, int(rng.integers(1, 12)))
            if not f.is_zero():
                polys.append(f)
        soa = soa_pack(polys, ring)
        rows = sorted({Row(tuple(int(x) for x in rng.integers(0, 3, n)), int(rng.integers(0, 5)),
                           RowRole.SPOLY_HALF, int(rng.integers(0, 4))) for _ in range(int(rng.integers(1, 9)))},
                      key=lambda r: (r.provenance, mon_key_pack(r.shift, ring), r.basis_index))
        for closure in (Closure.SUPPORT_ONLY, Closure.ONE_STEP_REDUCTION):
            plan = compile_batch(rows, soa, closure)
            _check_plan(plan, rows, soa, closure is Closure.ONE_STEP_REDUCTION)
            # the copy-stream download of every dictionary path equals the synchronous one
            pf = compile_batch(rows, soa, closure).prefetch()
            for k in ("row_ptr", "col_ind", "val", "dict_keys"):
                assert np.array_equal(getattr(pf, k), getattr(plan, k)), k


# ---------------------------------------------------------------------------
# psge_reduce against the oracle (reference tests/test_sparselin.py)
# ---------------------------------------------------------------------------
def _random_sparse(rng, r, c, density, p):
    mat = (rng.random((r, c)) < density) * rng.integers(1, p, (r, c), dtype=np.int64)
    return mat.astype(np.uint64)


def _oracle_rref(mat, p):
    A = csr_from_dense(mat, FieldModulus(p))
    e = oracle.psge_arrays(A.n_rows, A.n_cols, A.row_ptr, A.col_ind, A.val, p)
    return e, oracle.rref_sha256(e["pivot_rows"], e["nonpivot_rows"])


@pytest.mark.parametrize("p", [7, 101, 32003, 65521, 1048573, 2147483629])
@pytest.mark.parametrize("density", [0.01, 0.05, 0.2, 0.6])
def test_psge_random_against_oracle(cuda, p, density):
    m = FieldModulus(p)
    rng = np.random.default_rng(p % 997 + int(density * 1000))
    for _ in range(5):
        r, c = (int(x) for x in rng.integers(5, 90, 2))
        mat = _random_sparse(rng, r, c, density, p)
        if rng.random() < 0.5:  # duplicate rows -> zero reductions
            mat[rng.integers(0, r, r // 3)] = mat[rng.integers(0, r, r // 3)]
        e, want = _oracle_rref(mat, p)
        ech = psge_reduce(csr_from_dense(mat, m), panel_width=int(rng.integers(1, 17)))
        assert ech.rank == e["rank"] and ech.zero_row_count == e["zero_row_count"]
        assert ech.pivot_cols == e["pivot_cols"]
        assert _rref_digest(ech) == want


@pytest.mark.parametrize("p", [32003, 1048573])
def test_psge_many_windows_against_oracle(cuda, p):
    """Hundreds of C rows over several 32-column A windows: the windowed
    sweep (packed tails for p < 2^16, (col, val) pairs above) and the D'
    stage against the oracle."""
    m = FieldModulus(p)
    rng = np.random.default_rng(p % 1009)
    r, c = 420, 360
    mat = _random_sparse(rng, r, c, 0.04, p)
    mat[rng.integers(0, r, r // 4)] = mat[rng.integers(0, r, r // 4)]
    e, want = _oracle_rref(mat, p)
    ech = psge_reduce(csr_from_dense(mat, m))
    assert ech.rank == e["rank"] and ech.zero_row_count == e["zero_row_count"]
    assert ech.pivot_cols == e["pivot_cols"]
    assert _rref_digest(ech) == want


def test_psge_zero_and_empty(cuda):
    A = CsrMatrix(3, 4, np.zeros(4, np.int64), np.zeros(0, np.int64), np.zeros(0, np.uint64), M7)
    res = psge_reduce(A)
    assert res.rank == 0 and res.zero_row_count == 3 and res.pivot_cols == []
    with pytest.raises(errors.PreconditionError):
        psge_reduce(A, panel_width=0)
    res = psge_reduce(csr_from_dense(np.array([[1, 2, 0], [0, 1, 3], [0, 0, 1]], dtype=np.uint64), M7))
    assert res.rank == 3 and res.pivot_cols == [0, 1, 2] and res.zero_row_count == 0


def test_psge_wide_matrix_global_accumulator(cuda):
    # N beyond the shared-memory accumulator (200 KB) exercises the HBM path
    p = 32003
    rng = np.random.default_rng(5)
    r, c = 120, 60000
    rows, cols, vals = [], [], []
    for i in range(r):
        k = rng.choice(c, 40, replace=False)
        k.sort()
        rows += [i] * 40
        cols += k.tolist()
        vals += rng.integers(1, p, 40).tolist()
    rp = np.zeros(r + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=r), out=rp[1:])
    A = csr_from_arrays(r, c, rp, np.asarray(cols), np.asarray(vals, dtype=np.uint64), FieldModulus(p))
    e = oracle.psge_arrays(r, c, A.row_ptr, A.col_ind, A.val, p)
    ech = psge_reduce(A)
    assert _rref_digest(ech) == oracle.rref_sha256(e["pivot_rows"], e["nonpivot_rows"])


# ---------------------------------------------------------------------------
# whole F4 runs against the reference's per-step digests
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,gen,args", [("cyclic5_p32003", gen_cyclic, (5, 32003)),
                                           ("cyclic6_p32003", gen_cyclic, (6, 32003)),
                                           ("katsura5_p32003", gen_katsura, (5, 32003)),
                                           ("katsura6_p32003", gen_katsura, (6, 32003)),
                                           ("katsura8_p32003", gen_katsura, (8, 32003)),
                                           ("cyclic7_p65521", gen_cyclic, (7, 65521))])
def test_f4_steps_match_reference(cuda, name, gen, args):
    gold = load_golden(name)
    ring, polys = gen(*args)
    st = GroebnerState(ring)
    for f in polys:
        update_pairs(st, poly_monic(f))
    k = 0
    while st.n_pairs():
        plan, ech, _ = f4_step(st)
        g = gold["steps"][k]
        assert (plan.counters.r, plan.counters.N, plan.counters.M, plan.counters.closure_rounds) == \
            (g["r"], g["N"], g["M"], g["closure_rounds"]), f"step {k}"
        assert plan_digest(plan) == g["plan_sha256"], f"plan step {k}"
        assert _rref_digest(ech) == g["rref_sha256"], f"rref step {k}"
        k += 1
    assert k == len(gold["steps"])
    from paper_2601_06765_b200.groebner import reduce_basis

    text = format_system(ring, reduce_basis(st.basis, ring))
    assert hashlib.sha256(text.encode()).hexdigest() == gold["final_sha256"]


@pytest.mark.parametrize("name,gen,args", [("cyclic6_p32003", gen_cyclic, (6, 32003)),
                                           ("katsura6_p32003", gen_katsura, (6, 32003))])
def test_f4_steps_match_reference_sort_path(cuda, force_option, name, gen, args):
    """Same per-step digests with the radix-sort dictionary forced."""
    force_option("dict_sort", 1)
    gold = load_golden(name)
    ring, polys = gen(*args)
    st = GroebnerState(ring)
    for f in polys:
        update_pairs(st, poly_monic(f))
    k = 0
    while st.n_pairs():
        plan, ech, _ = f4_step(st)
        assert plan_digest(plan) == gold["steps"][k]["plan_sha256"], f"plan step {k}"
        assert _rref_digest(ech) == gold["steps"][k]["rref_sha256"], f"rref step {k}"
        k += 1


_FALLBACK_KERNELS = {("dict_sort", 1): "k_tile_dict", ("fbsp", 1): "k_rank_fill", ("sweep", 1): "k_sweep_blk",
                     ("sweep", 2): "k_sweep<0", ("dense", 1): "k_dense_forward",
                     ("dense_rows", 1): "k_dense_blk"}


@pytest.mark.parametrize("name", ["cyclic8_p32003", "katsura11_p32003"])
@pytest.mark.parametrize("option", list(_FALLBACK_KERNELS))
def test_large_step_replay_fallback_paths(cuda, force_option, name, option):
    """The north-star replays through every fallback path: radix-sort
    dictionary, multi-launch rank pipeline, blocked / generic C-row sweeps and
    the per-pivot D' elimination (each forced via f4b_ctx_set_option), with
    the in-library launch profile proving the forced kernel ran."""
    from paper_2601_06765_b200.engine import Engine

    force_option(*option)
    ring, _ = state_from_snapshot(next(iter(load_snapshots(name).values())))
    eng = Engine.for_ring(ring)
    eng.profile(True)
    test_large_step_replay(cuda, name)
    prof, _ = eng.profile_read()
    eng.profile(False)
    assert any(k.startswith(_FALLBACK_KERNELS[option]) for k in prof), sorted(prof)


def test_f4_groebner_entry_point(cuda):
    ring, polys = gen_cyclic(6, 32003)
    gb = f4_groebner(polys, ring)
    assert hashlib.sha256(format_system(ring, gb).encode()).hexdigest() == \
        load_golden("cyclic6_p32003")["final_sha256"]


@pytest.mark.parametrize("name", ["cyclic8_p32003", "katsura11_p32003", "mq16x32_p31", "cyclic7_p65521"])
def test_large_step_replay(cuda, name):
    """Full-size steps replayed from reference snapshots (north-star configs)."""
    snaps = load_snapshots(name)
    if not snaps:
        pytest.skip(f"no snapshots for {name}")
    gold = load_golden(name)
    for k, snap in sorted(snaps.items()):
        if k >= len(gold["steps"]):
            continue
        ring, st = state_from_snapshot(snap)
        spec, _ = select_batch(st)
        soa = st.soa()
        rows = select_rows(spec, soa)
        plan = compile_batch(rows, soa, Closure.ONE_STEP_REDUCTION)
        assert plan_digest(plan) == gold["steps"][k]["plan_sha256"], f"plan step {k}"
        ech = psge_reduce(csr_from_plan(plan, ring.modulus))
        assert _rref_digest(ech) == gold["steps"][k]["rref_sha256"], f"rref step {k}"


# ---------------------------------------------------------------------------
# SpMM / Wiedemann / left kernel (reference tests/test_sparselin.py:100-306)
# ---------------------------------------------------------------------------
def test_spmm_matches_numpy(cuda):
    for p in (101, 32003, 2147483629):
        m = FieldModulus(p)
        rng = np.random.default_rng(p % 1000)
        mat = _random_sparse(rng, 70, 50, 0.2, p)
        X = rng.integers(0, p, (50, 4), dtype=np.uint64)
        want = np.zeros((70, 4), dtype=object)
        for i in range(70):
            for j in range(4):
                want[i, j] = sum(int(a) * int(b) for a, b in zip(mat[i], X[:, j])) % p
        got = spmm(csr_from_dense(mat, m), X)
        assert np.array_equal(got.astype(object), want)
        assert np.array_equal(spmv(csr_from_dense(mat, m), X[:, 0]).astype(object), want[:, 0])


def test_left_kernel_small(cuda):
    kb = left_kernel(csr_from_dense(np.array([[1, 2, 3], [1, 2, 3]], dtype=np.uint64), M7), count=4, seed=0)
    assert kb.side == "left" and kb.dimension_found == 1
    v = kb.vectors[0]
    assert (int(v[0]) + int(v[1])) % 7 == 0 and v[0] != 0
    kb = left_kernel(csr_from_dense(np.array([[1, 0, 0], [0, 1, 0]], dtype=np.uint64), M7), count=4, seed=0)
    assert kb.dimension_found == 0


def test_wiedemann_nullity(cuda):
    m = FieldModulus(2147483629)
    rng = np.random.default_rng(31415)
    n, rank = 40, 34
    Lf = rng.integers(0, m.p, (n, rank), dtype=np.uint64)
    Rf = rng.integers(0, m.p, (rank, n), dtype=np.uint64)
    mat = np.array([[sum(int(Lf[i, k]) * int(Rf[k, j]) for k in range(rank)) % m.p for j in range(n)]
                    for i in range(n)], dtype=np.uint64)
    A = csr_from_dense(mat, m)
    kb = wiedemann_solve(A, KernelMode.RIGHT_KERNEL, seed=0)
    assert kb.dimension_found == n - psge_reduce(A).rank
    for v in kb.vectors:
        assert (spmv(A, v) == 0).all()
    eye = csr_from_dense(np.eye(3, dtype=np.uint64), FieldModulus(101))
    assert wiedemann_solve(eye, KernelMode.MINPOLY, seed=11) == [100, 1]


def test_basis_append_wide_matches_narrow(cuda):
    """f4b_basis_append_wide (reference int64 / uint64 streams, narrowed and
    checked on the device) == f4b_basis_append (host-narrowed u16 / u32)."""
    from paper_2601_06765_b200.engine import Engine

    rng = np.random.default_rng(7)
    ring = Ring(["a", "b", "c", "d"], "grevlex", FieldModulus(32003))
    polys = [_random_poly(rng, ring, 5, 12) for _ in range(9)]
    soa = soa_pack(polys, ring)
    rows = [Row(tuple(int(x) for x in rng.integers(0, 3, 4)), int(k), RowRole.SPOLY_HALF, 0) for k in range(9)]
    eng = Engine.for_ring(ring)
    eng.clear_basis()
    eng.append_polys(soa.length, soa.exps, soa.coeff)  # int64 / uint64 -> wide path
    plan_w = eng.compile(np.array([r.basis_index for r in rows]), np.array([r.shift for r in rows]), True)
    dw = plan_w.download()
    eng.clear_basis()
    eng.append_polys(soa.length, soa.exps.astype(np.uint16), soa.coeff.astype(np.uint32))  # narrow path
    plan_n = eng.compile(np.array([r.basis_index for r in rows]), np.array([r.shift for r in rows]), True)
    dn = plan_n.download()
    for k in dw:
        assert np.array_equal(dw[k], dn[k]), k
    keys = plan_w.download_ref_keys(ring.n_key_words)
    from paper_2601_06765_b200.monomials import key_pack_vec

    assert np.array_equal(keys, key_pack_vec(dw["dict_exps"].astype(np.int64), ring))
    eng.clear_basis()
    bad = soa.exps.copy()
    bad[3, 1] = 70000
    with pytest.raises(errors.LaneOverflowError):
        eng.append_polys(soa.length, bad, soa.coeff)
    badc = soa.coeff.copy()
    badc[5] = 0
    with pytest.raises(errors.PropertyViolationError):
        eng.append_polys(soa.length, soa.exps, badc)
    eng.clear_basis()


@pytest.mark.parametrize("order", ["grevlex", "deglex", "lex"])
def test_basis_append_keys_matches_exps(cuda, order):
    """f4b_basis_append_keys_async (the SoaPolySet's reference keys uploaded
    instead of the int64 exponent rows, lanes unpacked on the device) builds
    the same device basis as the exponent path; a corrupt key (degree lane
    != lane sum, or nonzero padding) is PropertyViolationError."""
    from paper_2601_06765_b200.engine import Engine

    rng = np.random.default_rng(11)
    ring = Ring(["a", "b", "c", "d", "e", "f"], order, FieldModulus(32003))
    assert ring.n_key_words < ring.n_vars
    polys = [_random_poly(rng, ring, 5, 12) for _ in range(9)]
    soa = soa_pack(polys, ring)
    rows = [Row(tuple(int(x) for x in rng.integers(0, 3, 6)), int(k), RowRole.SPOLY_HALF, 0) for k in range(9)]
    rb, sh = np.array([r.basis_index for r in rows]), np.array([r.shift for r in rows])
    eng = Engine.for_ring(ring)
    got = []
    for keys in (soa.mon_key, None):
        eng.clear_basis()
        eng.append_polys(soa.length, soa.exps, soa.coeff, defer=True, keys=keys)
        got.append(eng.compile(rb, sh, True).download())
    for k in got[0]:
        assert np.array_equal(got[0][k], got[1][k]), k
    # a shift that passes on the exact maximum exponent but not on the deg(LM)
    # bound the pending key append starts from: both paths compile it alike
    g = 0
    mx = int(soa.exps[soa.offset[g]:soa.offset[g + 1], 0].max())
    if ring.graded and int(soa.exps[soa.offset[g]].sum()) > mx:
        sh1 = np.zeros((1, 6), np.int64)
        sh1[0, 0] = 0xFFFF - mx
        res = []
        for keys in (soa.mon_key, None):
            eng.clear_basis()
            eng.append_polys(soa.length, soa.exps, soa.coeff, defer=True, keys=keys)
            try:
                res.append(eng.compile(np.array([g]), sh1, False).download())
            except errors.FpgbError as e:
                res.append(type(e))
        if isinstance(res[0], dict):
            assert isinstance(res[1], dict) and all(np.array_equal(res[0][k], res[1][k]) for k in res[0])
        else:
            assert res[0] == res[1]
    bad = soa.mon_key.copy()
    if ring.graded:
        bad[4, 0] += np.uint64(1 << 32)  # degree lane off by one
    else:
        bad[4, -1] |= np.uint64(1)  # padding bit below the last lane
    eng.clear_basis()
    eng.append_polys(soa.length, soa.exps, soa.coeff, defer=True, keys=bad)
    with pytest.raises(errors.PropertyViolationError):
        eng.compile(rb, sh, True)
    eng.clear_basis()


@pytest.mark.parametrize("name,gen,args", [("cyclic5_p32003", gen_cyclic, (5, 32003)),
                                           ("katsura6_p32003", gen_katsura, (6, 32003))])
def test_reduce_basis_device_matches_host(cuda, name, gen, args):
    """§8f.1: the final interreduction as one Macaulay matrix on the GPU equals
    the reference's normal-form loop (host reduce_basis) and the golden digest."""
    from paper_2601_06765_b200.groebner import reduce_basis, reduce_basis_device

    ring, polys = gen(*args)
    st = GroebnerState(ring)
    for f in polys:
        update_pairs(st, poly_monic(f))
    while st.n_pairs():
        f4_step(st)
    dev = reduce_basis_device(st.basis, ring)
    host = reduce_basis(st.basis, ring)
    assert format_system(ring, dev) == format_system(ring, host)
    assert hashlib.sha256(format_system(ring, dev).encode()).hexdigest() == load_golden(name)["final_sha256"]


def _run_checking_steps(ring, polys, gold, max_checked=None):
    """The F4 loop on the GPU, every step's (r, N, M, rounds), plan digest and
    RREF digest against the reference's (up to max_checked steps)."""
    st = GroebnerState(ring)
    for f in polys:
        update_pairs(st, poly_monic(f))
    k = 0
    steps = gold["steps"]
    while st.n_pairs():
        plan, ech, _ = f4_step(st)
        if k < len(steps) and (max_checked is None or k < max_checked):
            g = steps[k]
            assert (plan.counters.r, plan.counters.N, plan.counters.M, plan.counters.closure_rounds) == \
                (g["r"], g["N"], g["M"], g["closure_rounds"]), f"step {k}"
            assert ech.rank == g["rank"], f"rank step {k}"
            assert plan_digest(plan) == g["plan_sha256"], f"plan step {k}"
            assert _rref_digest(ech) == g["rref_sha256"], f"rref step {k}"
        k += 1
    return st, k


@pytest.mark.parametrize("name,gen,args", [("cyclic8_p32003", gen_cyclic, (8, 32003)),
                                           ("katsura9_p32003", gen_katsura, (9, 32003)),
                                           ("cyclic7_p65521", gen_cyclic, (7, 65521))])
def test_full_run_final_basis_matches_reference(cuda, name, gen, args):
    """Whole north-star runs on the GPU: EVERY F4 step's plan and RREF digests
    (all 38 for cyclic-8) and the final reduced basis (device
    interreduction) against the reference's digests (reference: 3,258 s +
    66 s for cyclic-8 on one CPU core)."""
    from paper_2601_06765_b200.groebner import reduce_basis_device

    ring, polys = gen(*args)
    ref = load_golden(name)
    st, k = _run_checking_steps(ring, polys, ref)
    assert k == len(ref["steps"])
    gb = reduce_basis_device(st.basis, ring)
    assert len(gb) == ref["gb_size"]
    assert hashlib.sha256(format_system(ring, gb).encode()).hexdigest() == ref["final_sha256"]


def _in_ideal_device(gb, gens, ring):
    """Ideal membership of every generator on the device: one Macaulay matrix
    through compile_batch -> psge_reduce.  Rows: for each generator f a
    reducer t*g with LM(t*g) = LM(f) (g = first basis element whose LM divides
    LM(f)), then f itself; the closure (restricted to the basis) adds a
    reducer for every other monomial divisible by a leading monomial.  The
    reducer rows have distinct leads, so they are independent, and f reduces
    to zero by the Gröbner basis iff its row is in their span: the number of
    zero rows of the echelon form must equal the number of generators."""
    from paper_2601_06765_b200.monomials import mon_divides

    soa = soa_pack(list(gb) + list(gens), ring)
    lms = [g.lm() for g in gb]
    red = {}
    for f in gens:
        m = f.lm()
        k = next(i for i, lm in enumerate(lms) if mon_divides(lm, m))
        red[m] = Row(tuple(a - b for a, b in zip(m, lms[k])), k, RowRole.REDUCER, 0)
    rows = list(red.values()) + [Row((0,) * ring.n_vars, len(gb) + j, RowRole.SPOLY_HALF, 1)
                                 for j in range(len(gens))]
    plan = compile_batch(rows, soa, Closure.ONE_STEP_REDUCTION, candidates=list(range(len(gb))))
    ech = psge_reduce(csr_from_plan(plan, ring.modulus))
    return ech.zero_row_count, len(gens), plan


@pytest.mark.slow
def test_katsura11_full_run_pinned(cuda):
    """Katsura-11 / F_32003 (north-star system the reference cannot finish):
    steps 0-4 of the live GPU run against the reference's per-step digests,
    2^11 standard monomials, and every generator reduces to zero by the final
    basis on the device (ideal membership, one Macaulay matrix); a perturbed
    generator does not."""
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    from full_run import standard_monomials
    from paper_2601_06765_b200.groebner import reduce_basis_device
    from paper_2601_06765_b200.polynomials import Poly

    ring, polys = gen_katsura(11, 32003)
    gold = load_golden("katsura11_p32003")
    assert len(gold["steps"]) >= 5
    st, _ = _run_checking_steps(ring, polys, gold, max_checked=5)
    gb = reduce_basis_device(st.basis, ring)
    assert standard_monomials([f.lm() for f in gb], ring.n_vars) == 2 ** 11
    zero, n, _ = _in_ideal_device(gb, polys, ring)
    assert zero == n
    # shift the constant term of a generator that has one: f + 1 is in the
    # ideal iff 1 is, and Katsura-11 has solutions
    bad = list(polys)
    j = next(i for i, f in enumerate(bad) if sum(f.terms[-1][0]) == 0)
    t = bad[j].terms
    c = (t[-1][1] + 1) % 32003
    bad[j] = Poly(ring, t[:-1] + (((t[-1][0], c),) if c else ()))
    zero, n, _ = _in_ideal_device(gb, bad, ring)
    assert zero == n - 1


@pytest.mark.parametrize("n", [8, 10])
def test_katsura_full_run_staircase(cuda, n):
    """Katsura-n is zero-dimensional with 2^n solutions, so its reduced grevlex
    basis leaves exactly 2^n standard monomials.  Katsura-11 is a north-star
    system the reference cannot finish (its step 4 alone takes 1,556 s on one
    core); its steps 3-4 are pinned by test_large_step_replay, the
    whole run by this count.  Katsura-8 also matches the reference digest."""
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    from full_run import standard_monomials

    ring, polys = gen_katsura(n, 32003)
    gb = f4_groebner(polys, ring)
    assert standard_monomials([f.lm() for f in gb], ring.n_vars) == 2 ** n
    if n == 8:
        assert hashlib.sha256(format_system(ring, gb).encode()).hexdigest() == load_golden("katsura8_p32003")["final_sha256"]


def test_berlekamp_massey_device_matches_reference(cuda):
    """k_bm (csrc/bm.cu) against the real reference's Berlekamp–Massey outputs
    (tests/golden/bm_golden.json.gz), one sequence at a time through the
    public berlekamp_massey and batched per prime through Engine.bm; plus long
    Krylov-length sequences against the oracle restatement."""
    import gzip
    import json

    from paper_2601_06765_b200.sparselin import _engine_for, berlekamp_massey

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "bm_golden.json.gz")
    with gzip.open(path, "rt") as fh:
        cases = json.load(fh)["cases"]
    for c in cases:
        assert berlekamp_massey(c["seq"], FieldModulus(c["p"])) == c["poly"]
    by_len = {}
    for c in cases:
        by_len.setdefault((c["p"], len(c["seq"])), []).append(c)
    for (p, n), group in by_len.items():
        seqs = np.array([c["seq"] for c in group], dtype=np.uint64).T
        assert _engine_for(FieldModulus(p)).bm(seqs) == [c["poly"] for c in group]
    rng = np.random.default_rng(5)
    for p in (31, 32003):
        long = rng.integers(0, p, (3000, 2), dtype=np.uint64)
        got = _engine_for(FieldModulus(p)).bm(long)
        for j in range(2):
            assert got[j] == oracle.berlekamp_massey(long[:, j].tolist(), p)


@pytest.mark.parametrize("shape", [(37, 37), (53, 29)])
def test_resident_operator_matches_numpy(cuda, shape):
    """f4b_op_*: Krylov projections, Horner evaluation and the power loop of
    wiedemann_solve (reference sparselin.py:408-434) against the NumPy loop."""
    from paper_2601_06765_b200.sparselin import _engine_for, csr_transpose, spmm

    p = 65521
    m = FieldModulus(p)
    rng = np.random.default_rng(3)
    r, c = shape
    dense = rng.integers(0, p, (r, c), dtype=np.uint64) * (rng.random((r, c)) < 0.2)
    A = csr_from_dense(dense, m)
    normal = r != c
    op = _engine_for(m).operator(A.n_rows, A.n_cols, A.row_ptr, A.col_ind, A.val, normal)
    P = np.uint64(p)
    At = csr_transpose(A) if normal else None
    apply_b = (lambda X: spmm(At, spmm(A, X))) if normal else (lambda X: spmm(A, X))
    b = 3
    V = rng.integers(0, p, (c, b), dtype=np.uint64)
    U = rng.integers(0, p, (c, b), dtype=np.uint64)
    steps = 12
    ref = np.empty((steps, b), dtype=np.uint64)
    W = V.copy()
    for k in range(steps):
        ref[k] = ((U * W) % P).sum(axis=0, dtype=np.uint64) % P
        W = apply_b(W)
    assert np.array_equal(op.krylov(U, V, steps), ref)
    g = rng.integers(0, p, 6, dtype=np.uint64)
    v = V[:, :1]
    acc = g[-1] * v % P
    for cc in g[:-1][::-1].tolist():
        acc = (apply_b(acc) + np.uint64(cc) * v) % P
    assert np.array_equal(op.horner(g, V[:, 0]), acc[:, 0])
    assert np.array_equal(op.apply(V), apply_b(V))
    # the power loop (stop before the first zero vector) on a nilpotent
    # operator and on this one (which runs all max_steps)
    N = np.triu(rng.integers(0, p, (c, c), dtype=np.uint64) * (rng.random((c, c)) < 0.3), 1)
    Nc = csr_from_dense(N, m)
    nop = _engine_for(m).operator(c, c, Nc.row_ptr, Nc.col_ind, Nc.val, False)
    for o, app, steps_max in ((nop, lambda x: spmm(Nc, x), 3 * c), (op, apply_b, 7)):
        x = V[:, 0].copy()
        kept = 0
        for _ in range(steps_max):
            y = app(x.reshape(-1, 1))[:, 0]
            if not y.any():
                break
            x, kept = y, kept + 1
        got, taken = o.power_until_zero(V[:, 0], steps_max)
        assert taken == kept and np.array_equal(got, x)


def test_verify_kernel_syzygy_device(cuda):
    """§8f.3: the left-kernel recombination check on the device plan agrees
    with the reference's polynomial recombination (host path)."""
    from paper_2601_06765_b200.groebner import verify_kernel_syzygy
    from paper_2601_06765_b200.sparselin import KernelBasis
    from paper_2601_06765_b200.symbolic import LayoutPlan

    ring, polys = gen_cyclic(5, 32003)
    st = GroebnerState(ring)
    for f in polys:
        update_pairs(st, poly_monic(f))
    for _ in range(4):
        f4_step(st)
    spec, _ = select_batch(st)
    soa = st.soa()
    plan = compile_batch(select_rows(spec, soa), soa, Closure.ONE_STEP_REDUCTION)
    kb = left_kernel(csr_from_plan(plan, ring.modulus), count=3, seed=0)
    assert kb.vectors, "expected dependent rows in this batch"
    host = LayoutPlan(ring, plan.row_ptr, plan.col_ind, plan.val, plan.dict_keys, plan.row_meta, plan.counters)
    assert verify_kernel_syzygy(plan, st.basis, kb).ok and verify_kernel_syzygy(host, st.basis, kb).ok
    bad = [np.array(v, dtype=np.uint64).copy() for v in kb.vectors]
    bad[0][int(np.flatnonzero(bad[0])[0])] += 1
    kbad = KernelBasis(kb.side, bad, len(bad), kb.seed_trail)
    assert not verify_kernel_syzygy(plan, st.basis, kbad).ok
    assert not verify_kernel_syzygy(host, st.basis, kbad).ok


def test_mq16_wiedemann_kernel_matches_reference(cuda):
    """BASELINE config 4 (MQ n=16, m=32 over F_31, Block Wiedemann): the first
    two F4 steps with F4Config(numeric="wiedemann") return the same left
    kernel as the real reference — step 0 via the dense path (62 x 153),
    step 1 via Wiedemann on Aᵀ (584 x 968, 12 seeded rounds, nullity 41):
    identical vectors (sha256), dimension and seed trail
    (tests/golden/make_golden_wiedemann.py; reference left_kernel,
    sparselin.py:551-569, 136 s for step 1 on one core)."""
    import json

    from paper_2601_06765_b200.groebner import F4Config
    from paper_2601_06765_b200.systems import gen_random_quadratic

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "mq16x32_p31_wiedemann.json")
    with open(path) as fh:
        gold = json.load(fh)
    ring, polys = gen_random_quadratic(16, 32, 1.0, 0, 31)
    st = GroebnerState(ring)
    for f in polys:
        update_pairs(st, poly_monic(f))
    cfg = F4Config(numeric="wiedemann", block_width=4, seed=0)
    for g in gold["steps"]:
        plan, ech, kb = f4_step(st, cfg)
        assert plan_digest(plan) == g["plan_sha256"] and _rref_digest(ech) == g["rref_sha256"]
        assert kb.side == g["kernel_side"] and kb.dimension_found == g["dimension_found"]
        assert [list(t) for t in kb.seed_trail] == g["seed_trail"]
        assert [int(x) for x in kb.vectors[0]] == g["first_vector"]
        h = hashlib.sha256()
        for v in kb.vectors:
            h.update(("v:" + ",".join(str(int(x)) for x in v) + ";").encode())
        assert h.hexdigest() == g["kernel_sha256"]


@pytest.mark.parametrize("shape,density", [((40, 30), 0.2), ((300, 1200), 0.02), ((1, 5), 1.0), ((7, 3), 0.0)])
def test_csr_transpose_device(cuda, shape, density):
    """f4b_csr_transpose (reference sparselin.py:108-121: stable counting-sort
    transpose) against NumPy's stable argsort."""
    from paper_2601_06765_b200.sparselin import csr_transpose

    p = 32003
    rng = np.random.default_rng(shape[0] * 7 + shape[1])
    mat = _random_sparse(rng, shape[0], shape[1], density, p)
    A = csr_from_dense(mat, FieldModulus(p))
    T = csr_transpose(A)
    want = csr_from_dense(np.ascontiguousarray(mat.T), FieldModulus(p))
    assert (T.n_rows, T.n_cols) == (shape[1], shape[0])
    assert np.array_equal(T.row_ptr, want.row_ptr) and np.array_equal(T.col_ind, want.col_ind)
    assert np.array_equal(T.val, want.val)


def test_plan_text_streamed_from_device(cuda):
    """plan_to_text of a device plan streams its number lists from the device
    (f4b_plan_text); the text equals the host formatting of the downloaded
    arrays and the reference digest (cyclic-8 step 19, M = 2.68 M)."""
    from paper_2601_06765_b200.symbolic import LayoutPlan

    snaps = load_snapshots("cyclic8_p32003")
    gold = load_golden("cyclic8_p32003")
    ring, st = state_from_snapshot(snaps[19])
    spec, _ = select_batch(st)
    soa = st.soa()
    plan = compile_batch(select_rows(spec, soa), soa, Closure.ONE_STEP_REDUCTION)
    dev_text = plan_to_text(plan)
    host = LayoutPlan(ring, plan.row_ptr, plan.col_ind, plan.val, plan.dict_keys, plan.row_meta, plan.counters)
    assert dev_text == plan_to_text(host)
    assert hashlib.sha256(dev_text.encode()).hexdigest() == gold["steps"][19]["plan_sha256"]


@pytest.mark.parametrize("which,fault", [
    ("none", None),
    ("col_desc", "columns not strictly ascending"),
    ("col_range", "column out of range"),
    ("val_zero", "zero value stored in plan"),
    ("row_empty", "(basis members are nonzero)"),
    ("row_tile", "row_ptr does not tile the value stream"),
])
def test_device_validate_matches_host(cuda, which, fault):
    """compile_batch validates device plans on the device (f4b_plan_validate,
    reference symbolic.py:125-163 / :383-387); an injected fault raises the
    same PropertyViolationError message the host check gives on the same
    (downloaded, equally corrupted) arrays."""
    from paper_2601_06765_b200.symbolic import LayoutPlan

    snaps = load_snapshots("cyclic8_p32003")
    ring, st = state_from_snapshot(snaps[10])
    spec, _ = select_batch(st)
    soa = st.soa()
    plan = compile_batch(select_rows(spec, soa), soa, Closure.ONE_STEP_REDUCTION)  # validated inside
    rp, ci, va = plan.row_ptr.copy(), plan.col_ind.copy(), plan.val.copy()
    r, N = plan.n_rows, plan.n_cols
    i = r // 3  # a row in the middle, > 1 term
    while rp[i + 1] - rp[i] < 2:
        i += 1
    a = int(rp[i])
    if which == "col_desc":
        plan.device.poke("col_ind", a + 1, int(ci[a]))
        ci[a + 1] = ci[a]
    elif which == "col_range":
        last = int(rp[i + 1]) - 1
        plan.device.poke("col_ind", last, N)
        ci[last] = N
    elif which == "val_zero":
        plan.device.poke("val", a + 1, 0)
        va[a + 1] = 0
    elif which == "row_empty":
        plan.device.poke("row_ptr", i + 1, a)
        rp[i + 1] = a
    elif which == "row_tile":
        plan.device.poke("row_ptr", r, int(rp[r]) - 1)
        rp[r] -= 1
    host = LayoutPlan(ring, rp, ci, va, plan.dict_keys, plan.row_meta, plan.counters)
    if fault is None:
        plan.validate()
        host.validate()
        return
    with pytest.raises(errors.PropertyViolationError) as dev_err:
        plan.validate()
    with pytest.raises(errors.PropertyViolationError) as host_err:
        host.validate()
    assert fault in str(dev_err.value)
    assert str(host_err.value) in str(dev_err.value)


def test_plan_prefetch_matches_download(cuda):
    """LayoutPlan.prefetch (f4b_plan_prefetch on the copy stream, overlapped
    with the next compile) returns the same host arrays and dictionary keys
    as the synchronous download (cyclic-8 step 10 compiled twice, the second
    compile issued while the first plan's arrays are in flight)."""
    snaps = load_snapshots("cyclic8_p32003")
    gold = load_golden("cyclic8_p32003")
    ring, st = state_from_snapshot(snaps[10])
    spec, _ = select_batch(st)
    soa = st.soa()
    rows = select_rows(spec, soa)
    a = compile_batch(rows, soa, Closure.ONE_STEP_REDUCTION).prefetch()
    b = compile_batch(rows, soa, Closure.ONE_STEP_REDUCTION)  # runs while a's arrays download
    for k in ("row_ptr", "col_ind", "val", "dict_keys"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    assert a.col_ind.dtype == np.int64 and a.val.dtype == np.uint64
    assert plan_digest(a) == gold["steps"][10]["plan_sha256"]
    c = compile_batch(rows, soa, Closure.ONE_STEP_REDUCTION).prefetch().prefetch()  # idempotent
    del c  # freed with the copy pending: the free waits for it


@pytest.mark.parametrize("p", [101, 32003, 2147483629])
def test_echelon_complete_rows_subset(cuda, p):
    """f4b_echelon_complete_rows: the pivot rows led by the chosen columns are
    exactly the FULL_RREF ones (every other pivot row comes back empty)."""
    m = FieldModulus(p)
    rng = np.random.default_rng(p % 1000)
    mat = _random_sparse(rng, 120, 160, 0.08, p)
    full = psge_reduce(csr_from_dense(mat, m))
    want = {lead: (c.tolist(), v.tolist()) for lead, c, v in full.pivot_rows}
    pick = sorted(want)[::3]
    part = psge_reduce(csr_from_dense(mat, m))
    part.device.complete_rows(np.asarray(pick + [10**6], dtype=np.int64))  # out-of-range columns are ignored
    assert part.device.info()["full"] == 2
    leads, rp, cols, vals = part.device.rows(0)
    got = {}
    for k, lead in enumerate(leads.tolist()):
        a, b = int(rp[k]), int(rp[k + 1])
        if b > a:
            got[lead] = (cols[a:b].tolist(), vals[a:b].tolist())
    assert sorted(got) == pick
    for lead in pick:
        assert got[lead] == want[lead]


def test_snapshot_resume_gpu(cuda, tmp_path):
    """A binary state snapshot taken mid-run (snapshot.py) resumes the GPU F4
    loop to the reference's final reduced basis (cyclic-6)."""
    from paper_2601_06765_b200.groebner import reduce_basis_device
    from paper_2601_06765_b200.snapshot import load_state, save_state

    ring, polys = gen_cyclic(6, 32003)
    st = GroebnerState(ring)
    for f in polys:
        update_pairs(st, poly_monic(f))
    for _ in range(6):
        f4_step(st)
    path = str(tmp_path / "c6.f4bsnap")
    save_state(st, path)
    st2 = load_state(path)
    while st2.n_pairs():
        f4_step(st2)
    gb = reduce_basis_device(st2.basis, ring)
    assert hashlib.sha256(format_system(ring, gb).encode()).hexdigest() == load_golden("cyclic6_p32003")["final_sha256"]
