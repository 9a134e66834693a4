"""Host-side logic (CPU suite): C-ABI surface, data model, keys, pair logic,
generators, and a whole F4 run driven by the host glue with the oracle as
the per-step engine (checked against the reference's final-basis digest)."""

import hashlib
import re

import numpy as np
import pytest

import oracle
from conftest import ROOT, load_golden
from paper_2601_06765_b200 import errors
from paper_2601_06765_b200.fp import FieldModulus
from paper_2601_06765_b200.groebner import (GroebnerState, Pair, _minimal_mask, reduce_basis, select_batch,
                                            update_pairs)
from paper_2601_06765_b200.monomials import (DeviceKeyFormat, Ring, key_pack_vec, key_unpack_vec, mon_compare,
                                             mon_key_pack)
from paper_2601_06765_b200.polynomials import Poly, poly_format, poly_monic, poly_parse
from paper_2601_06765_b200.symbolic import Closure, select_rows
from paper_2601_06765_b200.systems import format_system, gen_cyclic, gen_katsura, gen_random_quadratic, parse_system

M7 = FieldModulus(7)
R2 = Ring(["x", "y"], "grevlex", M7)


# ---------------------------------------------------------------------------
# C ABI
# ---------------------------------------------------------------------------
def test_library_exports_every_header_symbol(built_lib):
    header = open(f"{ROOT}/include/f4b200.h").read()
    names = set(re.findall(r"\b(f4b_[a-z_0-9]+)\s*\(", header)) - {"f4b_alloc_fn", "f4b_free_fn"}
    assert len(names) >= 20
    for name in sorted(names):
        assert hasattr(built_lib, name), name
    assert built_lib.f4b_abi_version() == 2


def test_status_codes_map_to_reference_exceptions():
    for code, exc in [(1, errors.MissingKeyError), (2, errors.SizeCapError), (3, errors.LaneOverflowError),
                      (4, errors.PropertyViolationError), (5, errors.PreconditionError), (6, errors.DeviceError)]:
        with pytest.raises(exc):
            errors.raise_for_code(code, "x")


def test_engine_refuses_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2601_06765_b200.symbolic import compile_batch
    from paper_2601_06765_b200.polynomials import soa_pack
    from paper_2601_06765_b200.symbolic import Row, RowRole

    soa = soa_pack([poly_parse("x - 1", R2)], R2)
    with pytest.raises(errors.DeviceError):
        compile_batch([Row((1, 0), 0, RowRole.SPOLY_HALF, 0)], soa)


# ---------------------------------------------------------------------------
# data model
# ---------------------------------------------------------------------------
def test_parse_and_format_examples():
    assert poly_parse("x^2*y + 3*x - 1", R2).terms == (((2, 1), 1), ((1, 0), 3), ((0, 0), 6))
    assert poly_parse("0", R2).is_zero() and poly_parse("7", R2).is_zero()
    assert poly_parse("-3", R2).terms == (((0, 0), 4),)
    assert poly_format(poly_parse("x*y - 1", R2)) == "x*y + 6"
    with pytest.raises(errors.PolyParseError):
        poly_parse("x + z", R2)
    with pytest.raises(errors.PolyParseError):
        poly_parse("x^70000", R2)


def test_generators_match_reference_texts():
    assert [poly_format(f) for f in gen_cyclic(2, 7)[1]] == ["x0 + x1", "x0*x1 + 6"]
    assert [poly_format(f) for f in gen_cyclic(3, 7)[1]] == ["x0 + x1 + x2", "x0*x1 + x0*x2 + x1*x2",
                                                            "x0*x1*x2 + 6"]
    assert [poly_format(f) for f in gen_katsura(1, 101)[1]] == ["x0 + 2*x1 + 100", "x0^2 + 2*x1^2 + 100*x0"]
    ring, polys = gen_random_quadratic(3, 2, 0.5, 7, 101)
    r2, p2 = parse_system(format_system(ring, polys))
    assert [f.terms for f in p2] == [f.terms for f in polys]


@pytest.mark.parametrize("order", ["grevlex", "deglex", "lex"])
@pytest.mark.parametrize("n", [1, 3, 8, 12])
def test_reference_keys_refine_the_order(order, n):
    ring = Ring([f"v{i}" for i in range(n)], order, M7)
    rng = np.random.default_rng(n)
    a = rng.integers(0, 6, (400, n))
    b = rng.integers(0, 6, (400, n))
    ka, kb = key_pack_vec(a, ring), key_pack_vec(b, ring)
    assert np.array_equal(key_unpack_vec(ka, ring), a)
    for i in range(400):
        want = mon_compare(tuple(a[i]), tuple(b[i]), ring)
        ta, tb = tuple(int(w) for w in ka[i]), tuple(int(w) for w in kb[i])
        assert (ta > tb) - (ta < tb) == want
        assert ta == mon_key_pack(tuple(int(x) for x in a[i]), ring)


@pytest.mark.parametrize("order", ["grevlex", "deglex", "lex"])
@pytest.mark.parametrize("n,D", [(5, 7), (8, 15), (12, 7), (16, 4), (9, 31)])
def test_device_key_order_isomorphic_and_shift_additive(order, n, D):
    ring = Ring([f"v{i}" for i in range(n)], order, M7)
    fmt = DeviceKeyFormat(ring, D)
    rng = np.random.default_rng(D * 100 + n)
    mons = [tuple(int(x) for x in rng.multinomial(int(rng.integers(0, D + 1)), [1.0 / n] * n))
            for _ in range(300)]
    dk = [fmt.pack_int(m) for m in mons]
    rk = [mon_key_pack(m, ring) for m in mons]
    for i in range(0, 300, 3):
        for j in range(1, 300, 7):
            assert (dk[i] < dk[j]) == (rk[i] < rk[j]) and (dk[i] == dk[j]) == (mons[i] == mons[j])
    one = fmt.pack_int((0,) * n)
    for i in range(0, 300, 5):
        t, m = mons[i], mons[(i * 7 + 1) % 300]
        tm = tuple(a + b for a, b in zip(t, m))
        if sum(tm) <= D:
            assert fmt.pack_int(tm) == fmt.pack_int(m) + fmt.pack_int(t) - one


# ---------------------------------------------------------------------------
# pair logic
# ---------------------------------------------------------------------------
def test_update_pairs_product_and_chain_criteria():
    st = GroebnerState(R2)
    update_pairs(st, poly_parse("x + 6", R2))
    update_pairs(st, poly_parse("y + 6", R2))
    assert st.pairs == []
    r3 = Ring(["x", "y", "z"], "grevlex", M7)
    st = GroebnerState(r3)
    update_pairs(st, poly_parse("x^2*z + y", r3))
    update_pairs(st, poly_parse("y^2*z + x", r3))
    assert [(q.i, q.j) for q in st.pairs] == [(0, 1)]
    update_pairs(st, poly_parse("x*y*z + 1", r3))
    assert [(q.i, q.j) for q in st.pairs] == [(1, 2), (0, 2)]
    with pytest.raises(errors.PreconditionError):
        update_pairs(st, poly_parse("2*x + 1", r3))


def test_minimal_mask():
    u = np.array([[1, 0], [2, 0], [0, 1], [1, 1], [0, 3]])
    assert _minimal_mask(u).tolist() == [True, False, True, False, False]


def test_select_batch_groups_minimal_degree():
    st = GroebnerState(R2)
    st.basis = [poly_parse("x^2", R2)] * 4
    k = R2.sort_key
    st.pairs = sorted([Pair(0, 1, (2, 1), 3, k((2, 1))), Pair(1, 2, (1, 2), 3, k((1, 2))),
                       Pair(2, 3, (4, 1), 5, k((4, 1)))], key=Pair.sort_tuple)
    spec, d = select_batch(st)
    assert d == 3 and len(spec.targets) == 2 and len(st.pairs) == 1
    with pytest.raises(errors.PreconditionError):
        select_batch(st)
        select_batch(st)


# ---------------------------------------------------------------------------
# whole F4 run: host glue + oracle per step == reference final basis
# ---------------------------------------------------------------------------
def _f4_with_oracle(ring, polys):
    st = GroebnerState(ring)
    for f in polys:
        update_pairs(st, poly_monic(f))
    while st.n_pairs():
        spec, _ = select_batch(st)
        soa = st.soa()
        rows = select_rows(spec, soa)
        plan = oracle.compile_batch_arrays([(r.shift, r.basis_index, r.role.value, r.provenance) for r in rows],
                                           (soa.exps, soa.coeff, soa.offset, soa.length), ring.order)
        e = oracle.psge_arrays(len(plan["row_ptr"]) - 1, plan["counters"]["N"], plan["row_ptr"],
                               plan["col_ind"], plan["val"], ring.modulus.p)
        dexp = oracle.fbsp.ref_unkeys(plan["dict_keys"], ring.n_vars, ring.order)
        new = [Poly(ring, tuple((tuple(int(x) for x in dexp[c]), int(v)) for c, v in zip(cols, vals)))
               for _, cols, vals in e["nonpivot_rows"]]
        for f in sorted(new, key=lambda f: ring.sort_key(f.lm())):
            update_pairs(st, f)
    return reduce_basis(st.basis, ring)


@pytest.mark.parametrize("name,gen,args", [("cyclic5_p32003", gen_cyclic, (5, 32003)),
                                           ("katsura5_p32003", gen_katsura, (5, 32003))])
def test_host_f4_loop_with_oracle_matches_reference(name, gen, args):
    ring, polys = gen(*args)
    gb = _f4_with_oracle(ring, polys)
    assert hashlib.sha256(format_system(ring, gb).encode()).hexdigest() == load_golden(name)["final_sha256"]


def test_compat_shim_rebinds_reference_names():
    """compat.install rebinds fpgb.groebner's hot-path names (uses a stand-in
    module object: the reference itself is not needed)."""
    import types

    from paper_2601_06765_b200 import compat, sparselin, symbolic

    from paper_2601_06765_b200 import bench

    g = types.SimpleNamespace(compile_batch=1, csr_from_plan=2, psge_reduce=3, left_kernel=6)
    b, cli = types.SimpleNamespace(microbench=4), types.SimpleNamespace(microbench=5)
    fake = types.SimpleNamespace(groebner=g, bench=b, cli=cli)
    compat.install(fake)
    assert g.compile_batch is symbolic.compile_batch and g.psge_reduce is sparselin.psge_reduce
    assert g.csr_from_plan is sparselin.csr_from_plan and g.left_kernel is sparselin.left_kernel
    assert b.microbench is bench.microbench and cli.microbench is bench.microbench
    compat.uninstall(fake)
    assert (g.compile_batch, g.csr_from_plan, g.psge_reduce, g.left_kernel) == (1, 2, 3, 6)
    assert (b.microbench, cli.microbench) == (4, 5)


def test_microbench_host_logic_and_no_cpu_fallback():
    """The microbench inputs follow the reference generator (bench.py:237-241:
    pool of round(size*(1-dup)) 48-bit keys, uniform picks) and the host check
    equals np.unique; without a GPU the device primitives raise (no fallback)."""
    import numpy as np

    from paper_2601_06765_b200 import bench as mb
    from paper_2601_06765_b200.errors import DeviceError

    k = mb._synth_keys(np.random.default_rng(5), 10_000, 0.9)
    assert k.shape == (10_000, 2) and k.dtype == np.uint64 and int(k.max()) < 1 << 48
    assert len(np.unique(k, axis=0)) <= 1000
    assert np.array_equal(mb._host_unique(k), np.unique(k, axis=0))
    assert len(mb._synth_keys(np.random.default_rng(1), 5000, 1.0)) == 5000
    import torch

    if not torch.cuda.is_available():
        with pytest.raises(DeviceError):
            mb.microbench("mod_fma", 16)


def test_row_pack_matches_python_conversion():
    """csrc/hostglue.cpp pack_rows (compile_batch's Row list -> int32 basis
    index + u16 shift lanes) against the plain Python conversion, and its
    error paths."""
    from paper_2601_06765_b200 import _build
    from paper_2601_06765_b200.hostglue import native as _rowpack
    from paper_2601_06765_b200.symbolic import Row, RowRole

    _build.build_hostglue()
    rng = np.random.default_rng(3)
    n = 6
    rows = [Row(tuple(int(x) for x in rng.integers(0, 0xFFFF, n)), int(rng.integers(0, 900)), RowRole.REDUCER, i)
            for i in range(257)]
    rows.append(Row(tuple(np.int64(x) for x in range(n)), np.int32(7), RowRole.SPOLY_HALF, 0))  # numpy scalars
    rb = np.empty(len(rows), np.int32)
    sh = np.empty((len(rows), n), np.uint16)
    bmin, bmax, ok = _rowpack().pack_rows(rows, n, rb, sh)
    assert ok and (bmin, bmax) == (min(r.basis_index for r in rows), max(r.basis_index for r in rows))
    assert (rb == [r.basis_index for r in rows]).all()
    assert (sh == np.array([r.shift for r in rows], dtype=np.int64)).all()
    # lane overflow / negative exponent / negative index are reported, not wrapped silently
    bad = [Row((0,) * (n - 1) + (0x10000,), 1, RowRole.REDUCER, 0), Row((0,) * n, -3, RowRole.REDUCER, 0)]
    assert _rowpack().pack_rows(bad, n, np.empty(2, np.int32), np.empty((2, n), np.uint16)) == (-3, 1, False)
    assert _rowpack().pack_rows([Row((0, -1) + (0,) * (n - 2), 0, RowRole.REDUCER, 0)], n, np.empty(1, np.int32),
                                np.empty((1, n), np.uint16))[2] is False
    with pytest.raises(ValueError):  # shift of the wrong length
        _rowpack().pack_rows([Row((1,) * (n - 1), 0, RowRole.REDUCER, 0)], n, np.empty(1, np.int32),
                             np.empty((1, n), np.uint16))
    with pytest.raises(ValueError):  # output too small
        _rowpack().pack_rows(rows, n, np.empty(3, np.int32), sh)


def _gm_numpy(L, lm_t, pi, pj, plcm):
    """NumPy statement of the Gebauer–Möller criteria (reference
    groebner.py:154-201), the checker for csrc/hostglue.cpp."""
    from paper_2601_06765_b200.groebner import _unique_rows

    t = len(L)
    lcm = np.maximum(L, lm_t[None, :])
    if t:
        uq, inv = _unique_rows(lcm)
        kept_idx = np.flatnonzero(_minimal_mask(uq)[inv])
        _, first = np.unique(inv[kept_idx], return_index=True)
        reps = np.sort(kept_idx[first])
        coprime = (np.minimum(L[reps], lm_t[None, :]) == 0).all(axis=1)
        surv = reps[~coprime]
    else:
        surv = np.zeros(0, dtype=np.int64)
    if len(plcm):
        hit = (plcm >= lm_t[None, :]).all(axis=1)
        hit &= (np.maximum(L[pi], lm_t) != plcm).any(axis=1)
        hit &= (np.maximum(L[pj], lm_t) != plcm).any(axis=1)
    else:
        hit = np.zeros(0, dtype=bool)
    return surv, ~hit


@pytest.mark.parametrize("seed", range(6))
def test_gm_criteria_native_matches_numpy(seed):
    """gm_new_pairs / gm_prune against the NumPy statement on random leading
    monomials (small exponents: many equal lcms, divisibility chains and
    coprime pairs), including the queued pairs a run accumulates."""
    from paper_2601_06765_b200 import _build
    from paper_2601_06765_b200.hostglue import native

    _build.build_hostglue()
    hg = native()
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 7))
    L = np.zeros((0, n), np.int64)
    pi = np.zeros(0, np.int64)
    pj = np.zeros(0, np.int64)
    plcm = np.zeros((0, n), np.int64)
    for t in range(120):
        lm_t = np.ascontiguousarray(rng.integers(0, 4, n) * (rng.random(n) < 0.6), dtype=np.int64)
        want_s, want_k = _gm_numpy(L, lm_t, pi, pj, plcm)
        surv = np.empty(t, np.int64)
        surv = surv[:hg.gm_new_pairs(np.ascontiguousarray(L), t, n, lm_t, surv)]
        keep = np.ones(len(pi), np.uint8)
        if len(pi):
            assert hg.gm_prune(plcm, pi, pj, len(pi), np.ascontiguousarray(L), n, lm_t, keep) == int(want_k.sum())
        assert surv.tolist() == want_s.tolist()
        assert keep.view(bool).tolist() == want_k.tolist()
        keep = keep.view(bool)
        pi = np.concatenate([pi[keep], surv])
        pj = np.concatenate([pj[keep], np.full(len(surv), t, np.int64)])
        plcm = np.ascontiguousarray(np.concatenate([plcm[keep], np.maximum(L[surv], lm_t)]))
        L = np.ascontiguousarray(np.concatenate([L, lm_t[None, :]]))
        if rng.random() < 0.2 and len(pi):  # a select_batch pops a prefix
            k = int(rng.integers(1, len(pi) + 1))
            pi, pj, plcm = pi[k:], pj[k:], np.ascontiguousarray(plcm[k:])
    with pytest.raises(IndexError):
        hg.gm_prune(np.zeros((1, n), np.int64), np.array([5], np.int64), np.array([0], np.int64), 1,
                    np.zeros((2, n), np.int64), n, np.zeros(n, np.int64), np.ones(1, np.uint8))


def test_select_rows_arrays_match_row_loop():
    """select_rows (shifts and keys over arrays) equals the per-row statement
    (reference symbolic.py:166-201), with and without an admissibility filter,
    and raises the same errors."""
    import dataclasses

    from paper_2601_06765_b200.symbolic import _select_rows_loop

    for ring, polys in (gen_cyclic(6, 32003), gen_katsura(5, 32003)):
        st = GroebnerState(ring)
        for f in polys:
            update_pairs(st, poly_monic(f))
        spec, _ = select_batch(st)
        soa = st.soa()
        assert select_rows(spec, soa) == _select_rows_loop(spec, soa, list(spec.targets))
        adm = dataclasses.replace(spec, adm=lambda sh, b, role, prov: (b + prov) % 3 != 0)
        try:
            want = _select_rows_loop(adm, soa, list(adm.targets))
        except errors.UncoverableTargetError:
            with pytest.raises(errors.UncoverableTargetError):
                select_rows(adm, soa)
        else:
            assert select_rows(adm, soa) == want
        t0 = spec.targets[0]
        bad = dataclasses.replace(spec, targets=(dataclasses.replace(t0, lcm=tuple(0 for _ in t0.lcm)),))
        with pytest.raises(errors.DivisionError):
            select_rows(bad, soa)
        bad = dataclasses.replace(spec, targets=(dataclasses.replace(t0, gi=len(soa)),))
        with pytest.raises(errors.UncoverableTargetError):
            select_rows(bad, soa)


@pytest.mark.parametrize("order", ["grevlex", "lex", "deglex"])
@pytest.mark.parametrize("seed", range(3))
def test_gm_update_native_matches_numpy_queue(order, seed):
    """gm_update (criteria + reference keys + merge into the sorted queue)
    against the NumPy update: concatenate, key_pack_vec, lexsort on
    (degree, key(lcm), i, j) — reference Pair.sort_tuple, groebner.py:110-116."""
    from paper_2601_06765_b200 import _build
    from paper_2601_06765_b200.hostglue import native

    _build.build_hostglue()
    hg = native()
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(2, 7))
    ring = Ring([f"x{i}" for i in range(n)], order, FieldModulus(32003))
    W = ring.n_key_words
    L = np.zeros((0, n), np.int64)
    q = {"pi": np.zeros(0, np.int64), "pj": np.zeros(0, np.int64), "plcm": np.zeros((0, n), np.int64),
         "pdeg": np.zeros(0, np.int64), "pkey": np.zeros((0, W), np.uint64)}
    for t in range(100):
        lm_t = np.ascontiguousarray(rng.integers(0, 4, n) * (rng.random(n) < 0.6), dtype=np.int64)
        surv, keep = _gm_numpy(L, lm_t, q["pi"], q["pj"], q["plcm"])
        nl = np.maximum(L[surv], lm_t)
        pi = np.concatenate([q["pi"][keep], surv])
        pj = np.concatenate([q["pj"][keep], np.full(len(surv), t, np.int64)])
        plcm = np.concatenate([q["plcm"][keep], nl])
        pdeg = np.concatenate([q["pdeg"][keep], nl.sum(axis=1)])
        pkey = np.concatenate([q["pkey"][keep], key_pack_vec(nl, ring) if len(nl) else np.zeros((0, W), np.uint64)])
        o = np.lexsort((pj, pi) + tuple(pkey[:, w] for w in reversed(range(W))) + (pdeg,))
        want = {"pi": pi[o], "pj": pj[o], "plcm": plcm[o], "pdeg": pdeg[o], "pkey": pkey[o]}
        P, cap = len(q["pi"]), len(q["pi"]) + t
        out = {"pi": np.empty(cap, np.int64), "pj": np.empty(cap, np.int64), "plcm": np.empty((cap, n), np.int64),
               "pdeg": np.empty(cap, np.int64), "pkey": np.empty((cap, W), np.uint64)}
        c = np.ascontiguousarray
        m = hg.gm_update(c(L), t, n, lm_t, int(ring.graded), int(order == "grevlex"), W, c(q["pi"]), c(q["pj"]),
                         c(q["plcm"]), c(q["pdeg"]), c(q["pkey"]), P, out["pi"], out["pj"], out["plcm"],
                         out["pdeg"], out["pkey"])
        assert m == len(want["pi"])
        for k in want:
            assert np.array_equal(out[k][:m], want[k]), (t, k)
        q = {k: c(v[:m]) for k, v in out.items()}
        L = np.concatenate([L, lm_t[None, :]])
        if rng.random() < 0.2 and m:
            k = int(rng.integers(1, m + 1))
            q = {kk: c(v[k:]) for kk, v in q.items()}


@pytest.mark.parametrize("order", ["grevlex", "deglex", "lex"])
def test_key_pack_native_matches_numpy(order):
    """key_pack_vec on >= 4096 int64 rows (csrc/hostglue.cpp pack_keys) equals
    the NumPy packing of the same rows in smaller blocks; lane overflow is
    LaneOverflowError on both."""
    from paper_2601_06765_b200 import _build

    _build.build_hostglue()
    for n in (2, 8, 11):
        ring = Ring([f"x{i}" for i in range(n)], order, FieldModulus(32003))
        e = np.random.default_rng(n).integers(0, 0x10000, (9000, n)).astype(np.int64)
        big = key_pack_vec(e, ring)
        small = np.concatenate([key_pack_vec(e[i:i + 1000], ring) for i in range(0, len(e), 1000)])
        assert np.array_equal(big, small)
        for i in range(0, len(e), 997):
            assert tuple(int(x) for x in big[i]) == mon_key_pack(tuple(int(x) for x in e[i]), ring)
        e[1234, n - 1] = 0x10000
        with pytest.raises(errors.LaneOverflowError):
            key_pack_vec(e, ring)
