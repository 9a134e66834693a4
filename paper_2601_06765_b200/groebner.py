"""F4 driver over the GPU hot path — drop-in for ``pkg/src/fpgb/groebner.py``.

The host keeps the reference's pair logic bit for bit (Gebauer–Möller update
:154-201, normal strategy :204-213, harvest order :285-290), vectorized over
NumPy arrays of leading exponents; each F4 step calls the device
``compile_batch`` -> ``psge_reduce`` and appends the harvested rows straight
to the HBM-resident basis (no whole-basis re-pack per step).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from .bulk import ExecPolicy
from .errors import LaneOverflowError, NonterminationError, PreconditionError, PropertyViolationError
from .fp import FieldModulus
from .hostglue import native
from .monomials import Ring, key_pack_vec, mon_div, mon_divides, mon_lcm
from .polynomials import ArrayPoly, Poly, SoaPolySet, poly_add_scaled, poly_monic, poly_mul_mon
from .sparselin import (EchelonResult, KernelBasis, KernelMode, csr_from_plan, dense_gauss, left_kernel,
                        psge_reduce)
from .symbolic import BatchSpec, Closure, LayoutPlan, PairTarget, compile_batch, row_lead_cols, select_rows

MAX_STEPS_DEFAULT = 10_000


@dataclass
class Pair:
    i: int
    j: int
    lcm: tuple
    degree: int
    key: tuple

    def sort_tuple(self):
        return (self.degree, self.key, self.i, self.j)


@dataclass
class BatchStats:
    degree: int
    r: int
    N: int
    M: int
    nnz: int
    rank: int
    new_polys: int
    zero_reductions: int
    closure_rounds: int
    timings_ns: dict


class _HostBasis:
    """Growable SoA copy of the basis (exps, coeffs, reference keys)."""

    def __init__(self, ring: Ring):
        self.ring = ring
        n, W = ring.n_vars, ring.n_key_words
        self.T = 0
        self.keyed = 0  # terms [0, keyed) have their reference keys (packed in soa(), once per batch of appends)
        self.exps = np.zeros((1024, n), dtype=np.int64)
        self.coeff = np.zeros(1024, dtype=np.uint64)
        self.keys = np.zeros((1024, W), dtype=np.uint64)
        self.lengths: list = []
        self.lm = np.zeros((64, n), dtype=np.int64)

    def append(self, exps: np.ndarray, coeff: np.ndarray):
        k = len(exps)
        need = self.T + k
        if need > len(self.coeff):
            cap = max(need, 2 * len(self.coeff))
            for name in ("exps", "coeff", "keys"):
                old = getattr(self, name)
                new = np.zeros((cap,) + old.shape[1:], dtype=old.dtype)
                new[:self.T] = old[:self.T]
                setattr(self, name, new)
        self.exps[self.T:need] = exps
        self.coeff[self.T:need] = coeff
        t = len(self.lengths)
        if t >= len(self.lm):
            grown = np.zeros((2 * len(self.lm), self.lm.shape[1]), dtype=np.int64)
            grown[:t] = self.lm[:t]
            self.lm = grown
        self.lm[t] = exps[0] if k else 0
        self.lengths.append(k)
        self.T = need

    def soa(self) -> SoaPolySet:
        if self.keyed < self.T:
            self.keys[self.keyed:self.T] = key_pack_vec(self.exps[self.keyed:self.T], self.ring)
            self.keyed = self.T
        lengths = np.asarray(self.lengths, dtype=np.int64)
        offset = np.zeros(len(lengths) + 1, dtype=np.int64)
        np.cumsum(lengths, out=offset[1:])
        return SoaPolySet(self.ring, self.keys[:self.T], self.coeff[:self.T], offset, lengths, self.exps[:self.T])


class GroebnerState:
    """Basis + pair queue.  ``pairs`` is a list of Pair (reference API) backed
    by NumPy arrays for the vectorized criteria."""

    def __init__(self, ring: Ring, basis=None, pairs=None):
        self.ring = ring
        self.basis: list = []
        self.stats: list = []
        self.zero_reductions = 0
        self._hb = _HostBasis(ring)
        self._soa = None
        self._dev_token = None  # engine token matching len(basis) polys
        self._dev_n = -1
        n, W = ring.n_vars, ring.n_key_words
        self._pi = np.zeros(0, np.int64)
        self._pj = np.zeros(0, np.int64)
        self._plcm = np.zeros((0, n), np.int64)
        self._pdeg = np.zeros(0, np.int64)
        self._pkey = np.zeros((0, W), np.uint64)
        self._pairs_cache = []
        for f in basis or []:
            self._push_basis(f)
        if pairs:
            self.pairs = pairs

    def _push_basis(self, f: Poly, arrays=None):
        self.basis.append(f)
        if arrays is not None:  # (int64 exps [len, n], uint64 coeffs): the caller's arrays of f's terms
            ex, cf = arrays
        elif f.terms:
            ex = np.asarray([e for e, _ in f.terms], dtype=np.int64)
            cf = np.asarray([c for _, c in f.terms], dtype=np.uint64)
        else:
            ex = np.zeros((0, self.ring.n_vars), np.int64)
            cf = np.zeros(0, np.uint64)
        self._hb.append(ex, cf)
        self._soa = None

    # -- pair queue as a list of Pair ------------------------------------------
    @property
    def pairs(self):
        if self._pairs_cache is None:
            self._pairs_cache = [
                Pair(int(i), int(j), tuple(int(x) for x in l), int(d), tuple(int(w) for w in k))
                for i, j, l, d, k in zip(self._pi.tolist(), self._pj.tolist(), self._plcm, self._pdeg.tolist(),
                                         self._pkey)]
        return self._pairs_cache

    @pairs.setter
    def pairs(self, plist):
        plist = list(plist)
        n, W = self.ring.n_vars, self.ring.n_key_words
        self._pi = np.asarray([q.i for q in plist], dtype=np.int64)
        self._pj = np.asarray([q.j for q in plist], dtype=np.int64)
        self._plcm = np.asarray([q.lcm for q in plist], dtype=np.int64).reshape(len(plist), n)
        self._pdeg = np.asarray([q.degree for q in plist], dtype=np.int64)
        self._pkey = np.asarray([q.key for q in plist], dtype=np.uint64).reshape(len(plist), W)
        self._pairs_cache = plist

    def n_pairs(self) -> int:
        return len(self._pi)

    def soa(self) -> SoaPolySet:
        if self._soa is None or len(self._soa) != len(self.basis):
            self._soa = self._hb.soa()
            if self._dev_n == len(self.basis) and self._dev_token is not None:
                self._soa._f4b_token = self._dev_token
        return self._soa


def _make_pair(state: GroebnerState, i: int, j: int) -> Pair:
    lcm = mon_lcm(state.basis[i].lm(), state.basis[j].lm())
    return Pair(i, j, lcm, sum(lcm), state.ring.sort_key(lcm))


def _minimal_mask(u: np.ndarray) -> np.ndarray:
    """True for rows of ``u`` (distinct exponent vectors) not divisible by any
    other row — processed by ascending degree against the minimal set."""
    deg = u.sum(axis=1)
    keep = np.zeros(len(u), dtype=bool)
    mins = np.zeros((0, u.shape[1]), dtype=u.dtype)
    for d in np.unique(deg):
        idx = np.flatnonzero(deg == d)
        blk = u[idx]
        if len(mins):
            dom = (blk[:, None, :] >= mins[None, :, :]).all(axis=2).any(axis=1)
        else:
            dom = np.zeros(len(idx), dtype=bool)
        keep[idx[~dom]] = True
        mins = np.concatenate([mins, blk[~dom]])
    return keep


def _unique_rows(a: np.ndarray):
    """np.unique(a, axis=0, return_inverse=True) for small non-negative
    exponent rows: rows packed into one int64 (most significant = column 0,
    so numeric order = lexicographic row order) when they fit, which replaces
    the structured-dtype sort by a plain integer sort."""
    if len(a):
        mx = int(a.max())
        bits = max(1, mx.bit_length())
        if int(a.min()) >= 0 and bits * a.shape[1] <= 62:
            key = np.zeros(len(a), dtype=np.int64)
            for j in range(a.shape[1]):
                key = (key << bits) | a[:, j]
            _, idx, inv = np.unique(key, return_index=True, return_inverse=True)
            return a[idx], inv.reshape(-1)
    uq, inv = np.unique(a, axis=0, return_inverse=True)
    return uq, inv.reshape(-1)


def update_pairs(state: GroebnerState, new_poly: Poly, *, _arrays=None) -> GroebnerState:
    """Append a monic polynomial with Gebauer–Möller pruning (reference :154-201).

    ``_arrays`` (internal, f4_step): the polynomial's terms as (int64 exps,
    uint64 coeffs) arrays, so the host basis copy skips re-reading the tuples."""
    if new_poly.is_zero() or new_poly.lc() != 1:
        raise PreconditionError("basis members must be monic and nonzero")
    t = len(state.basis)
    state._push_basis(new_poly, _arrays)
    lm_t = np.ascontiguousarray(new_poly.lm(), dtype=np.int64)
    L = np.ascontiguousarray(state._hb.lm[:t])
    ring = state.ring
    n, W = ring.n_vars, ring.n_key_words
    # chain criterion among the new pairs (i, t) (one representative per
    # minimal lcm, the lowest partner) + product criterion, chain criterion
    # on the queued pairs, and the merge into the sorted queue: one call
    # into csrc/hostglue.cpp (gm_update)
    P = len(state._pi)
    cap = P + t
    o_pi, o_pj, o_pdeg = np.empty(cap, np.int64), np.empty(cap, np.int64), np.empty(cap, np.int64)
    o_plcm, o_pkey = np.empty((cap, n), np.int64), np.empty((cap, W), np.uint64)
    c = np.ascontiguousarray
    m = native().gm_update(L, t, n, lm_t, int(ring.graded), int(ring.order == "grevlex"), W, c(state._pi),
                           c(state._pj), c(state._plcm), c(state._pdeg), c(state._pkey), P, o_pi, o_pj, o_plcm,
                           o_pdeg, o_pkey)
    if m < 0:
        raise LaneOverflowError("pair lcm does not fit the 16-bit lanes of the reference key")
    state._pi, state._pj, state._plcm, state._pdeg, state._pkey = o_pi[:m], o_pj[:m], o_plcm[:m], o_pdeg[:m], o_pkey[:m]
    state._pairs_cache = None
    return state


def select_batch(state: GroebnerState):
    """Normal strategy: all queued pairs of minimal lcm degree (reference :204-213)."""
    if state.n_pairs() == 0:
        raise PreconditionError("empty pair queue")
    d = int(state._pdeg[0])
    k = int(np.searchsorted(state._pdeg, d, side="right"))
    targets = [PairTarget(tuple(int(x) for x in state._plcm[q]), q, int(state._pi[q]), int(state._pj[q]))
               for q in range(k)]
    for name in ("_pi", "_pj", "_plcm", "_pdeg", "_pkey"):
        setattr(state, name, getattr(state, name)[k:])
    state._pairs_cache = None
    return BatchSpec(targets=targets, candidates=tuple(range(len(state.basis)))), d


@dataclass
class F4Config:
    numeric: str = "psge"  # psge | dense | wiedemann
    panel_width: int = 256
    block_width: int = 4
    seed: int = 0
    workers: int = 1
    max_steps: int = MAX_STEPS_DEFAULT
    policy: ExecPolicy | None = None

    def exec_policy(self) -> ExecPolicy:
        return self.policy if self.policy is not None else ExecPolicy(self.workers)


def _dense_echelon(plan: LayoutPlan, m: FieldModulus) -> EchelonResult:
    """Dense-oracle stand-in (reference :238-250), small batches only."""
    A = csr_from_plan(plan, m)
    rank, rref, pivots = dense_gauss(A.to_dense(), m)
    orig = set(row_lead_cols(plan).tolist())
    piv, nonpiv = [], []
    for k, col in enumerate(pivots):
        cols = np.flatnonzero(rref[k]).astype(np.int64)
        (piv if col in orig else nonpiv).append((col, cols, rref[k][cols]))
    return EchelonResult(list(pivots), piv, nonpiv, A.n_rows - rank, rank, 0)


def f4_step(state: GroebnerState, config: F4Config | None = None, _capture=None):
    """One batch: select, compile (GPU), eliminate (GPU), harvest.

    Returns (plan, echelon, kernel) like the reference (:253-311)."""
    from .engine import Engine

    config = config or F4Config()
    ring = state.ring
    spec, degree = select_batch(state)
    basis_snapshot = list(state.basis)
    soa = state.soa()
    rows = select_rows(spec, soa)
    plan = compile_batch(rows, soa, Closure.ONE_STEP_REDUCTION, config.exec_policy())
    if _capture is not None:
        _capture(rows, soa, plan)
    t0 = time.perf_counter_ns()
    if config.numeric == "dense":
        ech = _dense_echelon(plan, ring.modulus)
    else:
        ech = psge_reduce(csr_from_plan(plan, ring.modulus), config.panel_width)
    leads, rp, cols, vals = ech.nonpivot_arrays()
    numeric_ns = time.perf_counter_ns() - t0
    kernel = None
    if config.numeric == "wiedemann":
        A = csr_from_plan(plan, ring.modulus)
        kernel = left_kernel(A, count=max(1, A.n_rows), seed=config.seed)
        rep = verify_kernel_syzygy(plan, basis_snapshot, kernel)
        if not rep.ok:
            raise PropertyViolationError(f"kernel syzygy violation: {rep.detail}")
    # harvest: RREF rows are monic with terms descending (columns ascending);
    # key(LM) ascending == lead column descending (reference :285-290)
    exps_all = plan.dict_exps().astype(np.int64)
    new_ex, new_cf, new_len = [], [], []
    for k in range(len(leads) - 1, -1, -1):
        c = cols[rp[k]:rp[k + 1]]
        ex = exps_all[c]
        cf = vals[rp[k]:rp[k + 1]]
        cf64 = cf.astype(np.uint64, copy=False)
        update_pairs(state, ArrayPoly(ring, ex, cf64), _arrays=(ex, cf64))
        new_ex.append(ex)
        new_cf.append(cf)
        new_len.append(len(c))
    # keep the device basis in lockstep: the new rows go from the echelon
    # pool to the device basis on the device (§8f.2, no upload)
    eng = Engine.for_ring(ring)
    if getattr(soa, "_f4b_token", None) == eng.token and new_len:
        dplan, dech = plan.device, getattr(ech, "device", None)
        if dplan is not None and dech is not None and dplan.engine is eng and dech.engine is eng:
            eng.append_from_echelon(dplan, dech, np.asarray(new_len), np.concatenate(new_ex),
                                    np.concatenate(new_cf))
        else:
            eng.append_polys(np.asarray(new_len), np.concatenate(new_ex), np.concatenate(new_cf))
    if getattr(soa, "_f4b_token", None) is not None and soa._f4b_token[0] == eng.uid:
        state._dev_token, state._dev_n = eng.token, len(state.basis)
    state.zero_reductions += ech.zero_row_count
    dt = plan.timings_ns
    state.stats.append(BatchStats(
        degree=degree, r=plan.counters.r, N=plan.counters.N, M=plan.counters.M, nnz=plan.counters.nnz,
        rank=ech.rank, new_polys=len(new_len), zero_reductions=ech.zero_row_count,
        closure_rounds=plan.counters.closure_rounds,
        timings_ns={"dict_build": dt.get("dict_build_ns", 0), "row_assemble": dt.get("row_assemble_ns", 0),
                    "numeric_core": numeric_ns, "fill_generated": ech.fill_generated,
                    **{f"device_{k}": v for k, v in ech.timings().items()}}))
    return plan, ech, kernel


def spoly(f: Poly, g: Poly) -> Poly:
    if f.is_zero() or g.is_zero():
        raise PreconditionError("S-polynomial of a zero polynomial")
    p = f.ring.modulus.p
    L = mon_lcm(f.lm(), g.lm())
    a = poly_mul_mon(mon_div(L, f.lm()), f)
    b = poly_mul_mon(mon_div(L, g.lm()), g)
    ia, ib = pow(f.lc(), p - 2, p), pow(g.lc(), p - 2, p)
    left = Poly(f.ring, tuple((e, c * ia % p) for e, c in a.terms))
    return poly_add_scaled(left, (p - ib) % p, b)


def normal_form(f: Poly, basis: list) -> Poly:
    """Full remainder; reducer = smallest LM first, then lowest index
    (reference :70-105, the closure rule of compile_batch)."""
    live = [g for g in basis if not g.is_zero()]
    if f.is_zero() or not live:
        return f
    ring = f.ring
    p = ring.modulus.p
    table = sorted(range(len(live)), key=lambda i: (ring.sort_key(live[i].lm()), i))
    lms = [(live[i].lm(), i) for i in table]
    work, out = f, []
    while not work.is_zero():
        lead, lc = work.terms[0]
        hit = next((i for lm, i in lms if mon_divides(lm, lead)), None)
        if hit is None:
            out.append((lead, lc))
            work = Poly(ring, work.terms[1:])
            continue
        g = live[hit]
        coef = lc * pow(g.lc(), p - 2, p) % p
        work = poly_add_scaled(work, p - coef, poly_mul_mon(mon_div(lead, g.lm()), g))
    return Poly(ring, tuple(out))


def reduce_basis(polys: list, ring: Ring) -> list:
    """Canonical reduced basis: minimal, tail-reduced, monic, sorted by lead
    descending (reference :314-332).  Host-side; see DESIGN.md §next."""
    work = sorted((poly_monic(f) for f in polys if not f.is_zero()), key=lambda f: ring.sort_key(f.lm()))
    minimal = []
    for f in work:
        if not any(mon_divides(g.lm(), f.lm()) for g in minimal):
            minimal.append(f)
    changed = True
    while changed:
        changed = False
        for i in range(len(minimal)):
            r = normal_form(minimal[i], minimal[:i] + minimal[i + 1:])
            if r.terms != minimal[i].terms:
                minimal[i] = poly_monic(r)
                changed = True
    minimal.sort(key=lambda f: ring.sort_key(f.lm()), reverse=True)
    return minimal


def _minimal_monic(polys: list, ring: Ring) -> list:
    work = sorted((poly_monic(f) for f in polys if not f.is_zero()), key=lambda f: ring.sort_key(f.lm()))
    minimal = []
    for f in work:
        if not any(mon_divides(g.lm(), f.lm()) for g in minimal):
            minimal.append(f)
    return minimal


def _minimal_order(polys: list, ring: Ring) -> np.ndarray:
    """Indices of the minimal basis (reference reduce_basis :314-332: ascending
    sort_key(LM), keep a polynomial unless an earlier kept LM divides its LM)
    with NumPy: divisibility is transitive, so "no earlier LM divides it"
    decides; ties keep the first (stable order)."""
    idx = [i for i, f in enumerate(polys) if not f.is_zero()]
    if not idx:
        return np.zeros(0, np.int64)
    L = np.asarray([polys[i].lm() for i in idx], dtype=np.int64).reshape(len(idx), ring.n_vars)
    keys = key_pack_vec(L, ring)
    order = np.lexsort(keys.T[::-1])  # ascending key = ascending term order, stable
    Ls = L[order]
    kept = np.ones(len(order), dtype=bool)
    for i0 in range(0, len(order), 256):
        blk = Ls[i0:i0 + 256]
        div = (Ls[None, :, :] <= blk[:, None, :]).all(axis=2)  # div[i, j]: LM_j divides LM_(i0+i)
        div &= np.arange(len(order))[None, :] < np.arange(i0, i0 + len(blk))[:, None]
        kept[i0:i0 + len(blk)] = ~div.any(axis=1)
    return np.asarray(idx, dtype=np.int64)[order[kept]]


def reduce_basis_device(polys: list, ring: Ring, soa: SoaPolySet | None = None) -> list:
    """Final interreduction of a Gröbner basis as ONE extra Macaulay matrix on
    the GPU: the minimal basis (same selection as
    reduce_basis, reference :314-332) as shift-0 rows, closed under one-step
    reduction by compile_batch, then the fully reduced echelon form.  With all
    reducers of every non-leading monomial present, the RREF row led by LM(g)
    has no other term divisible by a leading monomial: it is the reduced basis
    element for g — the unique reduced Gröbner basis the reference's
    normal-form loop converges to (for a Gröbner basis input)."""
    from .polynomials import soa_pack
    from .symbolic import Row, RowRole

    sel = _minimal_order(polys, ring)
    if not len(sel):
        return []
    monic = all(polys[i].lc() == 1 for i in sel.tolist())
    minimal = [polys[i] if monic else poly_monic(polys[i]) for i in sel.tolist()]
    if soa is not None and monic and len(soa) == len(polys):
        # the caller's flat streams (e.g. GroebnerState.soa()): gather the
        # minimal polynomials' term ranges instead of re-packing tuples
        off, ln = soa.offset[sel], soa.length[sel]
        new_off = np.zeros(len(sel) + 1, dtype=np.int64)
        np.cumsum(ln, out=new_off[1:])
        tix = np.repeat(off - new_off[:-1], ln) + np.arange(int(new_off[-1]), dtype=np.int64)
        soa = SoaPolySet(ring, soa.mon_key[tix], soa.coeff[tix], new_off, ln.astype(np.int64), soa.exps[tix])
    else:
        soa = soa_pack(minimal, ring)
    zero = (0,) * ring.n_vars
    rows = [Row(zero, k, RowRole.SPOLY_HALF, 0) for k in range(len(minimal))]
    # the reference's normal-form loop has no dictionary cap: neither has this
    # matrix (only the device's 2^30-term plan limit applies)
    plan = compile_batch(rows, soa, Closure.ONE_STEP_REDUCTION, dict_cap=1 << 62)
    ex = plan.dict_exps()
    out = []
    if plan.device is not None:
        # only the rows led by the basis LMs are back-reduced (the closure
        # rows are pivots for them, never output): f4b_echelon_complete_rows
        from .engine import Engine

        eng = Engine.for_ring(ring)
        col_of = {tuple(r): c for c, r in enumerate(ex.tolist())}
        lead_cols = np.unique(np.asarray([col_of[tuple(f.lm())] for f in minimal], dtype=np.int64))
        ech = eng.psge_plan(plan.device, full=False)
        ech.complete_rows(lead_cols)
        leads, prp, cols, vals = ech.rows(0)
        want = set(lead_cols.tolist())
        cl, vl = cols.tolist(), vals.tolist()
        ex_t = [tuple(r) for r in ex.tolist()]  # one tuple per column, shared by every term
        for k, lead in enumerate(leads.tolist()):
            if lead in want:
                a, b = int(prp[k]), int(prp[k + 1])
                out.append(Poly(ring, tuple(zip(map(ex_t.__getitem__, cl[a:b]), vl[a:b]))))
    else:
        ech = psge_reduce(csr_from_plan(plan, ring.modulus))
        rp, ci = plan.row_ptr, plan.col_ind
        lead_cols = {int(ci[rp[k]]) for k in range(len(minimal))}
        for lead, cols, vals in ech.pivot_rows:
            if lead in lead_cols:
                out.append(Poly(ring, tuple((tuple(int(x) for x in ex[c]), int(v)) for c, v in zip(cols.tolist(),
                                                                                              vals.tolist()))))
    out.sort(key=lambda f: ring.sort_key(f.lm()), reverse=True)
    return out


def f4_groebner(system: list, ring: Ring, config: F4Config | None = None) -> list:
    """Reduced Gröbner basis via the GPU F4 driver (reference :335-350)."""
    config = config or F4Config()
    if any(f.is_zero() for f in system):
        raise PreconditionError("zero polynomial in input system")
    state = GroebnerState(ring)
    for f in system:
        update_pairs(state, poly_monic(f))
    steps = 0
    while state.n_pairs():
        if steps >= config.max_steps:
            raise NonterminationError(f"f4 exceeded {config.max_steps} batches")
        f4_step(state, config)
        steps += 1
    return reduce_basis_device(state.basis, ring, state.soa())


@dataclass
class GroebnerReport:
    ok: bool
    detail: str = ""
    witness: tuple | None = None


def is_groebner(G: list, ring: Ring) -> GroebnerReport:
    live = [g for g in G if not g.is_zero()]
    for a in range(len(live)):
        for b in range(a + 1, len(live)):
            if not normal_form(spoly(live[a], live[b]), live).is_zero():
                return GroebnerReport(False, f"S-poly of members {a},{b} does not reduce to zero", (a, b))
    return GroebnerReport(True)


def verify_kernel_syzygy(plan: LayoutPlan, basis: list, kernel: KernelBasis) -> GroebnerReport:
    """Exact recombination sum_i v_i (t_i g_{k_i}) == 0 (reference :409-428).

    For a device plan this is one Aᵀ·V over the resident CSR:
    row i of the plan is exactly t_i g_{k_i} over the dictionary monomials,
    so Aᵀ v = 0 is the recombination itself."""
    ring = plan.ring
    dev = getattr(plan, "device", None)
    if dev is not None and kernel.vectors:
        for n, v in enumerate(kernel.vectors):
            if len(v) != plan.n_rows:
                return GroebnerReport(False, f"kernel vector {n} has wrong length")
        V = np.stack([np.asarray(v, dtype=np.uint64) % np.uint64(ring.modulus.p) for v in kernel.vectors], axis=1)
        Y = dev.left_apply(V)
        for n in range(V.shape[1]):
            if Y[:, n].any():
                return GroebnerReport(False, f"kernel vector {n} recombines to a nonzero polynomial")
        return GroebnerReport(True)
    for n, v in enumerate(kernel.vectors):
        if len(v) != plan.n_rows:
            return GroebnerReport(False, f"kernel vector {n} has wrong length")
        total = Poly(ring)
        for i, row in enumerate(plan.row_meta):
            c = int(v[i])
            if c:
                total = poly_add_scaled(total, c, poly_mul_mon(row.shift, basis[row.basis_index]))
        if not total.is_zero():
            return GroebnerReport(False, f"kernel vector {n} recombines to {total}")
    return GroebnerReport(True)
