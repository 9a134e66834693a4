"""Batch compilation (FBSP symbolic preprocessing) — drop-in for
``pkg/src/fpgb/symbolic.py``.

``compile_batch`` keeps the reference signature (:293-299) and returns a
``LayoutPlan`` byte-identical to the reference's (same ``plan_to_text``),
but the work runs in the CUDA engine (``csrc/fbsp.cu``): the basis stays in
HBM, the plan's CSR arrays stay on the device for ``psge_reduce``, and the
host copies are materialized only when a caller touches them.
"""

from __future__ import annotations

import enum
import hashlib
from dataclasses import dataclass, field

import numpy as np

from .bulk import DEFAULT_POLICY, ExecPolicy
from .errors import LaneOverflowError, PropertyViolationError, UncoverableTargetError
from .hostglue import native
from .monomials import Ring, key_cmp_rows, key_pack_vec, key_unpack_vec, mon_div, mon_key_pack
from .polynomials import Poly, SoaPolySet

DICT_CAP = 10**6  # reference symbolic.py:46


class RowRole(enum.Enum):
    SPOLY_HALF = 0
    REDUCER = 1


class Closure(enum.Enum):
    SUPPORT_ONLY = "support_only"
    ONE_STEP_REDUCTION = "one_step_reduction"


@dataclass(frozen=True)
class Row:
    shift: tuple
    basis_index: int
    role: RowRole
    provenance: int  # pair id for S-halves, discovery round for closure rows


@dataclass(frozen=True)
class PairTarget:
    lcm: tuple
    pair_id: int
    fi: int
    gi: int


@dataclass
class BatchSpec:
    targets: list
    candidates: tuple
    adm: object = None  # callable(shift, basis_index, role, provenance) -> bool


@dataclass
class PlanCounters:
    r: int = 0
    N: int = 0
    M: int = 0
    nnz: int = 0
    closure_rounds: int = 0
    keys_emitted: int = 0
    keys_generated_total: int = 0


_ARRAYS = ("row_ptr", "col_ind", "val", "dict_keys", "row_meta")


class LayoutPlan:
    """Write-once sparse plan of one batch matrix (reference :99-163).

    Columns index ``dict_keys`` in descending term order; column indices
    ascend within each row.  A plan produced by the device keeps its arrays
    in HBM (``self.device``); the host attributes below are downloaded on
    first access.
    """

    def __init__(self, ring: Ring, row_ptr=None, col_ind=None, val=None, dict_keys=None, row_meta=None,
                 counters: PlanCounters | None = None, timings_ns: dict | None = None, *, device=None,
                 input_rows=()):
        self.ring = ring
        self.counters = counters if counters is not None else PlanCounters()
        self.timings_ns = timings_ns if timings_ns is not None else {}
        self.device = device
        self._input_rows = tuple(input_rows)
        self._host = {}
        self._dict_exps = None
        for k, v in zip(_ARRAYS, (row_ptr, col_ind, val, dict_keys, row_meta)):
            if v is not None:
                self._host[k] = v

    # -- lazy host materialization --------------------------------------------
    def _materialize(self, name):
        if name in self._host:
            return self._host[name]
        if self.device is None:
            raise AttributeError(name)
        dev = self.device
        n = self.ring.n_vars
        pf = dev.prefetched() if name in ("row_ptr", "col_ind", "val", "dict_keys") else None
        if pf is not None and (name != "dict_keys" or pf["dict_keys"] is not None):
            for k in ("row_ptr", "col_ind", "val", "dict_keys"):
                if pf[k] is not None:
                    self._host[k] = pf[k]
            return self._host[name]
        if name in ("row_ptr", "col_ind", "val"):
            got = dev.download(arrays=True, dict_exps=False, closure=False)
            for k in ("row_ptr", "col_ind", "val"):
                self._host[k] = got[k]
        elif name == "dict_keys":
            self._host["dict_keys"] = dev.download_ref_keys(self.ring.n_key_words)
        elif name == "row_meta":
            got = dev.download(arrays=False, dict_exps=False, closure=True)
            extra = tuple(
                Row(tuple(int(x) for x in sh), int(b), RowRole.REDUCER, int(rd))
                for sh, b, rd in zip(got["cl_shift"].reshape(-1, n).tolist(), got["cl_basis"].tolist(),
                                     got["cl_round"].tolist()))
            self._host["row_meta"] = self._input_rows + extra
        return self._host[name]

    def prefetch(self) -> "LayoutPlan":
        """Start downloading the host arrays (row_ptr, col_ind, val,
        dict_keys) of a device plan in the background (copy stream); the
        attributes then wait for it instead of downloading.  Lets a caller
        compile the next batch while this one's arrays cross PCIe."""
        if self.device is not None and not self._host and getattr(self.device, "_pf", None) is None:
            self.device.prefetch(self.ring.n_key_words)
        return self

    def dict_exps(self) -> np.ndarray:
        """Exponent rows of the dictionary, descending (column order)."""
        if self._dict_exps is None:
            if self.device is not None:
                self._dict_exps = self.device.download(arrays=False, dict_exps=True, closure=False)["dict_exps"]
            else:
                self._dict_exps = key_unpack_vec(self.dict_keys, self.ring)
        return self._dict_exps

    row_ptr = property(lambda self: self._materialize("row_ptr"))
    col_ind = property(lambda self: self._materialize("col_ind"))
    val = property(lambda self: self._materialize("val"))
    dict_keys = property(lambda self: self._materialize("dict_keys"))
    row_meta = property(lambda self: self._materialize("row_meta"))

    @property
    def n_rows(self) -> int:
        return self.counters.r if self.device is not None else len(self.row_ptr) - 1

    @property
    def n_cols(self) -> int:
        return self.counters.N if self.device is not None else len(self.dict_keys)

    def _check_device_counters(self):
        c, info = self.counters, self.device.info
        if not (c.r == info["r"] and c.N == info["N"] and c.M == info["M"] and c.nnz == c.M
                and c.keys_emitted == c.M and c.keys_generated_total >= c.M):
            raise PropertyViolationError(f"counters inconsistent: {c}")

    def validate(self):
        """Structural invariants (reference :125-163); PropertyViolationError.

        A device plan is checked where it lives (f4b_plan_validate: one
        kernel over rows, terms and dictionary entries); the counters on
        the host.
        """
        c = self.counters
        if self.device is not None:
            self.device.validate()
            self._check_device_counters()
            return
        rp, ci, va, dk = self.row_ptr, self.col_ind, self.val, self.dict_keys
        if not (rp[0] == 0 and rp[-1] == len(ci) == len(va)):
            raise PropertyViolationError("row_ptr does not tile the value stream")
        lens = np.diff(rp)
        if (lens < 0).any():
            raise PropertyViolationError("negative row segment length")
        if len(self.row_meta) != len(rp) - 1:
            raise PropertyViolationError("row_meta length mismatch")
        if (lens < 1).any():
            raise PropertyViolationError(f"empty row {int(np.flatnonzero(lens < 1)[0])} (basis members are nonzero)")
        if len(ci):
            starts = np.zeros(len(ci), dtype=bool)
            starts[rp[:-1]] = True
            d = np.diff(ci)
            bad = (d <= 0) & ~starts[1:]
            if bad.any():
                row = int(np.searchsorted(rp, np.flatnonzero(bad)[0] + 1, side="right") - 1)
                raise PropertyViolationError(f"row {row} columns not strictly ascending")
            oob = (ci < 0) | (ci >= len(dk))
            if oob.any():
                row = int(np.searchsorted(rp, np.flatnonzero(oob)[0], side="right") - 1)
                raise PropertyViolationError(f"row {row} column out of range")
        if len(va) and (va == 0).any():
            raise PropertyViolationError("zero value stored in plan")
        if len(dk) > 1 and not (key_cmp_rows(dk[:-1], dk[1:]) == 1).all():
            raise PropertyViolationError("dictionary keys not strictly descending")
        if not (c.r == len(rp) - 1 and c.N == len(dk) and c.M == int(rp[-1]) and c.nnz == c.M
                and c.keys_emitted == c.M and c.keys_generated_total >= c.M):
            raise PropertyViolationError(f"counters inconsistent: {c}")


def row_sort_key(row: Row, ring: Ring):
    return (row.role.value, row.provenance, mon_key_pack(row.shift, ring), row.basis_index)


def select_rows(spec: BatchSpec, basis: SoaPolySet) -> list:
    """Two S-pair halves per target, optional admissibility filter, then the
    deterministic order (role, pair id, key(shift), basis index)
    (reference :166-201).  Shifts and sort keys are computed over arrays;
    a malformed target takes the per-row path, which raises the reference's
    error for it."""
    ring = basis.ring
    n_basis = len(basis)
    targets = list(spec.targets)
    if not targets:
        return []
    n = ring.n_vars
    fg = np.array([(t.fi, t.gi) for t in targets], dtype=np.int64)
    bad = np.flatnonzero(((fg < 0) | (fg >= n_basis)).any(axis=1))
    if len(bad):
        raise UncoverableTargetError(f"pair {targets[int(bad[0])].pair_id} references unknown basis index")
    try:
        lcm = np.array([t.lcm for t in targets], dtype=np.int64)
    except (ValueError, TypeError):
        lcm = None
    idx = fg.reshape(-1)
    lead = np.asarray(basis.exps)[np.asarray(basis.offset)[idx]].astype(np.int64, copy=False)
    if lcm is None or lcm.shape != (len(targets), n) or lead.shape != (len(idx), n) or \
            (np.repeat(lcm, 2, axis=0) < lead).any():
        return _select_rows_loop(spec, basis, targets)
    shift = np.repeat(lcm, 2, axis=0) - lead
    pid = np.repeat(np.array([t.pair_id for t in targets], dtype=np.int64), 2)
    rows = [Row(sh, k, RowRole.SPOLY_HALF, q)
            for sh, k, q in zip(map(tuple, shift.tolist()), idx.tolist(), pid.tolist())]
    if spec.adm is not None:
        keep = np.fromiter((bool(spec.adm(r.shift, r.basis_index, r.role, r.provenance)) for r in rows),
                           dtype=bool, count=len(rows))
        alive = set(pid[keep].tolist())
        for tgt in targets:
            if tgt.pair_id not in alive:
                raise UncoverableTargetError(f"target {tgt.lcm} of pair {tgt.pair_id} has no admissible rows")
        sel = np.flatnonzero(keep)
        rows = [rows[i] for i in sel.tolist()]
        shift, idx, pid = shift[sel], idx[sel], pid[sel]
    if not rows:
        return rows
    # (role, pair id, key(shift), basis index); every row here is an S-half
    keys = key_pack_vec(shift, ring)
    order = np.lexsort((idx,) + tuple(keys[:, w] for w in reversed(range(keys.shape[1]))) + (pid,))
    return [rows[i] for i in order.tolist()]


def _select_rows_loop(spec: BatchSpec, basis: SoaPolySet, targets: list) -> list:
    ring = basis.ring
    rows = []
    for tgt in targets:
        for k in (tgt.fi, tgt.gi):
            lead = tuple(int(x) for x in basis.exps[int(basis.offset[k])])
            rows.append(Row(mon_div(tgt.lcm, lead), k, RowRole.SPOLY_HALF, tgt.pair_id))
    if spec.adm is not None and rows:
        kept = [r for r in rows if spec.adm(r.shift, r.basis_index, r.role, r.provenance)]
        alive = {r.provenance for r in kept}
        for tgt in targets:
            if tgt.pair_id not in alive:
                raise UncoverableTargetError(f"target {tgt.lcm} of pair {tgt.pair_id} has no admissible rows")
        rows = kept
    rows.sort(key=lambda r: row_sort_key(r, ring))
    return rows


def _empty_plan(ring: Ring) -> LayoutPlan:
    return LayoutPlan(ring, np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0, np.uint64),
                      np.zeros((0, ring.n_key_words), np.uint64), (), PlanCounters(),
                      {"dict_build_ns": 0, "row_assemble_ns": 0})


def compile_batch(rows, basis: SoaPolySet, closure: Closure = Closure.ONE_STEP_REDUCTION,
                  policy: ExecPolicy = DEFAULT_POLICY, candidates=None, *, dict_cap: int | None = None) -> LayoutPlan:
    """Compile a deterministic row list into a layout plan on the GPU.

    Same contract as the reference (:293-388): closure rows are appended per
    discovery round; the result is independent of ``policy``.  Errors map
    to the reference exceptions (MissingKeyError, SizeCapError,
    LaneOverflowError, PropertyViolationError).  ``dict_cap`` (keyword only,
    not in the reference signature) overrides DICT_CAP for internal callers
    whose reference counterpart has no cap (the final interreduction).
    """
    from .engine import Engine

    ring = basis.ring
    rows = list(rows)
    if not rows:
        return _empty_plan(ring)
    eng = Engine.for_ring(ring)
    eng.sync_basis(basis)
    n = ring.n_vars
    # the Row list -> (int32 basis index, u16 shift lanes), walked in C
    rb = np.empty(len(rows), dtype=np.int32)
    sh = np.empty((len(rows), n), dtype=np.uint16)
    bmin, bmax, lane_ok = native().pack_rows(rows, n, rb, sh)
    if bmin < 0 or bmax >= len(basis):
        raise IndexError("row references a basis index out of range")
    if not lane_ok:
        raise LaneOverflowError("shift exponent does not fit a 16-bit lane")
    # compare by value: callers may pass the reference's own Closure enum
    one_step = getattr(closure, "value", closure) == Closure.ONE_STEP_REDUCTION.value
    dev = eng.compile(rb, sh, one_step,
                      None if candidates is None else list(candidates), DICT_CAP if dict_cap is None else dict_cap)
    info = dev.info
    M = info["M"]
    counters = PlanCounters(r=info["r"], N=info["N"], M=M, nnz=M, closure_rounds=info["closure_rounds"],
                            keys_emitted=M, keys_generated_total=M)
    timings = {"dict_build_ns": info["dict_build_ns"], "row_assemble_ns": info["row_assemble_ns"]}
    plan = LayoutPlan(ring, counters=counters, timings_ns=timings, device=dev, input_rows=rows)
    # reference :383-387, on the device: fused into the compile launch
    # (info["validated"]) or one f4b_plan_validate pass
    if info.get("validated"):
        plan._check_device_counters()
    else:
        plan.validate()
    return plan


def closure_expand(dict_keys_desc: np.ndarray, basis: SoaPolySet, done=None, candidates=None,
                   round_id: int = 1) -> list:
    """One standalone closure round (reference :238-278), host-side utility.

    ``compile_batch`` never calls this: its closure rounds run on the device
    (``k_closure_search`` in ``csrc/fbsp.cu``).  Kept for API compatibility.
    """
    ring = basis.ring
    nd = len(dict_keys_desc)
    if nd == 0:
        return []
    done = np.zeros(nd, dtype=bool) if done is None else np.asarray(done, dtype=bool)
    cands = list(range(len(basis))) if candidates is None else list(candidates)
    todo = np.flatnonzero(~done)
    if todo.size == 0:
        return []
    mons = key_unpack_vec(np.asarray(dict_keys_desc)[todo], ring)
    lms = basis.exps[basis.offset[np.asarray(cands, dtype=np.int64)]]
    lmk = key_pack_vec(lms, ring)
    order = sorted(range(len(cands)), key=lambda q: (tuple(int(w) for w in lmk[q]), cands[q]))
    red = np.full(todo.size, -1, dtype=np.int64)
    for q in order:
        hit = (red < 0) & (mons >= lms[q]).all(axis=1)
        red[hit] = cands[q]
    out = []
    for j in range(todo.size - 1, -1, -1):
        k = int(red[j])
        if k >= 0:
            lead = tuple(int(x) for x in basis.exps[int(basis.offset[k])])
            out.append(Row(mon_div(tuple(int(x) for x in mons[j]), lead), k, RowRole.REDUCER, round_id))
    return out


def decode_row(plan: LayoutPlan, i: int) -> Poly:
    if not 0 <= i < plan.n_rows:
        raise IndexError(f"row {i} out of range")
    s, e = int(plan.row_ptr[i]), int(plan.row_ptr[i + 1])
    exps = plan.dict_exps()[plan.col_ind[s:e]]
    return Poly(plan.ring, tuple((tuple(int(x) for x in ex), int(v))
                                 for ex, v in zip(exps.tolist(), plan.val[s:e].tolist())))


def row_lead_cols(plan: LayoutPlan) -> np.ndarray:
    if plan.n_rows == 0:
        return np.zeros(0, dtype=np.int64)
    return plan.col_ind[plan.row_ptr[:-1]]


_BUCKETS = (1, 2, 4, 8, 16, 32, 64, 128, 256, 1 << 62)


def plan_stats(plan: LayoutPlan) -> dict:
    lens = np.diff(plan.row_ptr)
    hist = {}
    lo = 0
    for b in _BUCKETS:
        k = int(((lens > lo) & (lens <= b)).sum())
        if k:
            hist[f"<={b}" if b < (1 << 62) else f">{lo}"] = k
        lo = b
    c = plan.counters
    return {"r": c.r, "N": c.N, "M": c.M, "nnz": c.nnz, "closure_rounds": c.closure_rounds,
            "keys_emitted": c.keys_emitted, "keys_generated_total": c.keys_generated_total,
            "row_length_histogram": hist}


def _plan_text_parts(plan: LayoutPlan):
    """The lines of plan_to_text as byte chunks.  A device plan whose arrays
    were never touched on the host streams its number lists from the device
    (f4b_plan_text) instead of formatting millions of ints in
    Python; the bytes are identical either way."""
    c = plan.counters
    yield (f"fpgb-plan v1\np {plan.ring.modulus.p}\norder {plan.ring.order}\nvars " + " ".join(plan.ring.var_names)
           + f"\ncounters r={c.r} N={c.N} M={c.M} nnz={c.nnz} closure_rounds={c.closure_rounds} "
           f"keys_emitted={c.keys_emitted} keys_generated_total={c.keys_generated_total}\n").encode()
    dev = plan.device
    for name in ("row_ptr", "col_ind", "val", "dict_keys"):
        yield f"{name} ".encode()
        if dev is not None and name not in plan._host:
            yield dev.text(name)
        else:
            yield " ".join(map(str, np.asarray(getattr(plan, name)).ravel().tolist())).encode()
        yield b"\n"
    meta = " ".join(",".join([*map(str, r.shift), str(r.basis_index), str(r.role.value), str(r.provenance)])
                    for r in plan.row_meta)
    yield ("row_meta " + meta + "\n").encode()


def plan_to_text(plan: LayoutPlan) -> str:
    """Canonical dump (reference :438-460), byte-identical."""
    return b"".join(_plan_text_parts(plan)).decode()


def plan_digest(plan: LayoutPlan) -> str:
    h = hashlib.sha256()
    for part in _plan_text_parts(plan):
        h.update(part)
    return h.hexdigest()
