"""Benchmark: Macaulay nnz/s assembled + F_p reduction s/F4 step on cyclic-8 / F_32003.

Workload (BASELINE.json metric config, fits one GPU): every F4 batch of the
cyclic-8 / F_32003 grevlex run.  Setup runs the full F4 computation once on
the GPU (bit-exact with the reference) and captures each batch's row list and
basis prefix; the device basis (final, HBM-resident) then serves all batches
(closure candidates restricted to the batch's basis prefix, which reproduces
the live plans exactly).

One bench *step* = all 38 batches of the run through compile_batch ->
psge_reduce (new-row mode, what the F4 driver consumes).  L2 is flushed
(a 256 MiB write) before every batch, outside the CUDA-event intervals.

  value      = sum(M) / sum(t_sym): nnz assembled per second, t_sym = device
               time of compile_batch (CUDA events inside the engine), inputs
               resident in HBM.
  e2e        = the same metric through the public Python API / C ABI with
               host buffers: each batch uploads its basis + rows (fresh device
               basis) and downloads the assembled LayoutPlan arrays.
  reduction  = F_p reduction seconds per F4 step (psge, device time).

--impl reference times the CPU oracle (a NumPy restatement of the reference
fpgb algorithm, tests pin it byte-for-byte) on a bounded sample: cyclic-8
steps restored from committed reference snapshots.
"""

from __future__ import annotations

import argparse
import gzip
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Macaulay nnz/s assembled + F_p reduction s/F4 step (cyclic-8, 1-8 GPU)"
UNIT = "nnz/s"
WORKLOAD = "cyclic-8 over F_32003, grevlex, all 38 F4 batches (compile_batch + psge_reduce)"
CPU_SAMPLE_STEPS = (5, 6, 7)


def _traffic_from_profiles():
    """DRAM bytes per launch (dram__bytes_read + write) from the committed
    `ncu --set full` summary (profiles/*/traffic.json), keyed by kernel."""
    out = {}
    pdir = os.path.join(ROOT, "profiles")
    for sub in sorted(os.listdir(pdir)) if os.path.isdir(pdir) else []:
        path = os.path.join(pdir, sub, "traffic.json")
        if os.path.exists(path):
            try:
                with open(path) as fh:
                    out.update(json.load(fh))
            except Exception:
                pass
    return out


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# CPU baseline: the oracle on reference snapshots
# ---------------------------------------------------------------------------
def cpu_sample(steps=CPU_SAMPLE_STEPS):
    import oracle
    from paper_2601_06765_b200.groebner import GroebnerState, Pair, _make_pair, select_batch
    from paper_2601_06765_b200.symbolic import select_rows
    from paper_2601_06765_b200.systems import parse_system

    path = os.path.join(ROOT, "tests", "golden", "cyclic8_p32003.snap.json.gz")
    if not os.path.exists(path):
        return {"M": 0, "t_sym": 0.0, "t_num": 0.0, "steps": []}
    with gzip.open(path, "rt") as fh:
        snaps = json.load(fh)["snapshots"]
    tot_M = tot_sym = tot_num = 0.0
    done = []
    for k in steps:
        snap = snaps.get(str(k))
        if snap is None:
            continue
        ring, basis = parse_system(snap["basis"])
        st = GroebnerState(ring)
        for f in basis:
            st._push_basis(f)
        st.pairs = sorted([_make_pair(st, i, j) for i, j in snap["pairs"]], key=Pair.sort_tuple)
        spec, _ = select_batch(st)
        soa = st.soa()
        rows = [(r.shift, r.basis_index, r.role.value, r.provenance) for r in select_rows(spec, soa)]
        t0 = time.perf_counter()
        plan = oracle.compile_batch_arrays(rows, (soa.exps, soa.coeff, soa.offset, soa.length), ring.order)
        t1 = time.perf_counter()
        oracle.psge_arrays(len(plan["row_ptr"]) - 1, plan["counters"]["N"], plan["row_ptr"], plan["col_ind"],
                           plan["val"], ring.modulus.p)
        t2 = time.perf_counter()
        tot_M += plan["counters"]["M"]
        tot_sym += t1 - t0
        tot_num += t2 - t1
        done.append(k)
    return {"M": tot_M, "t_sym": tot_sym, "t_num": tot_num, "steps": done}


def run_reference(args, rank):
    if rank != 0:
        return
    for _ in range(args.warmup):
        cpu_sample()
    tM = tS = tN = 0.0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        s = cpu_sample()
        tM += s["M"]
        tS += s["t_sym"]
        tN += s["t_num"]
    wall = time.perf_counter() - t0
    value = tM / tS
    sample = (f"cyclic-8/F_32003 F4 steps {list(CPU_SAMPLE_STEPS)} restored from reference snapshots; "
              "NumPy oracle port of fpgb compile_batch + psge_reduce, single-threaded")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * wall / max(1, args.steps),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32 residues mod p",
        "data": "synthetic (generated cyclic-8 system)",
        "config": {"workload": WORKLOAD + " [CPU sample]", "sample_steps": list(CPU_SAMPLE_STEPS)},
        "reduction_s_per_f4_step": tN / (args.steps * len(CPU_SAMPLE_STEPS)),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU workload capture
# ---------------------------------------------------------------------------
def capture_workload():
    from paper_2601_06765_b200.groebner import GroebnerState, f4_step, update_pairs
    from paper_2601_06765_b200.polynomials import poly_monic
    from paper_2601_06765_b200.systems import gen_cyclic

    ring, polys = gen_cyclic(8, 32003)
    st = GroebnerState(ring)
    for f in polys:
        update_pairs(st, poly_monic(f))
    batches = []

    def cap(rows, soa, plan):
        n = ring.n_vars
        batches.append({
            "rows": rows,
            "rb": np.fromiter((r.basis_index for r in rows), dtype=np.int64, count=len(rows)),
            "sh": np.asarray([r.shift for r in rows], dtype=np.int64).reshape(len(rows), n),
            "n_basis": len(soa), "n_terms": soa.total_terms(),
            "r": plan.counters.r, "N": plan.counters.N, "M": plan.counters.M,
        })

    t0 = time.perf_counter()
    while st.n_pairs():
        f4_step(st, _capture=cap)
    return ring, st, batches, time.perf_counter() - t0


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled during the timed
    region: in-process NVML queries taken between engine calls, at most every
    100 ms (a concurrent poller — nvidia-smi -lms 100 or an NVML thread —
    measured to stall the driver now and then inside the event intervals and
    inflate a run by up to 30 %), with `nvidia-smi -lms 100` as the fallback
    when NVML is unavailable.  Only samples inside [t_begin, t_end] count."""

    # nvmlClocksEventReason bits
    _BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None
        self.thread = None
        self.rows = []
        self.max_mhz = None
        self.t_begin = self.t_end = None
        self._sample = None

    def start(self):
        if os.environ.get("F4B_BENCH_NO_SMI"):  # diagnostic: no sampling at all
            return self
        try:
            import threading

            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self._physical_index())
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def sample():
                try:
                    mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.rows.append((time.time(), float(mhz), self.max_mhz, int(rs)))
                except Exception:
                    pass

            self._sample = sample
            self.thread = True
            return self
        except Exception:
            self.thread = None
            self._sample = None
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        fields = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                  "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                  "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={fields}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(1.0)  # nvidia-smi needs a moment before its first sample
        return self

    def _physical_index(self):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            try:
                return int(vis.split(",")[self.device])
            except (ValueError, IndexError):
                pass
        return self.device

    def maybe_sample(self, period=0.1):
        """NVML mode: one sample from the calling thread, between engine calls
        (so a driver stall during the query lands outside the CUDA-event
        intervals the metric sums), at most every `period` seconds."""
        if self.thread is not None and self._sample is not None:
            now = time.time()
            if not self.rows or now - self.rows[-1][0] >= period:
                self._sample()

    def begin(self):
        self.t_begin = time.time()
        self.maybe_sample(0.0)

    def end(self):
        self.maybe_sample(0.0)
        self.t_end = time.time()

    def stop(self):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def _read_smi(self):
        import datetime

        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        rows = []
        try:
            for line in open(self.path):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 8:
                    continue
                try:
                    ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                except ValueError:
                    continue
                bits = 0
                for nm, flag in zip(names, parts[4:8]):
                    if flag.lower().startswith("active"):
                        bits |= self._BITS[nm]
                rows.append((ts, float(parts[1]), float(parts[2]), bits))
            os.unlink(self.path)
        except Exception:
            pass
        return rows

    def summary(self):
        rows = self.rows if self.thread is not None else (self._read_smi() if self.path else [])
        inside = [r for r in rows if self.t_begin is not None and self.t_begin - 0.05 <= r[0] <= self.t_end + 0.05]
        note = "samples inside the timed region"
        if not inside and rows and self.t_begin is not None:
            # timed region shorter than the sampling period: nearest samples
            inside = sorted(rows, key=lambda r: abs(r[0] - 0.5 * (self.t_begin + self.t_end)))[:2]
            note = "timed region shorter than the sampling period: nearest samples"
        reasons = sorted({nm for r in inside for nm, bit in self._BITS.items() if r[3] & bit})
        return {"sm_mhz": statistics.median([r[1] for r in inside]) if inside else None,
                "sm_max_mhz": max(r[2] for r in inside) if inside else None, "reasons": reasons,
                "samples": len(inside), "note": note,
                "source": "nvml" if self.thread is not None else ("nvidia-smi" if self.path else "none")}


# Algorithmic bytes per kernel per batch — DESIGN.md §4.
#   k_fbsp (whole compile_batch) : B_sym of SURVEY.md §8(d): every term's
#                                  source key + coefficient in, col_ind + val
#                                  out, row_ptr, the dictionary
#                                  M(8W+4) + 8M + 4(r+1) + 8W N
#   k_sweep<0> (C rows by A)     : every pivot-row application streams the
#                                  pivot tail (u32 col + u32 val) and its
#                                  16-byte descriptor; the C rows are read
#                                  and D' is written once
#                                  8 tail_nnz + 16 pivots + 8 nnz(C) + 4|C|K
#                                  (pivot rows are reused across C rows, so
#                                  this stream is L2-served, not HBM)
#   k_dense_forward              : read + write D' once       8|C|K
#   k_dense_blk                  : D' read + RREF(D') written 4|C|K + 4 rank(D') K
SYMBOLIC = ("k_fbsp", "k_rank_", "k_tile_dict", "k_join_gen", "k_os_", "k_small_sort", "k_unique_absent",
            "k_closure", "k_new_rows", "k_merge_corank", "k_rows0", "k_encode_basis", "k_mark_leads", "k_front0",
            "k_dict_exps")


def kernel_bytes(name, b, pinfo, einfo):
    M = b["M"]
    KW = pinfo["key_words"]
    C, K = einfo["dense_rows"], einfo["dense_cols"]
    if name.startswith("k_fbsp"):
        return M * (8 * KW + 4) + 8 * M + 4 * (b["r"] + 1) + 8 * KW * b["N"]
    if name.startswith(("k_rank_join", "k_join_gen")):
        return M * (8 * KW + 4) + 8 * M
    if name.startswith(("k_rank_fill", "k_tile_dict")):
        return M * 8 * KW
    if "k_sweep_win" in name:
        # packed pivot tails (4-byte col|val entries in 4-entry groups when
        # N < 2^16 and p < 2^16, else 8-byte pairs), streamed once per applied
        # pivot; the C rows read once, D' written once
        c_nnz = int(C * M / max(1, b["r"]))
        entry = 4 if "<true>" in name else 8
        return entry * einfo["sweep_tail_nnz"] + 8 * c_nnz + 4 * C * K
    if "k_sweep" in name:
        # C-row share of the nonzeros: |C| rows of mean length M / r
        c_nnz = int(C * M / max(1, b["r"]))
        return 8 * einfo["sweep_tail_nnz"] + 16 * einfo["sweep_pivots"] + 8 * c_nnz + 4 * C * K
    if name.startswith("k_dense_blk"):
        # compulsory: D' read once, RREF(D') written once (the per-block
        # products re-read L2-resident rows and are not credited)
        return 4 * C * K + 4 * einfo["n_nonpivot_rows"] * K
    if name in ("k_dense_forward", "k_dense_fwd_smem", "k_dense_forward_cta"):
        # D' read into the row state and the pivot rows written back once
        return 8 * C * K
    return None


def roofline_for(kprof, records, peak, peak_src, want):
    """Roofline of the most expensive kernel accepted by `want` (with a byte model)."""
    total = max(1.0, sum(v[1] for v in kprof.values()))
    for name, (cnt, ns) in sorted(kprof.items(), key=lambda kv: -kv[1][1]):
        if not want(name) or ns <= 0:
            continue
        tot = 0
        for b, pinfo, einfo in records:
            kb = kernel_bytes(name, b, pinfo, einfo)
            if kb is None:
                tot = None
                break
            tot += kb
        if tot is None:
            return {"bound": "latency", "kernel": name, "achieved": None, "peak": peak, "unit": "GB/s", "frac": None,
                    "traffic": None, "launches": cnt, "avg_launch_us": ns / cnt / 1e3, "share_of_step": ns / total,
                    "note": "no algorithmic byte model (schedule-dependent work)"}
        ach = tot / (ns * 1e-9) / 1e9
        out = {"bound": "hbm", "kernel": name, "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
               "traffic": None, "launches": cnt, "avg_launch_us": ns / cnt / 1e3, "peak_source": peak_src,
               "share_of_step": ns / total, "algorithmic_bytes_per_launch": tot / cnt}
        if "k_sweep_win" in name:
            out["note"] = ("pivot tails packed once per matrix and L2-resident (reused by every C row); fixed "
                           "32-A-column windows with precomputed block inverses: multipliers from one 32x32 "
                           "product, two CTA barriers per non-empty window, shared-atomic tail application")
        elif name.startswith("k_dense_blk"):
            out["note"] = ("latency-bound: RREF(D') in pivot blocks, two grid barriers per block of up to 32 "
                           "pivots; byte model counts D' read and RREF(D') written once")
        elif name.startswith("k_dense_fwd"):
            out["note"] = ("latency-bound: one grid barrier per pivot of D' (byte model counts D' once; the "
                           "per-pivot row updates stay in shared memory)")
        return out
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-micro", action="store_true", help="skip the primitive microbenchmarks")
    ap.add_argument("--no-katsura11", action="store_true",
                    help="skip the full Katsura-11 run reported next to the line (rank 0, after the timed region)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2601_06765_b200.engine import Engine
    from paper_2601_06765_b200.sparselin import csr_from_plan, psge_reduce
    from paper_2601_06765_b200.symbolic import compile_batch

    ring, st, batches, setup_s = capture_workload()
    # the whole run also ends with the device interreduction (§8f.1); report
    # both next to the reference's own timings of the same run (golden file)
    from paper_2601_06765_b200.groebner import reduce_basis_device

    t0 = time.perf_counter()
    gb = reduce_basis_device(st.basis, ring)
    reduce_s = time.perf_counter() - t0
    full_run = {"system": "cyclic-8 / F_32003", "f4_loop_s": round(setup_s, 3), "reduce_basis_s": round(reduce_s, 3),
                "gb_size": len(gb)}
    try:
        with open(os.path.join(ROOT, "tests", "golden", "cyclic8_p32003.json")) as fh:
            g = json.load(fh)
        full_run.update(reference_f4_loop_s=g["f4_loop_s"], reference_reduce_basis_s=g["reduce_basis_s"],
                        reference_gb_size=g["gb_size"])
    except Exception:
        pass
    eng = Engine.for_ring(ring, local)
    eng.sync_basis(st.soa())  # the interreduction above replaced the device basis
    total_M = sum(b["M"] for b in batches)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    _dbg = [] if os.environ.get("F4B_BENCH_DEBUG") else None

    def replay_step(record):
        ts = tn = 0
        for b in batches:
            clk.maybe_sample()
            flush.fill_(1)
            plan = eng.compile(b["rb"], b["sh"], True, list(range(b["n_basis"])))
            ech = eng.psge_plan(plan, full=False)
            inf = ech.info()
            ts += plan.info["dict_build_ns"] + plan.info["row_assemble_ns"]
            tn += inf["numeric_ns"]
            if _dbg is not None:
                _dbg.append((b["r"], (plan.info["dict_build_ns"] + plan.info["row_assemble_ns"]) / 1e6,
                             inf["numeric_ns"] / 1e6))
            if record is not None:
                record.append((b, plan.info, inf))
        return ts, tn

    clk = ClockSampler(local).start()
    for _ in range(args.warmup):
        replay_step(None)
    # timed region
    eng.profile(True)
    _, launches0 = eng.profile_read()
    records = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk.begin()
    w0 = time.perf_counter()
    t_sym = t_num = 0
    for _ in range(args.steps):
        a, c = replay_step(records)
        t_sym += a
        t_num += c
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    clk.end()
    clk.stop()
    if world > 1:
        dist.barrier()
    kprof, launches1 = eng.profile_read()
    eng.profile(False)
    t_tot_ns = float(t_sym + t_num)
    if world > 1:
        t = torch.tensor([t_tot_ns, float(t_sym)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_tot_ns, t_sym = float(t[0]), float(t[1])
    ms_per_step = t_tot_ns / 1e6 / args.steps
    value = world * total_M * args.steps / (t_sym / 1e9)
    red_s = t_num / 1e9 / (args.steps * len(batches))

    # roofline: the dominant kernel with an algorithmic byte model
    peak, peak_src = _peaks()
    ranked = sorted(kprof.items(), key=lambda kv: -kv[1][1])
    roof = roofline_for(kprof, records, peak, peak_src, lambda nm: True)
    roof_sym = roofline_for(kprof, records, peak, peak_src, lambda nm: nm.startswith(SYMBOLIC))
    traffic = _traffic_from_profiles()
    for rf in (roof, roof_sym):
        if rf and rf.get("kernel") in traffic:
            rf["traffic"] = traffic[rf["kernel"]]
    # symbolic (FBSP) effective roofline, B_sym per SURVEY.md §8(d)
    W = ring.n_key_words
    B_sym = sum(b["M"] * (8 * W + 4) + 8 * b["M"] + 4 * (b["r"] + 1) + b["N"] * 8 * W for b in batches)
    sym_frac = (B_sym * args.steps / (t_sym / 1e9) / 1e9) / peak

    # e2e: the public API with host buffers, replaying the run as the F4
    # driver does it: the device basis starts empty each step and grows batch
    # by batch (sync_basis appends the polynomials added since the previous
    # batch, from page-locked copies of the basis streams); per batch the row
    # list goes up, compile_batch runs, and the LayoutPlan arrays
    # (row_ptr, col_ind, val, dict_keys) come back to host memory.
    e2e = None
    if args.e2e_steps > 0:
        from paper_2601_06765_b200.engine import host_empty
        from paper_2601_06765_b200.polynomials import SoaPolySet

        final = st.soa()

        def pinned(a):
            out = host_empty(a.shape, a.dtype)
            out[...] = a
            return out

        f_key, f_coeff, f_exps = pinned(final.mon_key), pinned(final.coeff), pinned(final.exps)
        n = ring.n_vars
        h2d = d2h = 0
        e_sym = 0.0
        e_M = 0
        for it in range(args.e2e_steps + 1):  # iteration 0 warms the host caches, untimed
            if it == 1:
                h2d = d2h = e_M = 0
                e_sym = 0.0
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            eng.clear_basis()
            prev_nt = prev_nb = 0
            for b in batches:
                nb_, nt = b["n_basis"], b["n_terms"]
                soa = SoaPolySet(ring, f_key[:nt], f_coeff[:nt], final.offset[:nb_ + 1], final.length[:nb_],
                                 f_exps[:nt])
                plan = compile_batch(b["rows"], soa)
                rp, ci, va = plan.row_ptr, plan.col_ind, plan.val
                dk = plan.dict_keys
                e_M += b["M"]
                # bytes moved: new basis terms as the reference streams them
                # (int64 exps + uint64 coeff, narrowed on the device), their
                # lengths + offsets, back their LM / max exponents; rows (basis
                # index + shift); back: row_ptr / col_ind / val (64-bit) and
                # dict_keys (reference key words)
                h2d += (nt - prev_nt) * (8 * n + 8) + (nb_ - prev_nb) * 16 + len(b["rows"]) * (4 + 2 * n)
                d2h += ((nb_ - prev_nb) * 4 * n + (plan.counters.r + 1) * 8 + plan.counters.M * 16
                        + plan.counters.N * 8 * ring.n_key_words)
                prev_nt, prev_nb = nt, nb_
                del rp, ci, va, dk, plan
            torch.cuda.synchronize()
            e_sym += time.perf_counter() - t0
        e2e = {"value": world * e_M / e_sym, "unit": UNIT, "h2d_bytes_per_step": h2d // args.e2e_steps,
               "d2h_bytes_per_step": d2h // args.e2e_steps,
               "note": ("per step: empty device basis, then per batch the new basis polys + rows H2D, "
                        "compile_batch, LayoutPlan arrays D2H (page-locked); wall clock incl. Python API")}
        eng.clear_basis()

    # the other north-star system: the full Katsura-11 / F_32003 computation
    # (the reference cannot finish it: its step 4 alone takes 1,556 s on one
    # core).  Katsura-11 has 2^11 solutions, so the reduced basis must leave
    # exactly 2048 standard monomials; steps 3-4 are pinned to the reference
    # by tests/test_gpu_parity.py::test_large_step_replay.
    k11 = None
    if rank == 0 and not args.no_katsura11:
        from paper_2601_06765_b200.groebner import f4_groebner as _f4
        from paper_2601_06765_b200.systems import format_system, gen_katsura

        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from full_run import standard_monomials

        kring, kpolys = gen_katsura(11, 32003)
        t0 = time.perf_counter()
        kgb = _f4(kpolys, kring)
        k11 = {"system": "Katsura-11 / F_32003, grevlex, full F4 + device interreduction",
               "wall_s": round(time.perf_counter() - t0, 3), "gb_size": len(kgb),
               "standard_monomials": standard_monomials([f.lm() for f in kgb], kring.n_vars),
               "expected_standard_monomials": 2 ** 11,
               "sha256": __import__("hashlib").sha256(format_system(kring, kgb).encode()).hexdigest(),
               "reference": "does not finish (SURVEY.md 6.2: step 4 alone 1,556 s)"}

    # kernel capability at large M: the reference's own microbenchmarks
    # (fpgb.bench.microbench, SURVEY.md §8d "synthetic dict_build") on the
    # device primitives, inputs resident in HBM (larger than L2)
    micro = None
    if rank == 0 and not args.no_micro:
        from paper_2601_06765_b200.bench import microbench

        micro = []
        for kind, size, dup in (("dict_build", 1 << 24, 0.5), ("dict_build", 1 << 24, 0.99),
                                ("row_assemble", 1 << 24, 0.0), ("mod_fma", 1 << 26, 0.0)):
            m = microbench(kind, size, dup, seed=0)
            keep = ("kind", "size", "duplicate_rate", "unique_out", "radix_passes", "keys_per_s", "joins_per_s",
                    "updates_per_s.barrett", "algorithmic_bytes", "hbm_frac", "dict_path", "hbm_frac_streamed")
            ent = {k: m[k] for k in keep if k in m}
            ent["us"] = round(m.get("elapsed_ns", m.get("elapsed_ns.barrett", 0)) / 1e3, 1)
            micro.append(ent)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        s = cpu_sample()
        if s["t_sym"] > 0:
            cpu = {"value": s["M"] / s["t_sym"], "unit": UNIT, "cores": 1, "kind": "port",
                   "sample": f"cyclic-8 F4 steps {s['steps']} from reference snapshots, NumPy oracle port, "
                             f"compile {s['t_sym']:.2f}s + psge {s['t_num']:.2f}s"}
    if rank == 0:
        kernels = {k: {"launches": v[0], "ms": round(v[1] / 1e6, 3)} for k, v in ranked[:12]}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32 residues mod p (u64 monomial keys)",
            "data": "synthetic (generated cyclic-8 system, deterministic)",
            "config": {"workload": WORKLOAD, "batches": len(batches), "sum_M_per_step": total_M,
                       "parallelism": "replicas" if world > 1 else "single",
                       "l2": "flushed (256 MiB write) before every batch"},
            "reduction_s_per_f4_step": red_s,
            "symbolic_roofline": {"B_sym_bytes_per_step": B_sym, "frac": sym_frac, "peak": peak},
            "roofline": roof, "roofline_symbolic": roof_sym, "cpu_baseline": cpu, "e2e": e2e,
            "clocks": clk.summary(),
            "gpu_launches": launches1 - launches0, "wall_ms_per_step": 1000 * wall / args.steps,
            "debug_slowest": (sorted(_dbg, key=lambda x: -(x[1] + x[2]))[:8] if _dbg else None),
            "setup_s": round(setup_s, 2), "full_run": full_run, "full_run_katsura11": k11, "kernels_top": kernels,
            "microbench": micro,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
