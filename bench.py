"""Benchmark of the modular-determinant hot path (BASELINE.json metric:
mod-p n x n dets/s and end-to-end time per polynomial determinant).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5|c3] [--impl ours|reference]

Workload (default `--config c5`, BASELINE.json configs[4], the largest
single-GPU configuration): 40x40 matrix, 3 variables, entry degree <= 4,
256^3 = 16.7 M evaluation nodes per prime, 23 primes.  One STEP = the hot path
for one prime: forward evaluation of all 1600 unique entries (partial NTT +
fused last-axis evaluation), the 40x40 determinants mod p at the kept nodes
(the degree bound 160 per variable needs 168 x 168 x 176 = 4.97 M of the 16.7 M
nodes, csrc/expand.cu) and the coefficients interpolated straight from those
nodes (one pass per axis, pdb_grid_interpolate_u32; the residue tensor equals
the inverse NTT of the reference's full determinant grid).  Weak scaling: every rank runs one prime per step (ranks take
primes round-robin).

  value  determinants COMPUTED per second (elimination at the kept nodes) over
         all ranks, inputs resident in HBM (working set 2.2 GB per prime >> 126
         MB L2, so no flush is needed between steps).  `grid_dets_per_s` is the
         full 16.7 M-node determinant grid produced per second (every value
         bit-identical to the reference's det_grid there).
  e2e    same metric with, every step, the H2D copy of the step's input
         coefficients from pinned host memory and the D2H copy of the step's
         residue tensor (16.7 M x u32) inside the timed region
  roofline  the det kernel (fused evaluation + elimination): algorithmic
         elimination updates W(40) = (n^3 - n)/3 = 21320 per computed matrix /
         kernel time, against the measured peak of the 9-MAC + REDC primitive
         (and, for reference, the raw accumulating IMAD.WIDE ceiling)
  poly_e2e  seconds per polynomial determinant through the public run_report
         (C1, C2, C3, C4 rungs, C5; sharded when N > 1) next to the CPU path
         (the oracle port of the reference) timed on this host in the same run
  cpu_baseline  the oracle port timed on a bounded sample of the step on this
         host (rank 0, N = 1), extrapolated per step
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

HBM_FALLBACK = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=["c5", "c3"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-poly", action="store_true", help="skip the end-to-end run_report timings")
    return ap.parse_args()


def workload(name):
    from paper_2010_12117_b200 import plan, workloads

    m, cfg = workloads.c5() if name == "c5" else workloads.c3()
    return m, plan(m, cfg)


L2_BYTES = 126 * 2**20


def working_set_bytes(m, pl):
    """Device bytes a step touches: the fused entry layout [outer][E][k] + the
    determinant grid and the scratch denominators (u32 each)."""
    E = max(t.shape[-1] for t in m.unique_entries)
    return 4 * (pl.node_count // pl.shape[-1] * E * m.k + 2 * pl.node_count)


def describe(name, m, pl, ws_bytes):
    big = ws_bytes > 2 * L2_BYTES
    return {"workload": "%s: %dx%d polynomial matrix, %d vars, grid %s = %d nodes/prime, %d primes, k=%d unique entries"
                        % (name.upper(), m.r, m.r, len(pl.variables), "x".join(map(str, pl.shape)),
                           pl.node_count, pl.prime_count, m.k),
            "matrix_order": m.r, "nodes_per_prime": pl.node_count, "primes": pl.prime_count,
            "step": "one prime: forward evaluation + det at the degree-bound node set + the coefficients "
                    "interpolated from those nodes (direct mode) or exact grid extension + inverse NTT",
            "working_set_bytes": ws_bytes,
            "l2_policy": ("inputs larger than L2 (per-step working set %.2f GB >> 126 MB)" % (ws_bytes / 1e9)) if big
            else ("working set %.1f MB fits L2: a 256 MB buffer is written between timed steps (not timed)"
                  % (ws_bytes / 1e6))}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    path = ROOT / "MEASURED_PEAKS.json"
    if path.exists():
        data = json.loads(path.read_text())
        return data.get("hbm_gbs", HBM_FALLBACK), "measured"
    return HBM_FALLBACK, "fallback"


# -- CPU baseline: the oracle port on a bounded sample ---------------------------------------

def cpu_sample(m, pl, det_nodes=4096, threads=None):
    """Time the oracle's per-prime units on this host and extrapolate one step.

    FWD: one unique entry's full ntt_multi on the plan grid (the reference
    transforms every unique entry; its thread pool parallelises across
    entries, so k entries cost k/threads of this).  DET: det_grid on
    `det_nodes` random nodes with all threads.  INV: one ntt_multi inverse.
    """
    from oracle import polydet_oracle as O

    threads = threads or os.cpu_count() or 1
    spec = pl.primes[0]
    p, w, q = spec.p, spec.omega, spec.q
    shape = pl.shape
    entry = m.unique_entries[0].terms()
    t0 = time.perf_counter()
    grid = O.ntt_multi(O.reduce_entry(entry, shape, p), shape, p, w, q)
    t_fwd = time.perf_counter() - t0
    rng = np.random.default_rng(0)
    r = m.r
    grids = [rng.integers(0, p, det_nodes) for _ in range(m.k)]
    t0 = time.perf_counter()
    O.det_grid(grids, r, p, m.entry_ids, chunk=max(det_nodes // threads, 1), workers=threads)
    t_det = time.perf_counter() - t0
    t0 = time.perf_counter()
    O.ntt_multi(grid, shape, p, w, q, inverse=True)
    t_inv = time.perf_counter() - t0
    nodes = pl.node_count
    step = m.k * t_fwd / threads + t_det * nodes / det_nodes + t_inv
    return {"value": nodes / step, "unit": "dets/s", "cores": threads, "kind": "port",
            "sample": "oracle port (numpy restatement of the reference): one full ntt_multi of a unique entry "
                      "(%.2f s; x k=%d / %d threads), det_grid on %d nodes with %d threads (%.2f s), one inverse "
                      "ntt_multi (%.2f s); extrapolated to one prime = %.0f s"
                      % (t_fwd, m.k, threads, det_nodes, threads, t_det, t_inv, step),
            "step_seconds": step}


def run_reference(args):
    """The reference's CPU path on this host (oracle port: the reference itself
    is pure Python and cannot travel to the GPU box).  Each step is a bounded,
    really timed sample of one prime of the workload -- one unique entry's full
    forward transform, det_grid on 4096 nodes, one full inverse transform --
    extrapolated to the whole prime (the reference's own predict() method,
    pipeline.py:242-264); `ms_per_step` is the timed sample, `value` the
    extrapolated per-prime rate."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    m, pl = workload(args.config)
    vals = []
    t_start = time.perf_counter()
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        res = cpu_sample(m, pl, det_nodes=4096)
        res["sample_seconds"] = time.perf_counter() - t0
        if i >= args.warmup:
            vals.append(res)
    value = statistics.median(v["value"] for v in vals)
    base = vals[-1]
    sample_ms = 1e3 * statistics.median(v["sample_seconds"] for v in vals)
    out = {"impl": "reference", "metric": "mod-p %dx%d dets/sec (%s)" % (m.r, m.r, args.config.upper()),
           "value": value, "unit": "dets/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": sample_ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "int64", "data": "synthetic (seeded %s generator)" % args.config.upper(),
           "config": describe(args.config, m, pl, working_set_bytes(m, pl)),
           "extrapolated": True,
           "extrapolated_step_seconds": statistics.median(v["step_seconds"] for v in vals),
           "timed_region_seconds": time.perf_counter() - t_start,
           "cpu_baseline": {"value": value, "unit": "dets/s", "cores": base["cores"], "kind": "port",
                            "sample": base["sample"]},
           "e2e": {"value": value, "unit": "dets/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


POLY_CONFIGS = ("C1", "C2", "C3", "C4_3src_T5T7_m", "C4_4src_T5T11", "C4_4src_T5T11_m", "C4_5src_T7T11",
                "C4_5src_T5T7_m", "C5")


def _poly_workload(name):
    from paper_2010_12117_b200 import workloads
    return {"C1": workloads.c1, "C2": workloads.c2, "C3": workloads.c3, "C5": workloads.c5,
            "C4_3src_T5T7_m": lambda: workloads.harmonic(3, (5, 7), True),
            "C4_4src_T5T11": lambda: workloads.harmonic(4, (5, 11), False),
            "C4_4src_T5T11_m": lambda: workloads.harmonic(4, (5, 11), True),
            "C4_5src_T7T11": lambda: workloads.harmonic(5, (7, 11), False),
            "C4_5src_T5T7_m": lambda: workloads.harmonic(5, (5, 7), True)}[name]()


#: reference run_report seconds with 8 workers in the dev container (8 cores),
#: measured when the golden fixtures were made (tests/golden/c4_results.json,
#: c3_result.json) -- for context next to the same-run CPU timings below
REFERENCE_DEV_SECONDS = {"C3": 161.5, "C4_4src_T5T11": 2.09, "C4_4src_T5T11_m": 151.4,
                         "C4_5src_T7T11": 289.3, "C4_5src_T5T7_m": 600.5}


def cpu_poly(name, m, pl, threads):
    """The CPU path end to end on this host: the oracle port's run_pipeline
    (forward transforms over a thread pool, det_grid with `threads` workers,
    inverse, CRT).  Configurations the port finishes in seconds are timed
    whole; C3 (~7 min with one forward worker) is timed for one full prime plus
    the CRT of real residues and extrapolated to its 22 primes."""
    from oracle import polydet_oracle as O

    terms = [t.terms() for t in m.unique_entries]
    primes = [(s.p, s.omega, s.q) for s in pl.primes]
    if name in ("C1", "C2", "C4_3src_T5T7_m", "C4_4src_T5T11"):
        t0 = time.perf_counter()
        O.run_pipeline(terms, m.entry_ids, m.r, pl.shape, primes, workers=threads)
        return {"seconds": time.perf_counter() - t0, "cores": threads, "kind": "port", "sample": "whole run"}
    if name == "C3":
        t0 = time.perf_counter()
        _, res = O.run_pipeline(terms, m.entry_ids, m.r, pl.shape, primes[:1], workers=threads)
        t_prime = time.perf_counter() - t0
        rows = [res[0]] * len(primes)   # CRT cost is independent of the values' origin
        t0 = time.perf_counter()
        O.crt_combine(rows, [p for p, _, _ in primes])
        t_crt = time.perf_counter() - t0
        return {"seconds": t_prime * len(primes) + t_crt, "cores": threads, "kind": "port", "extrapolated": True,
                "sample": "one full prime timed (%.1f s) x %d primes + CRT of %d coefficients (%.1f s)"
                          % (t_prime, len(primes), pl.node_count, t_crt)}
    return None


def poly_e2e(world, rank, cpu=True):
    """Second half of the BASELINE metric: end-to-end seconds per polynomial
    determinant through the public API (`run_report`: upload, all primes, CRT,
    Python-int result), best of `reps` after one warm-up run.  With N > 1
    processes the run is sharded (executor.execute) and the time is the max
    over ranks.  Next to it: the CPU path on this host in the same run
    (cpu_poly), and the reference's own time from the dev container."""
    import torch
    import torch.distributed as dist

    from paper_2010_12117_b200 import plan, run_report

    threads = os.cpu_count() or 1
    out = []
    for name in POLY_CONFIGS:
        m, cfg = _poly_workload(name)
        pl = plan(m, cfg)
        reps = 1 if name in ("C5", "C4_5src_T5T7_m") else 3
        run_report(m, cfg)   # warm-up: prime contexts, tables, allocator, pinned staging buffer
        best = None
        for _ in range(reps):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            result, timings, _ = run_report(m, cfg)
            wall = time.perf_counter() - t0
            if world > 1:
                tw = torch.tensor([wall], dtype=torch.float64, device="cuda")
                dist.all_reduce(tw, op=dist.ReduceOp.MAX)
                wall = float(tw.item())
            if best is None or wall < best[0]:
                best = (wall, timings)
        wall, timings = best
        rec = {"config": name, "seconds": wall, "n_gpus": world, "primes": pl.prime_count, "nodes": pl.node_count,
               "r": m.r, "stages_s": {"fft": timings.fft, "det": timings.det, "ifft": timings.ifft,
                                      "crt": timings.crt},
               "nonzero_terms": sum(1 for c in result.coeffs if c),
               "reference_dev_container_s": REFERENCE_DEV_SECONDS.get(name)}
        if name in ("C3", "C5") and rank == 0:
            # the result printer (reference parsing.py:211-225 via cli.py:61-83), native
            from paper_2010_12117_b200 import format_polynomial
            t0 = time.perf_counter()
            text = format_polynomial(result, result.axis_vars)
            rec["format_s"] = time.perf_counter() - t0
            rec["format_chars"] = len(text)
            del text
        del result
        if cpu and rank == 0 and world == 1:
            c = cpu_poly(name, m, pl, threads)
            if c is not None:
                rec["reference_cpu_s"] = c.pop("seconds")
                rec["reference_cpu"] = c
            elif name == "C5":
                rec["reference_cpu_s"] = None
                rec["reference_cpu"] = {"note": "infeasible on the CPU path (>= 215 GB of entry grids; ~11.5 days "
                                                "extrapolated, SURVEY.md 6); per-prime rate: cpu_baseline"}
            else:
                rec["reference_cpu_s"] = None
                rec["reference_cpu"] = {"note": "not rerun here (minutes of CPU); reference_dev_container_s is "
                                                "the reference's own run_report with 8 workers"}
        out.append(rec)
    return out


# -- GPU arm --------------------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2010_12117_b200 import executor, native

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hooks: several ranks on one GPU (PDB_BENCH_DEVICE=0) with gloo for the
    # barrier / max-over-ranks plumbing (PDB_DIST_BACKEND=gloo); defaults: NCCL, GPU = local rank
    local = int(os.environ.get("PDB_BENCH_DEVICE", local))
    backend = os.environ.get("PDB_DIST_BACKEND", "nccl")
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)

    m, pl = workload(args.config)
    stages = executor.PrimeStages(m, pl, staged=False)
    P = pl.prime_count
    for spec in pl.primes:
        ctx = native.prime_context(spec, local)
        for n in set(pl.shape):
            ctx.prepare(n)
    stream = torch.cuda.current_stream()

    def prime_of(step):
        return (rank + step * world) % P

    # integer-pipe peaks (no memory traffic), measured on this device now
    peak_delayed = native.mulmod_peak(pl.primes[0].p, 1)
    peak_imadwide = native.mulmod_peak(pl.primes[0].p, 2)

    for s in range(args.warmup):
        stages.step(prime_of(s))
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident timing ----
    sampler = ClockSampler(local)
    launches0 = native.launch_count()
    det_events = []
    barrier()
    sampler.start()
    ws_bytes = working_set_bytes(m, pl)
    flush = None if ws_bytes > 2 * L2_BYTES else torch.empty(64 * 2**20, dtype=torch.int32, device=dev)
    step_events = []
    native.kernel_timing(True)   # CUDA events around every det_gj launch, on its launch stream
    for s in range(args.steps):
        pi = prime_of(s)
        if flush is not None:
            flush.zero_()      # evict the previous step's data from L2 (outside the step's events)
        t0 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        stages.forward(pi)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        stages.det_kernels(pi)
        e1.record(stream)
        det_events.append((e0, e1))
        stages.finish(pi)
        t1 = torch.cuda.Event(enable_timing=True)
        t1.record(stream)
        step_events.append((t0, t1))
    barrier()
    clocks = sampler.stop()
    kern_ms, kern_launches = native.kernel_timing_read()
    native.kernel_timing(False)
    launches = native.launch_count() - launches0
    ms = sum(a.elapsed_time(b) for a, b in step_events)
    det_ms = sum(a.elapsed_time(b) for a, b in det_events)
    tmax = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms = float(tmax.item())
    nodes = pl.node_count
    sel = stages.dp.sel          # determinants computed per step (the kept nodes)
    value = world * sel * args.steps / (ms / 1e3)
    grid_rate = world * nodes * args.steps / (ms / 1e3)

    # ---- end to end: host coefficients in, host residues out, every step ----
    dp = stages.dp
    host_mag = dp.mag.cpu().pin_memory()
    host_neg = dp.neg.cpu().pin_memory()
    host_pos = dp.pos.cpu().pin_memory()
    # the step's residues leave the device on a side stream (double-buffered)
    # while the next step computes; the timed region ends when the last copy lands
    host_out = [torch.empty(nodes, dtype=torch.int32).pin_memory() for _ in range(2)]
    dev_out = [torch.empty(nodes, dtype=torch.int32, device=dev) for _ in range(2)]
    copy_stream = torch.cuda.Stream(device=dev)
    h2d = host_mag.numel() * 4 + host_neg.numel() + host_pos.numel() * 8
    d2h = nodes * 4
    barrier()
    e_start = torch.cuda.Event(enable_timing=True)
    e_end = torch.cuda.Event(enable_timing=True)
    e_start.record(stream)
    for s in range(args.steps):
        pi = prime_of(s)
        dp.mag.copy_(host_mag, non_blocking=True)
        dp.neg.copy_(host_neg, non_blocking=True)
        dp.pos.copy_(host_pos, non_blocking=True)
        stages.step(pi)
        buf = s % 2
        stream.wait_stream(copy_stream)           # dev_out[buf]'s previous D2H is done
        dev_out[buf].copy_(stages.det, non_blocking=True)
        copy_stream.wait_stream(stream)
        with torch.cuda.stream(copy_stream):
            host_out[buf].copy_(dev_out[buf], non_blocking=True)
    stream.wait_stream(copy_stream)
    e_end.record(stream)
    barrier()
    e_ms = e_start.elapsed_time(e_end)
    emax = torch.tensor([e_ms], device=dev)
    if world > 1:
        dist.all_reduce(emax, op=dist.ReduceOp.MAX)
    e_ms = float(emax.item())
    e2e = world * sel * args.steps / (e_ms / 1e3)

    # parity guard on the timed path: the last step's residues vs a fresh recompute
    check = host_out[(args.steps - 1) % 2].clone()
    stages.step(prime_of(args.steps - 1))
    torch.cuda.synchronize()
    assert torch.equal(check, stages.det.cpu()), "non-deterministic residues"

    chunk, kept = stages.chunk, stages.dp.kept_u
    poly_e2e_all = None
    if not args.no_poly:
        del stages, dp
        torch.cuda.empty_cache()
        try:
            poly_e2e_all = poly_e2e(world, rank, cpu=not args.no_cpu_baseline)
        except Exception as exc:   # keep the measured line: report the failure in it
            poly_e2e_all = {"error": "%s: %s" % (type(exc).__name__, exc)}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    r = m.r
    W = (r ** 3 - r) // 3
    # the roofline's kernel: det_gj launches alone (device time from the events
    # around each launch); det_ms adds the finalize and row-table launches
    achieved = W * sel * args.steps / (kern_ms / 1e3)
    hbm, hbm_kind = measured_peaks()
    launch_nodes = chunk
    traffic = traffic_note = ncu_summary = None
    tpath = ROOT / "profiles" / "ncu" / "det_traffic_r02.json"
    if not tpath.exists():
        tpath = ROOT / "profiles" / "ncu" / "det_traffic_r01.json"
    if tpath.exists() and args.config == "c5":
        t = json.loads(tpath.read_text())
        traffic = t["dram_bytes_per_node"] * launch_nodes
        traffic_note = ("dram read+write bytes per launch of %d nodes, scaled from %s (%d-node launch)"
                        % (launch_nodes, t["source"], t["nodes_per_launch"]))
        ncu_summary = {k: t[k] for k in ("pipes_pct_of_peak", "issue_active_pct", "warp_instructions_per_det",
                                          "issue_model_cycles_per_det", "issue_model_cycles_frac",
                                          "dram_bytes_per_node", "source") if k in t}
    out = {
        "metric": "mod-p %dx%d dets/sec (%s)" % (r, r, args.config.upper()),
        "value": value, "unit": "dets/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32 (mod-p residues, p < 2^30)",
        "data": "synthetic (seeded %s generator, SURVEY.md 8(d))" % args.config.upper(),
        "config": describe(args.config, m, pl, ws_bytes),
        "matrices_n3_per_s": value * r ** 3,
        "computed_dets_per_step": sel, "grid_nodes_per_step": nodes,
        "grid_dets_per_s": grid_rate,
        "kept_u": kept,
        "e2e": {"value": e2e, "unit": "dets/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e_ms / args.steps,
                "scope": "per prime: the step's entry coefficients host->device, the prime's stages "
                         "(PrimeStages.step: evaluation, determinants, interpolation), its residue grid "
                         "device->host; whole polynomial determinants through the public run_report are "
                         "poly_e2e"},
        "roofline": {"bound": "int", "kernel": "det_gj_kernel<FusedSrc> (eval + elimination)",
                     "achieved": achieved / 1e9, "peak": peak_delayed / 1e9, "unit": "Gupd/s",
                     "frac": achieved / peak_delayed, "traffic": traffic, "traffic_note": traffic_note,
                     "hbm_achieved_gbs": (traffic / launch_nodes) * sel * args.steps / (kern_ms / 1e3) / 1e9
                     if traffic else None,
                     "peak_kind": "measured now: 9 MACs + one REDC, the trailing-update primitive "
                                  "(pdb_mulmod_peak variant 1)",
                     "imadwide_peak": peak_imadwide / 1e9,
                     "frac_vs_imadwide_ceiling": achieved / peak_imadwide,
                     "imadwide_note": "raw accumulating IMAD.WIDE stream measured now (variant 2): the integer "
                                      "multiplier's ceiling if every update were one bare MAC",
                     "kernel_ms_per_step": kern_ms / args.steps, "kernel_launches_per_step": kern_launches / args.steps,
                     "kernel_share": kern_ms / ms,
                     "kernel_timing": "CUDA events recorded by the library around every det_gj launch on its launch "
                                      "stream (pdb_kernel_timing), summed over the timed steps",
                     "det_ms_per_step": det_ms / args.steps, "det_share": det_ms / ms,
                     "frac_det_stage": W * sel * args.steps / (det_ms / 1e3) / peak_delayed,
                     "work_per_matrix": W, "hbm_peak_gbs": hbm, "hbm_peak_kind": hbm_kind,
                     "ncu": ncu_summary},
        "clocks": clocks,
        "gpu_launches": launches,
    }
    if not args.no_cpu_baseline and world == 1:
        out["cpu_baseline"] = cpu_sample(m, pl)
    out["poly_e2e"] = poly_e2e_all
    print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
