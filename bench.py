"""Benchmark of the modular-determinant hot path (BASELINE.json metric:
mod-p n x n dets/s and end-to-end time per polynomial determinant).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5|c3] [--impl ours|reference]

Workload (default `--config c5`, BASELINE.json configs[4], the largest
single-GPU configuration): 40x40 matrix, 3 variables, entry degree <= 4,
256^3 = 16.7 M evaluation nodes per prime, 23 primes.  One STEP = the hot path
for one prime: forward evaluation of all 1600 unique entries (partial NTT +
fused last-axis evaluation), 16.7 M determinants of 40x40 matrices mod p, and
the inverse NTT of the determinant grid.  Weak scaling: every rank runs one
prime per step (ranks take primes round-robin), so the units of a step are
N x 16.7 M determinants.

  value  dets/s over all ranks, inputs resident in HBM (working set 2.2 GB per
         prime >> 126 MB L2, so no flush is needed between steps)
  e2e    same metric with, every step, the H2D copy of the step's input
         coefficients from pinned host memory and the D2H copy of the step's
         residue tensor (16.7 M x u32) inside the timed region
  roofline  det kernel (eval + elimination, the dominant kernel): algorithmic
         elimination updates W(40) = (n^3 - n)/3 = 21320 per matrix / kernel time,
         against the measured peak of the delayed-reduction MAC primitive
  cpu_baseline  the oracle port (numpy restatement of the reference) timed on a
         bounded sample on this host (rank 0, N = 1), extrapolated per step
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
            "step": "one prime: forward evaluation + det at every node + inverse NTT",
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

def cpu_sample(m, pl, det_nodes=1024, threads=None):
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
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    m, pl = workload(args.config)
    vals = []
    for i in range(args.warmup + args.steps):
        res = cpu_sample(m, pl, det_nodes=512)
        if i >= args.warmup:
            vals.append(res)
    value = statistics.median(v["value"] for v in vals)
    base = vals[-1]
    out = {"impl": "reference", "metric": "mod-p %dx%d dets/sec (%s)" % (m.r, m.r, args.config.upper()),
           "value": value, "unit": "dets/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * statistics.median(v["step_seconds"] for v in vals),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
           "data": "synthetic (seeded C5 generator)", "config": describe(args.config, m, pl, working_set_bytes(m, pl)),
           "cpu_baseline": {"value": value, "unit": "dets/s", "cores": base["cores"], "kind": "port",
                            "sample": base["sample"]},
           "e2e": {"value": value, "unit": "dets/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def poly_e2e():
    """Second half of the BASELINE metric: end-to-end seconds per polynomial
    determinant through the public API (`run_report`: upload, all primes, CRT,
    Python-int result) for C3 (reference CPU: 161.5 s with 8 workers,
    SURVEY.md 6) and C5 (infeasible on the reference: ~11.5 days extrapolated)."""
    from paper_2010_12117_b200 import run_report, workloads

    res = []
    for name, make, reps in (("C3", workloads.c3, 3), ("C5", workloads.c5, 1)):
        m, cfg = make()
        best = None
        for _ in range(reps):
            t0 = time.perf_counter()
            result, timings, pl = run_report(m, cfg)
            wall = time.perf_counter() - t0
            if best is None or wall < best[0]:
                best = (wall, timings, pl)
        wall, timings, pl = best
        res.append({"config": name, "seconds": wall, "primes": pl.prime_count, "nodes": pl.node_count,
                    "stages_s": {"fft": timings.fft, "det": timings.det, "ifft": timings.ifft, "crt": timings.crt},
                    "reference_cpu_s": 161.5 if name == "C3" else None,
                    "reference_note": "SURVEY.md 6: reference run_report, 8 workers, dev container" if name == "C3"
                    else "reference infeasible (needs >= 215 GB RAM; ~11.5 days extrapolated, SURVEY.md 6)"})
    return res


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
    peak_shoup = native.mulmod_peak(pl.primes[0].p, 0)

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
        stages.determinants(pi)
        e1.record(stream)
        det_events.append((e0, e1))
        stages.interpolate(pi)
        t1 = torch.cuda.Event(enable_timing=True)
        t1.record(stream)
        step_events.append((t0, t1))
    barrier()
    clocks = sampler.stop()
    launches = native.launch_count() - launches0
    ms = sum(a.elapsed_time(b) for a, b in step_events)
    det_ms = sum(a.elapsed_time(b) for a, b in det_events)
    tmax = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms = float(tmax.item())
    nodes = pl.node_count
    value = world * nodes * args.steps / (ms / 1e3)

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
    e2e = world * nodes * args.steps / (e_ms / 1e3)

    # parity guard on the timed path: the last step's residues vs a fresh recompute
    check = host_out[(args.steps - 1) % 2].clone()
    stages.step(prime_of(args.steps - 1))
    torch.cuda.synchronize()
    assert torch.equal(check, stages.det.cpu()), "non-deterministic residues"

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    r = m.r
    W = (r ** 3 - r) // 3
    achieved = W * nodes * args.steps / (det_ms / 1e3)
    hbm, hbm_kind = measured_peaks()
    from paper_2010_12117_b200.executor import FUSED_CHUNK
    launch_nodes = min(nodes, FUSED_CHUNK)
    traffic = traffic_note = ncu_summary = None
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
        "e2e": {"value": e2e, "unit": "dets/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e_ms / args.steps},
        "roofline": {"bound": "int", "kernel": "det_gj_kernel<FusedSrc> (eval + elimination)",
                     "achieved": achieved / 1e9, "peak": peak_delayed / 1e9, "unit": "Gupd/s",
                     "frac": achieved / peak_delayed, "traffic": traffic, "traffic_note": traffic_note,
                     "hbm_achieved_gbs": (traffic / launch_nodes) * nodes * args.steps / (det_ms / 1e3) / 1e9
                     if traffic else None,
                     "peak_kind": "measured now: delayed 64-bit MAC + REDC primitive (pdb_mulmod_peak v1)",
                     "shoup_peak": peak_shoup / 1e9, "frac_vs_shoup_peak": achieved / peak_shoup,
                     "det_ms_per_step": det_ms / args.steps, "det_share": det_ms / ms,
                     "work_per_matrix": W, "hbm_peak_gbs": hbm, "hbm_peak_kind": hbm_kind,
                     "ncu": ncu_summary},
        "clocks": clocks,
        "gpu_launches": launches,
    }
    if not args.no_poly and world == 1:
        out["poly_e2e"] = poly_e2e()
    if not args.no_cpu_baseline and world == 1:
        out["cpu_baseline"] = cpu_sample(m, pl)
    print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
