"""End-to-end GPU executor -- drop-in for the reference's `run`, `run_report`,
`resume`, `resume_report` (pipeline.py:267-404).

Per prime (all on one device, residues never leave HBM between stages):

  FFT   reduce_scatter (coefficients -> padded residue grids)  +  pruned
        multivariate NTT (pdb_ntt_multi_u32)             [_fft_stage 349-371]
  DET   det mod p at every node (pdb_det_batch_u32)      [_det_stage 374-392]
  IFFT  inverse multivariate NTT, in place               [_ifft_stage 395-404]

then one CRT launch over the [P][nodes] residue block   [_execute 340-345].

Two FFT/DET modes, same results:
  * staged: every unique entry's grid is materialised ([k][nodes] u32), as in
    the reference; required when a workspace must receive p{i}/fft/e{j}
    artifacts, and used whenever the grids fit the memory budget.
  * fused:  entries are transformed along all axes but the last and each
    node's entries are evaluated inside the determinant kernel
    (pdb_eval_det_fused_u32), so the k x nodes grid never exists (config C5:
    1600 x 256^3 would be 107 GB per prime).  With a workspace, fused mode
    checkpoints at p{i}/ifft granularity only (a reference `_execute` resumes
    from such a workspace: it only consults has("p{i}/ifft")).

Unit names, notification order, skip-if-stored and the workspace header
logic follow the reference exactly, so kill/resume behaves identically.
Without a workspace, fused mode reports the reference's fine-grained units
too (p{i}/fft/e{j}, p{i}/det, p{i}/ifft, crt); with one, it reports and
persists the p{i}/ifft units only, because it never materialises the entry
grids or the determinant grid that the finer units name.
Stage timings are CUDA-event seconds of each stage's device work.
"""

from __future__ import annotations

import math
import os

import numpy as np

from . import native, shard
from .checkpoint import Workspace, digest_of
from .crt import device_lift, sharded_lift, wide_primes
from .errors import StaleWorkspaceError
from .layout import CoeffTensor, PolyMatrix, residue_dtype
from .planner import Plan, PipelineConfig, StageTimings, degree_bound, plan

INPUT_FILE = "input.json"
PLAN_FILE = "plan.json"

#: staged grids above this many bytes switch to fused evaluation (override: PDB_STAGED_LIMIT)
STAGED_LIMIT = int(os.environ.get("PDB_STAGED_LIMIT", str(8 << 30)))
#: nodes per determinant launch in fused mode
FUSED_CHUNK = 1 << 22


# -- public API -------------------------------------------------------------------------

def run(m: PolyMatrix, config: PipelineConfig = None, workspace=None) -> CoeffTensor:
    """Exact signed-integer determinant of a polynomial matrix."""
    return run_report(m, config, workspace)[0]


def run_report(m: PolyMatrix, config: PipelineConfig = None, workspace=None):
    """Like `run`, also returning (timings, plan)."""
    cfg = config or PipelineConfig()
    pl = plan(m, cfg)
    ws = None
    if workspace is not None:
        ws = Workspace(workspace)
        header = {"input_sha256": digest_of(m.to_dict()), "plan_sha256": pl.digest()}
        if ws.exists():
            if ws.open() != header:
                raise StaleWorkspaceError(
                    "stale workspace: manifest belongs to a different input or plan")
        else:
            ws.write_named(INPUT_FILE, m.to_dict())   # named files first: the manifest
            ws.write_named(PLAN_FILE, pl.to_dict())   # is the commit point
            ws.create(header)
    result, timings = execute(m, pl, cfg, ws)
    return result, timings, pl


def resume(workspace, config: PipelineConfig = None) -> CoeffTensor:
    """Continue (or just reload) a checkpointed run."""
    return resume_report(workspace, config)[0]


def resume_report(workspace, config: PipelineConfig = None):
    cfg = config or PipelineConfig()
    ws = Workspace(workspace)
    header = ws.open()
    ws.verify()
    m = PolyMatrix.from_dict(ws.read_named(INPUT_FILE))
    pl = Plan.from_dict(ws.read_named(PLAN_FILE))
    if (header.get("input_sha256") != digest_of(m.to_dict())
            or header.get("plan_sha256") != pl.digest()):
        raise StaleWorkspaceError("stale workspace: stored input or plan was altered")
    result, timings = execute(m, pl, cfg, ws)
    return result, timings, pl


# -- host preparation -----------------------------------------------------------------------

def _limbs_of(values):
    """Signed Python ints -> (magnitude limbs [n][L] u32, negative flags, L)."""
    vals = list(values)
    if not vals:
        return np.zeros((0, 1), dtype=np.uint32), np.zeros(0, dtype=np.uint8), 1
    top = max(abs(v) for v in vals)
    L = max(1, (top.bit_length() + 31) // 32)
    neg = np.fromiter((v < 0 for v in vals), dtype=np.uint8, count=len(vals))
    if L <= 2:
        mag = np.array([abs(v) for v in vals], dtype=np.uint64)
        limbs = np.stack([(mag & 0xFFFFFFFF).astype(np.uint32), (mag >> 32).astype(np.uint32)], axis=1)[:, :L]
    else:
        raw = b"".join(abs(v).to_bytes(4 * L, "little") for v in vals)
        limbs = np.frombuffer(raw, dtype="<u4").reshape(len(vals), L)
    return np.ascontiguousarray(limbs, dtype=np.uint32), neg, L


class DevicePlan:
    """Everything uploaded once per run: coefficient limbs, scatter positions
    for both layouts, entry ids; plus the mode decision."""

    def __init__(self, m: PolyMatrix, pl: Plan, device, staged: bool):
        torch = native._torch()
        self.m, self.pl, self.device = m, pl, device
        self.shape = tuple(pl.shape)
        self.vn = len(self.shape)
        self.nodes = pl.node_count
        self.k = m.k
        # primes >= 2^31 (reference int64/object dtype paths): u64 residues and kernels,
        # staged layout (the fused det kernel is the u32 throughput path)
        self.wide = wide_primes([s.p for s in pl.primes])
        self.word = native.word_dtype(self.wide)
        self.staged = staged or self.vn == 0 or self.wide
        for t in m.unique_entries:
            # the reference pads every entry to the plan shape (pipeline.py:361) and
            # pad_to refuses to shrink (tensor.py:219-220); a larger entry box would
            # otherwise walk into the neighbouring entry's lines
            if len(t.shape) != self.vn or any(a > b for a, b in zip(t.shape, self.shape)):
                raise ValueError("cannot shrink %s to %s" % (tuple(t.shape), self.shape))
        if not self.staged:
            self.E = max(t.shape[-1] for t in m.unique_entries)
            self.outer = self.nodes // self.shape[-1]
        prep = _vector_terms(m, self.shape, self.nodes, self.staged, self.E if not self.staged else 0)
        if prep is None:
            prep = _python_terms(m, self.shape, self.nodes, self.staged, self.E if not self.staged else 0)
        mag, neg, L, pos = prep
        self.count = len(neg)
        # coefficients are entry-major: entry e owns [entry_starts[e], entry_starts[e+1])
        owner = pos // self.nodes if self.staged else pos % self.k
        self.entry_starts = np.searchsorted(owner, np.arange(self.k + 1)).tolist()
        self.L = L
        self.mag = torch.from_numpy(mag.view(np.int32).copy()).to(device) if self.count else \
            torch.zeros(1, dtype=torch.int32, device=device)
        self.neg = torch.from_numpy(neg.copy()).to(device) if self.count else \
            torch.zeros(1, dtype=torch.uint8, device=device)
        self.pos = torch.from_numpy(np.ascontiguousarray(pos, dtype=np.int64)).to(device) if self.count else \
            torch.zeros(1, dtype=torch.int64, device=device)
        self.ids = torch.tensor(list(m.entry_ids), dtype=torch.int32, device=device)
        # per-axis coefficient extents (for NTT pruning): largest exponent + 1
        self.ext = [max(t.shape[a] for t in m.unique_entries) for a in range(self.vn)]
        # pruned node set (csrc/expand.cu): determinants only where the degree
        # bound needs them, the rest of the grid is extended exactly
        self.kept_u = kept_u(self.shape, degree_bound(m)) \
            if PRUNE and not self.wide else [0] * self.vn
        self.nmap = native.node_map(self.shape, self.kept_u) if self.vn else None
        self.sel = native.node_map_size(self.nmap) if self.nmap is not None else self.nodes
        self.klen = [8 * u if u else n for n, u in zip(self.shape, self.kept_u)]
        # fused runs with every axis pruned interpolate the coefficients straight
        # from the kept nodes (pdb_grid_interpolate_u32): no full determinant grid,
        # no grid extension, no inverse NTT; the box is the 8 U coefficients per
        # axis those nodes determine (zero beyond the degree bound)
        self.direct = (DIRECT and not self.staged and self.nmap is not None and self.vn > 0
                       and all(self.kept_u))
        self.box = [8 * u for u in self.kept_u] if self.direct else None

    def buffer_words(self) -> int:
        return self.k * self.nodes if self.staged else self.k * self.outer * self.E


#: determinants only at the kept nodes of the degree bound (False: every node, as the reference)
PRUNE = os.environ.get("PDB_NO_PRUNE", "") == ""
#: fused + pruned: the forward passes evaluate only the kept nodes of the leading axes
FORWARD_KEPT = os.environ.get("PDB_NO_FORWARD_KEPT", "") == ""
#: fused + fully pruned: coefficients interpolated straight from the kept nodes
DIRECT = os.environ.get("PDB_NO_DIRECT", "") == ""


def kept_u(shape, degrees, even_last: bool = False) -> list:
    """Per axis, the u-count U of the kept nodes {u + (N/8) v : u < U, v < 8}
    (0 = every node): det(M) has degree <= D_a in variable a, so
    U = floor(D_a / 8) + 1 suffices.  even_last rounds the last axis's U up to
    even (no caller needs it since the fused kernel's u-pairs may straddle
    rows; kept for experiments).  Axes shorter
    than 16 or with 8 U >= N keep every node."""
    out = []
    for a, (n, d) in enumerate(zip(shape, degrees)):
        u = min(int(d), n - 1) // 8 + 1
        if even_last and a == len(shape) - 1:
            u += u & 1
        out.append(u if n >= 16 and 8 * u < n else 0)
    return out


def _python_terms(m: PolyMatrix, shape, nodes, staged, E):
    """(limbs, negative flags, L, scatter positions) of every nonzero coefficient:
    staged layout e*nodes + flat(exps); fused layout [outer][E][k] (entries
    innermost, coalesced fills in the det kernel)."""
    entries, coeffs = [], []
    for e, t in enumerate(m.unique_entries):
        for exps, c in t._nonzero():
            entries.append((e, exps))
            coeffs.append(c)
    mag, neg, L = _limbs_of(coeffs)
    if staged:
        pos = [e * nodes + _flat(exps, shape) for e, exps in entries]
    else:
        pos = [(_flat(exps[:-1], shape[:-1]) * E + exps[-1]) * m.k + e for e, exps in entries]
    return mag, neg, L, np.array(pos, dtype=np.int64).reshape(-1)


def _vector_terms(m: PolyMatrix, shape, nodes, staged, E):
    """_python_terms in numpy, same order, when every unique entry has the same
    coefficient box and all coefficients fit in int64 (None otherwise)."""
    shapes = {tuple(t.shape) for t in m.unique_entries}
    if len(shapes) != 1 or not shape:
        return None
    box = shapes.pop()
    if len(box) != len(shape):
        return None
    try:
        C = np.array([t.coeffs for t in m.unique_entries], dtype=np.int64).reshape(m.k, -1)
    except (OverflowError, ValueError, TypeError):
        return None
    e_idx, off = np.nonzero(C)            # entry-major, then row-major offset: the _nonzero order
    vals = C[e_idx, off]
    if vals.size and vals.min() == np.iinfo(np.int64).min:
        return None
    neg = (vals < 0).astype(np.uint8)
    mag = np.abs(vals).astype(np.uint64)
    top = int(mag.max()) if mag.size else 0
    L = max(1, (top.bit_length() + 31) // 32)
    limbs = np.stack([(mag & 0xFFFFFFFF).astype(np.uint32), (mag >> np.uint64(32)).astype(np.uint32)], axis=1)[:, :L]
    exps = np.unravel_index(off, box)
    if staged:
        flat = np.zeros(off.shape, dtype=np.int64)
        for a, n in enumerate(shape):
            flat = flat * n + exps[a]
        pos = e_idx.astype(np.int64) * nodes + flat
    else:
        flat = np.zeros(off.shape, dtype=np.int64)
        for a, n in enumerate(shape[:-1]):
            flat = flat * n + exps[a]
        pos = (flat * E + exps[-1]) * m.k + e_idx
    return np.ascontiguousarray(limbs, dtype=np.uint32), neg, L, pos.astype(np.int64)


def _flat(exps, shape):
    pos = 0
    for e, n in zip(exps, shape):
        pos = pos * n + e
    return pos


#: None = automatic; "staged" / "fused" force a mode (tests, benchmarks)
FORCE_MODE = None


def choose_staged(m: PolyMatrix, pl: Plan, ws) -> bool:
    if len(pl.shape) == 0:
        return True
    if FORCE_MODE is not None and ws is None:
        return FORCE_MODE == "staged"
    wide = wide_primes([s.p for s in pl.primes])
    grid_bytes = (8 if wide else 4) * m.k * pl.node_count
    if wide:
        # the u64 path has no fused kernel: it is staged or nothing
        if grid_bytes > STAGED_LIMIT:
            raise ValueError("wide-prime plan needs %.1f GB of staged u64 grids (limit %.1f GB, "
                             "PDB_STAGED_LIMIT); primes >= 2^31 have no fused path"
                             % (grid_bytes / 1e9, STAGED_LIMIT / 1e9))
        return True
    if ws is not None and grid_bytes <= STAGED_LIMIT:
        return True
    return grid_bytes <= STAGED_LIMIT and pl.r <= 8 or grid_bytes <= STAGED_LIMIT // 4


# -- the executor ------------------------------------------------------------------------

class _Timer:
    def __init__(self, torch, stream):
        self.torch, self.stream = torch, stream
        self.marks = []

    def mark(self):
        ev = self.torch.cuda.Event(enable_timing=True)
        ev.record(self.stream)
        self.marks.append(ev)
        return ev


def execute(m: PolyMatrix, pl: Plan, cfg: PipelineConfig, ws):
    """Run the per-prime stages and the CRT (reference `_execute`, pipeline.py:323-346).

    Under torch.distributed with world size G > 1 (one process per GPU), whole
    rounds of G primes are prime-sharded (rank g computes primes g, g+G, ...;
    the residue blocks are all-gathered before the CRT) and the remaining
    P mod G primes are slab-sharded across all ranks (shard.py); every rank
    returns the same result.
    """
    timings = StageTimings()
    if ws is not None and ws.has("crt"):
        return _tensor_from_payload(ws.load_json("crt")), timings
    torch = native._torch()
    rank, size = shard.world()
    if size > 1 and ws is not None:
        raise ValueError("workspace checkpointing runs on a single device (world size %d)" % size)
    device = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream()
    staged = choose_staged(m, pl, ws)
    dp = DevicePlan(m, pl, device, staged)
    nodes = dp.nodes
    P = pl.prime_count
    whole, slab_primes = shard.split_primes(P, size) if dp.vn else (P, [])
    mine = shard.my_primes(whole, rank, size)
    # direct interpolation writes only the coefficient box: the rest stays zero
    residues = (torch.zeros if dp.direct else torch.empty)((len(mine), nodes), dtype=dp.word, device=device)
    work = torch.empty(dp.buffer_words() or 1, dtype=dp.word, device=device)
    det_chunk = det_chunk_size(dp)
    det_buf = torch.empty(dp.sel, dtype=dp.word, device=device)
    interp = torch.empty(dp.sel, dtype=dp.word, device=device) if dp.direct else None
    scratch = native.scratch_tensor(native.det_scratch_bytes(pl.r, det_chunk, dp.wide), device)
    events = []
    for row, pi in enumerate(mine):
        spec = pl.primes[pi]
        unit = "p%d/ifft" % pi
        if ws is not None and ws.has(unit):
            residues[row].copy_(native.to_device_words(_load_grid(ws, unit, pl), dp.wide))
            continue
        ctx = native.prime_context(spec, device.index, dp.wide)
        t0 = _Timer(torch, stream).mark()
        _fft_stage(dp, ctx, work, ws, pi, cfg)
        t1 = _Timer(torch, stream).mark()
        if dp.direct:
            _det_range(dp, ctx, work, det_buf, scratch, det_chunk, 0, dp.sel)
            if ws is None:
                cfg._notify("p%d/det" % pi)
            t2 = _Timer(torch, stream).mark()
            native.grid_interpolate(ctx, det_buf, interp, residues[row], dp.nmap, dp.box)
        else:
            _det_stage(dp, ctx, work, det_buf, scratch, det_chunk, ws, pi, cfg, residues[row])
            t2 = _Timer(torch, stream).mark()
            native.ntt_multi(ctx, residues[row], 1, dp.shape, None, range(dp.vn), True)
        t3 = _Timer(torch, stream).mark()
        events.append((t0, t1, t2, t3))
        if ws is not None:
            ws.store_residues(unit, native.to_host_words(residues[row], dp.wide), pl.shape)
        cfg._notify(unit)
    primes = [s.p for s in pl.primes]
    if size > 1 and not dp.wide:
        # sharded CRT: every prime's residues of my coefficient range (all-to-all),
        # lifted here; the compact results are all-gathered (crt.sharded_lift)
        lo, hi = shard.coefficient_range(nodes, rank, size)
        block = shard.exchange_residues(residues, whole, rank, size) if whole else None
        if slab_primes:
            # partial rows of every slab prime, summed over the ranks straight into
            # this rank's coefficient range (the only exchange besides the all-to-all)
            slab_rows = _slab_primes(dp, slab_primes, work, det_buf, scratch, det_chunk, rank, size, cfg, events,
                                     torch, stream, partial=True)
            slab_block = shard.reduce_scatter_rows(slab_rows, [primes[pi] for pi in slab_primes], rank, size)
            block = torch.cat([block, slab_block]) if whole else slab_block
        del residues
        t4 = _Timer(torch, stream).mark()
        coeffs = sharded_lift(block, primes, nodes, lo, rank, size)
        t5 = _Timer(torch, stream).mark()
    else:
        if size > 1:   # u64 residues: gather every row, lift on every rank
            residues = shard.gather_residues(residues, whole, rank, size)
            if slab_primes:
                slab_rows = _slab_primes(dp, slab_primes, work, det_buf, scratch, det_chunk, rank, size, cfg,
                                         events, torch, stream)
                residues = torch.cat([residues, slab_rows]) if whole else slab_rows
        t4 = _Timer(torch, stream).mark()
        coeffs = device_lift(residues, primes, nodes, nodes)
        t5 = _Timer(torch, stream).mark()
    torch.cuda.synchronize()
    for t0, t1, t2, t3 in events:
        timings.fft += t0.elapsed_time(t1) / 1e3
        timings.det += t1.elapsed_time(t2) / 1e3
        timings.ifft += t2.elapsed_time(t3) / 1e3
    timings.crt += t4.elapsed_time(t5) / 1e3
    result = CoeffTensor(tuple(pl.shape), tuple(coeffs), tuple(pl.variables))
    if ws is not None:
        ws.store_json("crt", _payload_from_tensor(result))
    cfg._notify("crt")
    return result, timings


def _slab_primes(dp: DevicePlan, primes, work, det_buf, scratch, chunk, rank, size, cfg, events, torch, stream,
                 partial: bool = False):
    """Slab-sharded primes (shard.py): every rank evaluates the entries and
    computes the determinants of its slab of the slowest axis.  partial: the
    rank interpolates its slab alone (zero elsewhere) and returns partial
    coefficient rows for shard.reduce_scatter_rows; otherwise the slabs are
    all-gathered and every rank interpolates the full grid (u64 path)."""
    pl = dp.pl
    k0 = dp.klen[0]           # slabs of the kept nodes' slowest axis
    inner = dp.sel // k0
    lo, hi = shard.my_slab(k0, rank, size)
    rows = (torch.zeros if dp.direct else torch.empty)((len(primes), dp.nodes), dtype=dp.word,
                                                        device=det_buf.device)
    for j, pi in enumerate(primes):
        ctx = native.prime_context(pl.primes[pi], det_buf.device.index, dp.wide)
        t0 = _Timer(torch, stream).mark()
        _fft_stage(dp, ctx, work, None, pi, cfg)
        t1 = _Timer(torch, stream).mark()
        _det_range(dp, ctx, work, det_buf, scratch, chunk, lo * inner, (hi - lo) * inner)
        if partial:
            full = det_buf[: dp.sel]
            full[: lo * inner].zero_()
            full[hi * inner:].zero_()
        else:
            full = shard.gather_slabs(det_buf[lo * inner: hi * inner], k0, inner, rank, size)
        if dp.direct:
            t2 = _Timer(torch, stream).mark()
            native.grid_interpolate(ctx, full, torch.empty_like(full), rows[j], dp.nmap, dp.box)
        else:
            _expand(dp, ctx, full, rows[j])
            t2 = _Timer(torch, stream).mark()
            native.ntt_multi(ctx, rows[j], 1, dp.shape, None, range(dp.vn), True)
        t3 = _Timer(torch, stream).mark()
        events.append((t0, t1, t2, t3))
        cfg._notify("p%d/ifft" % pi)
    return rows


def det_chunk_size(dp: DevicePlan) -> int:
    """Nodes per determinant launch: all of them staged; in fused mode chunks of
    ~FUSED_CHUNK made of whole kept last-axis rows (the DFT-8 fill's unit)."""
    if dp.staged:
        return max(dp.sel, 1)
    row = dp.klen[-1]
    return max(row, min(dp.sel, FUSED_CHUNK) // row * row)


def _det_range(dp: DevicePlan, ctx, work, det_buf, scratch, chunk, node_lo: int, count: int):
    """Determinants of the kept nodes [node_lo, node_lo + count) (compact order of
    dp.nmap; every node in natural order without pruning) into det_buf."""
    pl = dp.pl
    if count == 0:
        return
    if dp.staged:
        out = det_buf[node_lo:node_lo + count]
        if dp.nmap is None:
            native.det_batch(ctx, work, dp.nodes, dp.ids, pl.r, node_lo, count, out, scratch)
        else:
            native.det_batch_map(ctx, work, dp.nodes, dp.ids, pl.r, dp.nmap, node_lo, count, out, scratch)
        return
    n_last = dp.shape[-1]
    for lo in range(node_lo, node_lo + count, chunk):
        cnt = min(chunk, node_lo + count - lo)
        if dp.nmap is None:
            native.eval_det_fused(ctx, work, dp.outer, dp.E, dp.k, n_last, dp.ids, pl.r, lo, cnt,
                                  det_buf[lo:lo + cnt], scratch)
        else:
            native.eval_det_fused_map(ctx, work, dp.outer, dp.E, dp.k, n_last, dp.ids, pl.r, dp.nmap, lo, cnt,
                                      det_buf[lo:lo + cnt], scratch)


def _expand(dp: DevicePlan, ctx, compact, grid):
    """Determinants at the kept nodes -> the full determinant grid (csrc/expand.cu)."""
    if dp.nmap is None:
        grid.copy_(compact[:dp.nodes])
    else:
        native.grid_expand(ctx, compact, grid, dp.nmap)


def _sparse_axes(shape, ext) -> bool:
    """True when ntt.cu evaluates every one of these forward axes with the
    sparse kernel (<= 8 nonzero rows, length >= 16; or length 1), which reads
    only the coefficient box and writes every output position: then only the
    box needs zeroing before the scatter, not the whole grid buffer."""
    if os.environ.get("PDB_NTT_DENSE"):
        return False
    return all(n == 1 or (1 <= e <= 8 and n >= 16) for n, e in zip(shape, ext))


def _sparse_leading_axes(dp: DevicePlan) -> bool:
    return _sparse_axes(dp.shape[:-1], dp.ext[:-1])


def _fft_stage(dp: DevicePlan, ctx, work, ws, pi, cfg):
    """Entry grids of one prime: reduce + scatter + pruned NTT (staged or partial)."""
    m, pl = dp.m, dp.pl
    if not dp.staged:
        dims = dp.shape[:-1] + (dp.E, dp.k)
        ext = dp.ext[:-1] + [dp.E, dp.k]
        if _sparse_leading_axes(dp):
            # every leading axis is evaluated by the sparse kernel, which reads only
            # the coefficient box and writes every output: zero just the box
            box = work[: math.prod(dims)].view(dims)[tuple(slice(0, e) for e in dp.ext[:-1])]
            box.zero_()
        else:
            work.zero_()
        native.reduce_scatter(ctx, dp.mag, dp.neg, dp.pos, dp.count, dp.L, work)
        if dp.nmap is not None and FORWARD_KEPT and _sparse_leading_axes(dp):
            # pruned node set: evaluate the leading axes at their kept nodes only
            native.ntt_forward_kept(ctx, work, 1, dims, ext, list(dp.kept_u[:-1]) + [0, 0], range(dp.vn - 1))
        else:
            native.ntt_multi(ctx, work, 1, dims, ext, range(dp.vn - 1), False)
        if ws is None:
            # progress only: fused mode stores no fft/det artifacts, so with a
            # workspace it reports (and checkpoints) p{i}/ifft units alone
            for eid in range(dp.k):
                cfg._notify("p%d/fft/e%d" % (pi, eid))
        return
    todo = []
    for eid in range(dp.k):
        unit = "p%d/fft/e%d" % (pi, eid)
        if ws is not None and ws.has(unit):
            grid = _load_grid(ws, unit, pl)
            work[eid * dp.nodes:(eid + 1) * dp.nodes].copy_(native.to_device_words(grid, dp.wide))
        else:
            todo.append(eid)
    if not todo:
        return
    if len(todo) < dp.k:
        # keep the stored grids: scatter and transform only the todo entries, in
        # place (each entry's coefficients are one contiguous run of the upload)
        for eid in todo:
            sl = work[eid * dp.nodes:(eid + 1) * dp.nodes]
            sl.zero_()
            lo, hi = dp.entry_starts[eid], dp.entry_starts[eid + 1]
            if hi > lo:
                native.reduce_scatter(ctx, dp.mag[lo:], dp.neg[lo:], dp.pos[lo:], hi - lo, dp.L, work)
            native.ntt_multi(ctx, sl, 1, dp.shape, dp.ext, range(dp.vn), False)
    else:
        if dp.vn and not dp.wide and _sparse_axes(dp.shape, dp.ext):   # (the u64 NTT is dense)
            box = work[: dp.k * dp.nodes].view((dp.k,) + dp.shape)[(slice(None),) + tuple(slice(0, e) for e in dp.ext)]
            box.zero_()
        else:
            work.zero_()
        native.reduce_scatter(ctx, dp.mag, dp.neg, dp.pos, dp.count, dp.L, work)
        native.ntt_multi(ctx, work, dp.k, dp.shape, dp.ext, range(dp.vn), False)
    for eid in todo:
        unit = "p%d/fft/e%d" % (pi, eid)
        if ws is not None:
            ws.store_residues(unit, native.to_host_words(work[eid * dp.nodes:(eid + 1) * dp.nodes], dp.wide),
                              pl.shape)
        cfg._notify(unit)


def _det_stage(dp: DevicePlan, ctx, work, det_buf, scratch, chunk, ws, pi, cfg, out):
    """The full determinant grid of one prime into `out` ([nodes])."""
    pl = dp.pl
    unit = "p%d/det" % pi
    if ws is not None and ws.has(unit):
        out.copy_(native.to_device_words(_load_grid(ws, unit, pl), dp.wide))
        return
    if dp.nmap is None:
        _det_range(dp, ctx, work, out, scratch, chunk, 0, dp.nodes)
    else:
        _det_range(dp, ctx, work, det_buf, scratch, chunk, 0, dp.sel)
        _expand(dp, ctx, det_buf, out)
    if dp.staged:
        if ws is not None:
            ws.store_residues(unit, native.to_host_words(out, dp.wide), pl.shape)
        cfg._notify(unit)
    elif ws is None:   # fused mode: progress only (no det artifact; see _fft_stage)
        cfg._notify(unit)


def _load_grid(ws, unit, pl):
    values, shape = ws.load_array(unit)
    if tuple(shape) != tuple(pl.shape):
        raise StaleWorkspaceError("stale workspace: artifact shape %s != %s" % (shape, pl.shape))
    return values


def _payload_from_tensor(t: CoeffTensor) -> dict:
    return {"variables": list(t.axis_vars), "shape": list(t.shape), "coeffs": list(t.coeffs)}


def _tensor_from_payload(payload) -> CoeffTensor:
    return CoeffTensor(tuple(payload["shape"]), tuple(int(c) for c in payload["coeffs"]),
                       tuple(payload["variables"]))


# -- stage-level access (tests, benchmarks) ---------------------------------------------

class PrimeStages:
    """Device buffers + one prime's FWD/DET/INV, reusable across primes and steps.

    `forward(pi)` builds the entry grids (staged) or the partial transform
    (fused); `determinants(pi)` fills `det` for every node; `interpolate(pi)`
    turns `det` into the residue tensor in place.  Used by bench.py to time
    exactly the per-prime hot path and by the tests to replay stages.
    """

    def __init__(self, m: PolyMatrix, pl: Plan, staged: bool):
        torch = native._torch()
        self.torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.m, self.pl = m, pl
        self.dp = DevicePlan(m, pl, self.device, staged)
        dp = self.dp
        self.work = torch.empty(dp.buffer_words() or 1, dtype=dp.word, device=self.device)
        self.chunk = det_chunk_size(dp)
        # direct mode: `det` receives the coefficient box only (zero elsewhere, once)
        self.det = (torch.zeros if dp.direct else torch.empty)(dp.nodes, dtype=dp.word, device=self.device)
        self.compact = torch.empty(dp.sel, dtype=dp.word, device=self.device)
        self.interp = torch.empty(dp.sel, dtype=dp.word, device=self.device) if dp.direct else None
        self.scratch = native.scratch_tensor(native.det_scratch_bytes(pl.r, self.chunk, dp.wide), self.device)
        self._cfg = PipelineConfig()
        self._full_grid = False

    def ctx(self, pi):
        return native.prime_context(self.pl.primes[pi], self.device.index, self.dp.wide)

    def forward(self, pi):
        _fft_stage(self.dp, self.ctx(pi), self.work, None, pi, self._cfg)

    def determinants(self, pi):
        self._full_grid = True
        _det_stage(self.dp, self.ctx(pi), self.work, self.compact, self.scratch, self.chunk, None, pi, self._cfg,
                   self.det)

    def det_kernels(self, pi):
        """The determinant launches alone: every kept node (dp.sel of them) into
        `compact` (pruned) or `det` (unpruned)."""
        dp = self.dp
        out = self.det if dp.nmap is None else self.compact
        _det_range(dp, self.ctx(pi), self.work, out, self.scratch, self.chunk, 0, dp.sel)

    def expand(self, pi):
        """Kept-node determinants -> the full grid in `det` (no-op unpruned)."""
        self._full_grid = True
        if self.dp.nmap is not None:
            _expand(self.dp, self.ctx(pi), self.compact, self.det)

    def interpolate(self, pi):
        native.ntt_multi(self.ctx(pi), self.det, 1, self.dp.shape, None, range(self.dp.vn), True)

    def interpolate_direct(self, pi):
        """Kept-node determinants in `compact` -> the residue tensor in `det`
        (direct mode: straight from the kept nodes; `compact` is consumed)."""
        if self._full_grid:   # `det` last held a full grid: clear outside the box
            self.det.zero_()
            self._full_grid = False
        native.grid_interpolate(self.ctx(pi), self.compact, self.interp, self.det, self.dp.nmap, self.dp.box)

    def finish(self, pi):
        """After det_kernels: the residue tensor in `det` (direct interpolation, or
        grid extension + inverse NTT)."""
        if self.dp.direct:
            self.interpolate_direct(pi)
        else:
            self.expand(pi)
            self.interpolate(pi)

    def step(self, pi):
        self.forward(pi)
        if self.dp.direct:
            self.det_kernels(pi)
            self.interpolate_direct(pi)
        else:
            self.determinants(pi)
            self.interpolate(pi)
