"""Multi-GPU sharding of the (prime x node) work.

One process per GPU under torch.distributed (NCCL over NVLink on the GPU,
gloo in the CPU tests).  Two partitions, combined:

* prime-sharded: the first G*floor(P/G) primes go round-robin (rank g takes
  primes g, g+G, ...) and each rank runs FWD -> DET -> IFFT for them with no
  communication; their residue rows are all-gathered once before the CRT;
* slab-sharded: the remaining P mod G primes (all of them when P < G, e.g.
  a one-prime plan on 8 GPUs) are split by the slowest grid axis: rank g
  computes the determinants of the nodes with a_0 in its slab (a contiguous
  node range) and interpolates that slab alone, zero elsewhere -- the
  interpolation (inverse NTT, or the kept-node interpolation) is linear, so
  the ranks' partial coefficient rows sum to the prime's residues.  The sum
  is a reduce-scatter over the CRT's coefficient ranges (`reduce_scatter_rows`),
  so nothing crosses GPUs before the final exchange (partial
  inverse DFT + reduce).  The u64 path (p >= 2^31, where G partial sums would
  overflow 64 bits) all-gathers the determinant slabs instead (`gather_slabs`).

The CRT is sharded too (the reference does it once over every coefficient,
crt.py:94-130): an all-to-all leaves rank g with every prime's residues of
its coefficient range [lo_g, hi_g), it lifts those (nonzero compaction + the
mixed-radix kernel), and the compact limb rows of all ranks are all-gathered
so that every rank returns the same Python-int result.

Output is bit-identical for any device count because every residue is a pure
function of the prime and node (test_multiproc.py, test_gpu_parity.py).
"""

from __future__ import annotations


def world():
    """(rank, world_size) of the default process group, or (0, 1)."""
    try:
        import torch.distributed as dist
    except ImportError:  # pragma: no cover
        return 0, 1
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def my_primes(prime_count: int, rank: int, size: int):
    """Round-robin assignment: load balance (P/G)/ceil(P/G) (23 primes on 8 GPUs: 96 %)."""
    return list(range(rank, prime_count, size))


def split_primes(prime_count: int, size: int):
    """(prime-sharded count, slab-sharded prime indices): whole rounds of G primes
    go round-robin, the remainder is split across all ranks by grid slab."""
    whole = (prime_count // size) * size if size > 1 else prime_count
    return whole, list(range(whole, prime_count))


def my_slab(n0: int, rank: int, size: int):
    """[lo, hi) of the slowest axis owned by `rank` (sizes differ by at most 1)."""
    base, extra = divmod(n0, size)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_slabs(local, n0: int, inner: int, rank: int, size: int):
    """All-gather every rank's slab ([hi-lo][inner] rows of the slowest axis)
    into the full [n0 * inner] grid on every rank."""
    import torch
    import torch.distributed as dist

    width = -(-n0 // size) * inner
    buf = local.new_zeros(width)
    buf[: local.numel()] = local.reshape(-1)
    full = local.new_empty(size * width)
    dist.all_gather_into_tensor(full, buf)
    parts = []
    for g in range(size):
        lo, hi = my_slab(n0, g, size)
        parts.append(full[g * width: g * width + (hi - lo) * inner])
    return torch.cat(parts)


def gather_residues(local, prime_count: int, rank: int, size: int):
    """All-gather each rank's [ceil(P/G)][nodes] block of round-robin primes;
    return the [P][nodes] tensor in prime order (every rank receives it, so
    each can run the CRT or the caller can keep rank 0's)."""
    import torch
    import torch.distributed as dist

    rows = -(-prime_count // size)
    nodes = local.shape[1]
    if local.shape[0] != rows:
        pad = local.new_zeros((rows, nodes))
        pad[: local.shape[0]] = local
        local = pad
    full = local.new_empty((size * rows, nodes))
    dist.all_gather_into_tensor(full, local.contiguous())
    order = torch.empty(prime_count, dtype=torch.long)
    for g in range(size):
        for j, pi in enumerate(my_primes(prime_count, g, size)):
            order[pi] = g * rows + j
    return full[order.to(full.device)]


def coefficient_range(n: int, rank: int, size: int):
    """[lo, hi) of the n coefficient positions whose CRT `rank` owns."""
    base, extra = divmod(n, size)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _backend():
    import torch.distributed as dist
    return dist.get_backend()


def exchange_residues(local, prime_count: int, rank: int, size: int):
    """All-to-all of the round-robin residue rows: `local` is this rank's
    [prime_count / size][n] block (primes rank, rank + size, ...); returns the
    [prime_count][hi - lo] residues (prime order) of this rank's coefficient
    range.  NCCL: one all_to_all_single; other backends (gloo in the tests):
    an all-gather of the ranges, same result."""
    import torch
    import torch.distributed as dist

    rows, n = local.shape
    width = -(-n // size)
    lo, hi = coefficient_range(n, rank, size)
    send = local.new_zeros((size, rows, width))
    for g in range(size):
        glo, ghi = coefficient_range(n, g, size)
        send[g, :, : ghi - glo] = local[:, glo:ghi]
    if _backend() == "nccl":
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv.view(-1), send.view(-1))
    else:
        full = local.new_empty((size, size, rows, width))
        dist.all_gather_into_tensor(full.view(-1), send.view(-1))
        recv = full[:, rank]
    out = local.new_empty((prime_count, hi - lo))
    for g in range(size):
        for j, pi in enumerate(my_primes(prime_count, g, size)):
            out[pi] = recv[g, j, : hi - lo]
    return out


def reduce_scatter_rows(partial, moduli, rank: int, size: int):
    """Sum of every rank's partial rows [S][n] (residues in [0, p_s)), reduced
    mod p_s, restricted to this rank's coefficient range: [S][hi - lo].  The
    sum of G values < 2^31 is exact in int64.  NCCL: one reduce_scatter_tensor;
    other backends (gloo in the tests): an all-reduce, then the range."""
    import torch
    import torch.distributed as dist

    rows, n = partial.shape
    lo, hi = coefficient_range(n, rank, size)
    mod = torch.tensor(list(moduli), dtype=torch.int64, device=partial.device).view(-1, 1)
    wide = partial.to(torch.int64)
    if _backend() == "nccl":
        width = -(-n // size)
        send = wide.new_zeros((size, rows, width))
        for g in range(size):
            glo, ghi = coefficient_range(n, g, size)
            send[g, :, : ghi - glo] = wide[:, glo:ghi]
        recv = wide.new_empty((rows, width))
        dist.reduce_scatter_tensor(recv.view(-1), send.view(-1))
        out = recv[:, : hi - lo]
    else:
        dist.all_reduce(wide)
        out = wide[:, lo:hi]
    return (out % mod).to(partial.dtype)


def gather_compact(count: int, limbs, idx, neg, width: int, rank: int, size: int):
    """All-gather every rank's compact CRT output (count rows of `width` limbs,
    global positions, sign bytes) -> the concatenation in rank order (ascending
    positions, since the ranges are ascending), on every rank."""
    import torch
    import torch.distributed as dist

    dev = limbs.device
    counts = torch.tensor([count], dtype=torch.int64, device=dev)
    allc = torch.empty(size, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(allc, counts)
    allc = allc.tolist()
    mx = max(max(allc), 1)
    pl = limbs.new_zeros((mx, width))
    pl[:count] = limbs[:count, :width]
    pi = idx.new_zeros(mx)
    pi[:count] = idx[:count]
    pn = neg.new_zeros(mx)
    pn[:count] = neg[:count]
    gl = limbs.new_empty((size, mx, width))
    gi = idx.new_empty((size, mx))
    gn = neg.new_empty((size, mx))
    dist.all_gather_into_tensor(gl.view(-1), pl.view(-1))
    dist.all_gather_into_tensor(gi.view(-1), pi)
    dist.all_gather_into_tensor(gn.view(-1), pn)
    return (torch.cat([gl[g, :c] for g, c in enumerate(allc)]), torch.cat([gi[g, :c] for g, c in enumerate(allc)]),
            torch.cat([gn[g, :c] for g, c in enumerate(allc)]))
