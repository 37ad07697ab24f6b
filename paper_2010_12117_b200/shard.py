"""Multi-GPU sharding of the (prime x node) work.

One process per GPU under torch.distributed (NCCL over NVLink on the GPU,
gloo in the CPU tests).  Two partitions, combined:

* prime-sharded: the first G*floor(P/G) primes go round-robin (rank g takes
  primes g, g+G, ...) and each rank runs FWD -> DET -> IFFT for them with no
  communication; their residue rows are all-gathered once before the CRT;
* slab-sharded: the remaining P mod G primes (all of them when P < G, e.g.
  a one-prime plan on 8 GPUs) are split by the slowest grid axis: rank g
  computes the determinants of the nodes with a_0 in its slab (a contiguous
  node range), the slabs are all-gathered into the full determinant grid on
  every rank, and every rank runs that prime's (cheap) inverse NTT.

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
