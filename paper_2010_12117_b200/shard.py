"""Multi-GPU sharding of the (prime x node) work.

One process per GPU under torch.distributed.  Primes are independent until
the CRT, so rank g runs FWD -> DET -> IFFT for primes g, g+G, g+2G, ... with
no communication, and the only collective is the final gather of the residue
tensors ([P][nodes] u32, NCCL over NVLink on the GPU, gloo in the CPU tests),
after which the CRT runs on the gathered block.  Output is bit-identical for
any device count because every prime's residues are a pure function of the
prime (test_multiproc.py, test_gpu_parity.py).
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


def gather_residues(local, prime_count: int, rank: int, size: int):
    """All-gather each rank's [ceil(P/G)][nodes] block; return the [P][nodes]
    tensor in prime order (every rank receives it, so each can run the CRT or
    the caller can keep rank 0's)."""
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
