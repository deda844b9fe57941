"""Multi-GPU O-DU batches: cells sharded across ranks, one codebook all-gather.

SURVEY.md §8(e): slots and cells are independent (no cross-slot state; the
coupled bisection never spans two slots), so a batch of C cells is split in
contiguous blocks, one per rank (one process per GPU), with NO collective on
the data path.  The single exchange the north star asks for — assembling
every cell's codebook on every rank — is one all-gather of the int32
``[cells][cap+1][E]`` blocks (51,200 B at 256 cells x cap 4 x E 10): NCCL over
NVLink on GPUs, gloo in the CPU tests.  Node states stay on the rank that
built them.
"""

from __future__ import annotations


def shard_bounds(total: int, world: int, rank: int) -> tuple:
    """Contiguous block of ``total`` items owned by ``rank`` (balanced to 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(int(total), int(world))
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def max_shard(total: int, world: int) -> int:
    return -(-int(total) // int(world))


def gather_codebooks(local, total: int, group=None):
    """All-gather per-rank codebook blocks into (total, cap+1, E) on every rank.

    ``local`` is this rank's (n_r, cap+1, E) int32 tensor (device tensor for
    NCCL, CPU tensor for gloo).  Blocks are padded to the largest shard so
    the collective is one equal-size all_gather_into_tensor.
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    width = max_shard(total, world)
    cols, users = local.shape[1], local.shape[2]
    padded = torch.zeros((width, cols, users), dtype=local.dtype, device=local.device)
    padded[: local.shape[0]] = local
    out = torch.empty((world * width, cols, users), dtype=local.dtype, device=local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, padded, group=group)
    else:
        dist.all_gather(list(out.chunk(world)), padded, group=group)
    pieces = []
    for r in range(world):
        lo, hi = shard_bounds(total, world, r)
        pieces.append(out[r * width: r * width + (hi - lo)])
    return torch.cat(pieces)


def build_codebooks_sharded(compute, allocs, eps, group=None):
    """Each rank computes its block of cells with ``compute(allocs_blk,
    eps_blk) -> (n, cap+1, E) tensor`` and the blocks are all-gathered.

    ``allocs``/``eps`` hold the WHOLE batch (every rank sees the same O-DU
    input; each reads only its block).  Returns (codebooks of all cells,
    this rank's local block).
    """
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    total = int(allocs.shape[0])
    lo, hi = shard_bounds(total, world, rank)
    local = compute(allocs[lo:hi], None if eps is None else eps[lo:hi])
    return gather_codebooks(local, total, group), local
