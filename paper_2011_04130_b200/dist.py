"""Multi-GPU plumbing for block-sharded extraction (one process per GPU).

Blocks are independent (Fig. 5) and the seed is shared
and read-only, so the hot path shards by contiguous block ranges with NO
data-path collective.  The collectives here are setup/teardown only:

* ``broadcast_seed``    -- the packed seed from rank 0, once (NCCL over NVLink);
* ``allreduce_counts``  -- the 256 histogram counts of sharded samples, so any
                           rank can finalise ``qrng_entropy_from_counts``;
* ``gather_keys``       -- optional assembly of the full key stream (C4) from
                           per-rank packed shards at arbitrary bit offsets.

Everything takes a ``torch.distributed`` process group (NCCL on GPUs, gloo in
the CPU tests).
"""
from __future__ import annotations

import numpy as np


def shard_range(n_blocks: int, rank: int, world: int) -> tuple[int, int]:
    """Blocks [b0, b1) owned by `rank`: floor(r B / W) .. floor((r+1) B / W)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return (rank * n_blocks) // world, ((rank + 1) * n_blocks) // world


def shard_bit_offset(n_blocks: int, rank: int, world: int, m: int) -> int:
    """First key bit of the rank's shard in the full stream (C4: bit b*m + i)."""
    return shard_range(n_blocks, rank, world)[0] * m


def broadcast_seed(seed, src: int = 0, group=None):
    """Broadcast the packed seed tensor (uint8) from `src` in place."""
    import torch.distributed as dist
    dist.broadcast(seed, src, group=group)
    return seed


def allreduce_counts(counts, group=None):
    """Sum the 256 uint64 histogram counts (int64 tensor) over ranks in place."""
    import torch.distributed as dist
    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts


def concat_bitstreams(parts: list[np.ndarray], nbits: list[int]) -> np.ndarray:
    """Concatenate packed MSB-first bit streams of the given bit lengths."""
    bits = [np.unpackbits(np.asarray(p, np.uint8))[:k] for p, k in zip(parts, nbits)]
    return np.packbits(np.concatenate(bits)) if bits else np.zeros(0, np.uint8)


def gather_keys(local_key, n_local_blocks: int, m: int, group=None) -> np.ndarray:
    """All-gather per-rank packed keys and return the full key stream (C4).

    Shards may hold different block counts (shard_range); each shard is a
    self-contained packed stream of n_local_blocks*m bits.
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = local_key.device
    cnt = torch.tensor([n_local_blocks], dtype=torch.int64, device=dev)
    cnts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt, group=group)
    sizes = [int(c.item()) for c in cnts]
    maxbytes = max((s * m + 7) // 8 for s in sizes)
    pad = torch.zeros(maxbytes, dtype=torch.uint8, device=dev)
    pad[:local_key.numel()] = local_key
    outs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return concat_bitstreams([o.cpu().numpy()[:(s * m + 7) // 8] for o, s in zip(outs, sizes)],
                             [s * m for s in sizes])
