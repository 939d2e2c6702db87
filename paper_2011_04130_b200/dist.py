"""Multi-GPU plumbing for block-sharded extraction (one process per GPU).

Blocks are independent (Fig. 5) and the seed is shared
and read-only, so the hot path shards by contiguous block ranges with NO
data-path collective.  The collectives here are setup/teardown only:

* ``broadcast_seed``    -- the packed seed from rank 0, once (NCCL over NVLink);
* ``allreduce_counts``  -- the 256 histogram counts of sharded samples, so any
                           rank can finalise ``qrng_entropy_from_counts``;
* ``gather_keys``       -- optional assembly of the full key stream (C4) from
                           per-rank packed shards at arbitrary bit offsets;
* ``extract_block_distributed`` -- NEXT-4: ONE block across the group
                           (distributed four-step NTT, qrng_dist_*): the one
                           data-path exchange is a single all-to-all of N2
                           words per rank, then an OR (byte SUM of disjoint
                           bits) of the ranks' key bits.

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


def _unpack_dev(t, nbits):
    """MSB-first bits of a uint8 tensor (on its device)."""
    import torch
    shifts = torch.arange(7, -1, -1, device=t.device, dtype=torch.uint8)
    return ((t[:, None] >> shifts) & 1).reshape(-1)[:nbits]


def _pack_dev(bits):
    import torch
    pad = (-bits.numel()) % 8
    if pad:
        bits = torch.cat([bits, torch.zeros(pad, dtype=bits.dtype, device=bits.device)])
    w = torch.tensor([128, 64, 32, 16, 8, 4, 2, 1], dtype=torch.uint8, device=bits.device)
    return (bits.reshape(-1, 8) * w).sum(dim=1, dtype=torch.int32).to(torch.uint8)


def gather_keys(local_key, n_local_blocks: int, m: int, group=None):
    """All-gather per-rank packed keys and return the full key stream (C4) as a
    tensor on the local key's device.

    Shards may hold different block counts (shard_range); each shard is a
    self-contained packed stream of n_local_blocks*m bits.  When every shard
    ends on a byte boundary (every config on 1/2/4/8 GPUs) the streams are
    concatenated as bytes; otherwise bit-level on the device.  With gloo the
    exchange itself goes through host copies.
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = local_key.device
    cdev = dev if dist.get_backend(group) != "gloo" else torch.device("cpu")
    cnt = torch.tensor([n_local_blocks], dtype=torch.int64, device=cdev)
    cnts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt, group=group)
    sizes = [int(c.item()) for c in cnts]
    maxbytes = max((s * m + 7) // 8 for s in sizes)
    pad = torch.zeros(maxbytes, dtype=torch.uint8, device=cdev)
    pad[:local_key.numel()] = local_key.to(cdev)
    outs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    outs = [o.to(dev) for o in outs]
    if all((s * m) % 8 == 0 for s in sizes[:-1]):
        return torch.cat([o[:(s * m + 7) // 8] for o, s in zip(outs, sizes)])
    bits = torch.cat([_unpack_dev(o[:(s * m + 7) // 8], s * m) for o, s in zip(outs, sizes)])
    return _pack_dev(bits)


def four_step_exchange(ops, group=None):
    """The NEXT-4 data movement, independent of where the local steps run.

    ``ops.local()`` returns this rank's send buffer (N2 words; chunk r' of
    N2/world words goes to rank r'), ``ops.finish(recv)`` takes the received
    buffer (chunk k1 from rank k1) and returns this rank's key bytes (its bits
    only, zeros elsewhere).  One all-to-all of equal chunks, then a byte-wise
    SUM all-reduce of the keys -- the ranks' bits are disjoint, so the sum is
    their OR.  Collectives run on the tensors' device for NCCL and on host
    copies for gloo."""
    import torch
    import torch.distributed as dist
    send = ops.local()
    host = dist.get_backend(group) == "gloo" and send.device.type != "cpu"
    s = send.cpu() if host else send
    recv = torch.empty_like(s)
    dist.all_to_all_single(recv, s, group=group)
    key = ops.finish(recv.to(send.device) if host else recv)
    k = key.cpu() if host and key.device.type != "cpu" else key
    dist.all_reduce(k, op=dist.ReduceOp.SUM, group=group)
    return k.to(key.device) if k is not key else key


class _GpuOps:
    """The product's local steps: qrng_dist_local / qrng_dist_finish on this rank's GPU."""

    def __init__(self, plan, block, stream=None):
        self.plan, self.block, self.stream = plan, block, stream

    def local(self):
        return self.plan.local(self.block, self.plan.new_buffer(), stream=self.stream)

    def finish(self, recv):
        import torch
        from paper_2011_04130_b200 import out_bytes
        key = torch.zeros((out_bytes(1, self.plan.m) + 3) // 4 * 4, dtype=torch.uint8, device=recv.device)
        self.plan.finish(recv.contiguous(), key, stream=self.stream)
        return key[:out_bytes(1, self.plan.m)]


def extract_block_distributed(block, n: int, m: int, seed, group=None, plan=None, stream=None):
    """NEXT-4: the m key bits of ONE n-bit block (block bits replicated on every
    rank, seed on every rank -- broadcast_seed), computed across the group's
    GPUs; returns the full key (ceil(m/8) bytes) on every rank."""
    import torch.distributed as dist
    from paper_2011_04130_b200 import DistPlan
    own = plan is None
    if own:
        plan = DistPlan(n, m, seed, dist.get_world_size(group), dist.get_rank(group), stream=stream)
    try:
        return four_step_exchange(_GpuOps(plan, block, stream), group)
    finally:
        if own:
            plan.close()


def extract_block_emulated(block, n: int, m: int, seed, world: int):
    """TEST / single-GPU check of NEXT-4: the `world` ranks' local steps run one
    after another in this process on one GPU (no rank waits on another inside a
    kernel), the all-to-all is a device copy of chunks, the OR a byte sum."""
    import torch
    from paper_2011_04130_b200 import DistPlan, out_bytes
    plans = [DistPlan(n, m, seed, world, r) for r in range(world)]
    try:
        sends = [p.local(block, p.new_buffer()) for p in plans]
        C = plans[0].exchange_words // world
        key = torch.zeros(out_bytes(1, m), dtype=torch.int32, device=block.device)
        for r, p in enumerate(plans):
            recv = torch.cat([s[r * C:(r + 1) * C] for s in sends])
            k = torch.zeros((out_bytes(1, m) + 3) // 4 * 4, dtype=torch.uint8, device=block.device)
            p.finish(recv, k)
            key += k[:out_bytes(1, m)].to(torch.int32)
        return key.to(torch.uint8)
    finally:
        for p in plans:
            p.close()
