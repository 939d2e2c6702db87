"""Multi-rank host logic on CPU (gloo, world size 2): shard arithmetic, seed
broadcast, sharded-histogram all-reduce and key concatenation.  The per-rank
"extraction" is the CPU oracle here (no GPU in this container); on a B200 the
same plumbing wraps qrng_toeplitz_extract (bench.py under torchrun)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2011_04130_b200 import dist as qd
import qrng_synth as S


def test_shard_range_partitions():
    for B in (1, 7, 32, 256, 16384, 16385):
        for W in (1, 2, 3, 4, 8):
            if W > B:
                continue
            ranges = [qd.shard_range(B, r, W) for r in range(W)]
            assert ranges[0][0] == 0 and ranges[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            assert max(b - a for a, b in ranges) - min(b - a for a, b in ranges) <= 1
    # BASELINE configs on 8 GPUs: every shard starts on a 32-bit word boundary
    for w in S.CONFIGS.values():
        for r in range(8):
            assert qd.shard_bit_offset(w.n_blocks, r, 8, w.m) % 32 == 0


def test_concat_bitstreams_arbitrary_offsets():
    rng = np.random.default_rng(0)
    bits = rng.integers(0, 2, 1000).astype(np.uint8)
    cuts = [0, 13, 14, 333, 1000]
    parts = [np.packbits(bits[a:b]) for a, b in zip(cuts, cuts[1:])]
    got = qd.concat_bitstreams(parts, [b - a for a, b in zip(cuts, cuts[1:])])
    assert np.array_equal(got, np.packbits(bits))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        n, m, B = 256, 179, 13  # shard boundaries not byte aligned (13 blocks, m odd)
        raw_all = S.random_bytes(99, B * n // 8)
        seed = torch.zeros((n + m - 1 + 7) // 8, dtype=torch.uint8)
        if rank == 0:
            seed.copy_(torch.from_numpy(S.random_bytes(99, seed.numel(), tag=5)))
        qd.broadcast_seed(seed)
        b0, b1 = qd.shard_range(B, rank, world)
        local = oracle.extract(raw_all[b0 * n // 8:b1 * n // 8], b1 - b0, n, m, seed.numpy())
        full = qd.gather_keys(torch.from_numpy(local), b1 - b0, m)
        ref = oracle.extract(raw_all, B, n, m, seed.numpy())
        # sharded histogram: each rank counts its share of the samples
        samples = S.adc_samples(7, 100_003, 128, 20)
        lo, hi = qd.shard_range(samples.size, rank, world)
        counts = torch.from_numpy(oracle.hist256(samples[lo:hi]).astype(np.int64))
        qd.allreduce_counts(counts)
        q.put((rank, np.array_equal(full, ref),
               np.array_equal(counts.numpy().astype(np.uint64), oracle.hist256(samples))))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_plumbing(oracle_mod):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert sorted(r[0] for r in res) == [0, 1]
    assert all(r[1] for r in res), "concatenated shards differ from the single-process key"
    assert all(r[2] for r in res), "all-reduced histogram differs"


@pytest.mark.parametrize("cfg,scaling,blocks", [(2, "weak", 2 * 16384), (16, "strong", 16384)])
def test_bench_launcher_spawns_ranks(cfg, scaling, blocks):
    """`bench.py --gpus 2` outside torchrun re-launches itself with 2 ranks
    (torch.distributed.run, gloo for --dry-run): the line reports n_gpus 2,
    the SURVEY 8(e) contiguous partition and the seed broadcast on every rank."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run",
                        "--config", str(cfg)], capture_output=True, text=True, timeout=300, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["dry_run"] and line["scaling"] == scaling
    assert line["config"]["blocks_total"] == blocks
    assert line["shards"] == [list(qd.shard_range(blocks, k, 2)) for k in range(2)]
    assert line["seed_broadcast_ok_ranks"] == 2 and line["max_over_ranks"] == 2.0
