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
        full = qd.gather_keys(torch.from_numpy(local), b1 - b0, m).numpy()  # bit-level assembly
        ref = oracle.extract(raw_all, B, n, m, seed.numpy())
        # byte-aligned shards (every config on 1/2/4/8 GPUs): byte concatenation
        m2, B2 = 176, 16
        c0, c1 = qd.shard_range(B2, rank, world)
        raw2 = S.random_bytes(98, B2 * n // 8)
        seed2 = S.random_bytes(98, (n + m2 - 1 + 7) // 8, tag=5)
        loc2 = oracle.extract(raw2[c0 * n // 8:c1 * n // 8], c1 - c0, n, m2, seed2)
        full2 = qd.gather_keys(torch.from_numpy(loc2), c1 - c0, m2).numpy()
        ok2 = np.array_equal(full2, oracle.extract(raw2, B2, n, m2, seed2))
        # sharded histogram: each rank counts its share of the samples
        samples = S.adc_samples(7, 100_003, 128, 20)
        lo, hi = qd.shard_range(samples.size, rank, world)
        counts = torch.from_numpy(oracle.hist256(samples[lo:hi]).astype(np.int64))
        qd.allreduce_counts(counts)
        q.put((rank, np.array_equal(full, ref) and ok2,
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


# ---- NEXT-4: one block across ranks (distributed four-step NTT) ------------------
# The data movement of paper_2011_04130_b200.dist.four_step_exchange (one
# all-to-all of equal chunks, then an OR of the ranks' keys by byte SUM) is
# checked here on CPU with gloo.  The local steps -- the CUDA kernels
# qrng_dist_local / qrng_dist_finish on a GPU -- are modelled by a plain
# numpy reading of the four-step decomposition (natural-order DFT matrices mod
# p = 7*2^26 + 1), so a wrong twist exponent, chunk order or column range in
# the decomposition fails against the oracle.

P2 = 469762049  # 7 * 2^26 + 1, primitive root 3


def _dft(vec, root):
    """Natural-order DFT mod P2 by its matrix (small sizes)."""
    N = vec.size
    e = (np.arange(N)[:, None] * np.arange(N)[None, :]) % N
    pw = np.array([pow(root, int(k), P2) for k in range(N)], dtype=np.int64)
    return ((pw[e] * (vec % P2)[None, :]) % P2).sum(axis=1) % P2


class _NumpyFourStep:
    def __init__(self, x_bits, s_bits, n, m, world, rank):
        L = n + m - 1
        logW = world.bit_length() - 1
        logP = max(int(np.ceil(np.log2(L))), 10 + logW)
        self.P, self.N2, self.W, self.r, self.n, self.m = 1 << logP, 1 << (logP - logW), world, rank, n, m
        self.wP = pow(3, (P2 - 1) >> logP, P2)
        self.wW = pow(self.wP, self.N2, P2)
        self.wN2 = pow(self.wP, world, P2)
        self.x, self.s = x_bits, s_bits

    def _u(self, bits):
        N2, W, r = self.N2, self.W, self.r
        full = np.zeros(self.P, np.int64)
        full[:bits.size] = bits
        cols = full.reshape(W, N2)  # [n1][n2] = t = N2 n1 + n2
        c = np.array([pow(self.wW, n1 * r, P2) for n1 in range(W)], np.int64)
        tw = np.array([pow(self.wP, n2 * r, P2) for n2 in range(N2)], np.int64)
        return ((cols * c[:, None]).sum(axis=0) % P2) * tw % P2

    def local(self):
        import torch
        X = _dft(self._u(self.x), self.wN2)
        S = _dft(self._u(self.s), self.wN2)
        v = _dft(X * S % P2, pow(self.wN2, P2 - 2, P2))
        itw = np.array([pow(self.wP, (-(n2 * self.r)) % (P2 - 1), P2) for n2 in range(self.N2)], np.int64)
        return torch.from_numpy((v * itw % P2).astype(np.int32))

    def finish(self, recv):
        import torch
        W, N2, r = self.W, self.N2, self.r
        C = N2 // W
        V = recv.numpy().astype(np.int64).reshape(W, C)  # [k1][j]
        pinv = pow(self.P, P2 - 2, P2)
        key = np.zeros(self.m, np.uint8)
        for n1 in range(W):
            w = np.array([pow(self.wW, (-(n1 * k1)) % (P2 - 1), P2) for k1 in range(W)], np.int64)
            z = (V * w[:, None] % P2).sum(axis=0) % P2 * pinv % P2
            t = N2 * n1 + r * C + np.arange(C)
            i = t - (self.n - 1)
            ok = (i >= 0) & (i < self.m)
            key[i[ok]] = (z[ok] & 1).astype(np.uint8)
        return torch.from_numpy(np.packbits(key))


def _four_step_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        n, m = 256, 179
        x = np.unpackbits(S.random_bytes(31, n // 8))
        s = np.unpackbits(S.random_bytes(31, (n + m - 1 + 7) // 8, tag=4))[:n + m - 1]
        key = qd.four_step_exchange(_NumpyFourStep(x, s, n, m, world, rank))
        ref = oracle.extract(np.packbits(x), 1, n, m, np.packbits(s))
        q.put((rank, np.array_equal(key.numpy(), ref)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_four_step_exchange_gloo(oracle_mod, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_four_step_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert sorted(r[0] for r in res) == list(range(world))
    assert all(r[1] for r in res), "distributed four-step key differs from the oracle"


def test_bench_reference_arm_contract():
    """`bench.py --impl reference` (this tier's reference arm: the CPU oracle)
    prints one JSON line with the contract's keys."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--config", "1",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
