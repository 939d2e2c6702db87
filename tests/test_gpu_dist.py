"""NEXT-4 on the GPU: one block across `world` ranks (distributed four-step NTT,
qrng_dist_* through the C ABI), bit-exact against the CPU oracle.

* extract_block_emulated runs the world ranks' kernels one after another on
  one GPU (no rank waits on another inside a kernel) with the all-to-all as a
  device copy of chunks -- the layout and every kernel of every rank;
* two processes on one GPU with a gloo group run the real orchestration
  (paper_2011_04130_b200.dist.extract_block_distributed: all_to_all_single +
  the OR all-reduce);
* the single-GPU path for 2^23 < L <= 2^26 (world-1 four-step, block by
  block) through qrng_toeplitz_extract.

Run on a B200:  python -m pytest tests -m gpu
"""
import os
import socket

import numpy as np
import pytest

import qrng_synth as S

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2011_04130_b200 as q
    from paper_2011_04130_b200 import build
    build.build()
    q.load_library()
    yield q


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint8)).cuda()


def check_rows(oracle_mod, key, raw, seed, n, m, B=1, n_rows=300, key_seed=0):
    rng = np.random.default_rng(key_seed)
    bl = np.repeat(np.arange(B), n_rows + 4).astype(np.uint64)
    rw = np.concatenate([np.r_[0, 1, m - 2, m - 1, rng.integers(0, m, n_rows)] for _ in range(B)]).astype(np.uint64)
    ref = oracle_mod.extract_rows(raw, bl, rw, n, m, seed)
    pos = (bl * m + rw).astype(np.int64)
    got = (key[pos >> 3] >> (7 - (pos & 7))) & 1
    bad = np.nonzero(got != ref)[0]
    assert bad.size == 0, f"{bad.size} sampled bits differ (first row {rw[bad[0]]})"


@pytest.mark.parametrize("n,m", [(1024, 716), (4096, 2867), (8192, 100), (65536, 45875)])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_emulated_small_whole_key(q, oracle_mod, n, m, world):
    from paper_2011_04130_b200 import dist as qd
    raw = S.random_bytes(n + world, n // 8)
    seed = S.random_bytes(n + world, (n + m - 1 + 7) // 8, tag=6)
    key = qd.extract_block_emulated(dev(raw), n, m, dev(seed), world).cpu().numpy()
    assert np.array_equal(key, oracle_mod.extract(raw, 1, n, m, seed))


def test_emulated_all_ones(q, oracle_mod):
    """Every window sum at its maximum n (p > n) on the distributed path."""
    from paper_2011_04130_b200 import dist as qd
    n, m = 1 << 16, 45875
    raw = np.full(n // 8, 0xFF, np.uint8)
    seed = np.full((n + m - 1 + 7) // 8, 0xFF, np.uint8)
    for world in (1, 4):
        key = qd.extract_block_emulated(dev(raw), n, m, dev(seed), world).cpu().numpy()
        assert np.array_equal(key, oracle_mod.extract(raw, 1, n, m, seed)), world


@pytest.mark.parametrize("world", [1, 2, 8])
def test_emulated_n_2_24(q, oracle_mod, world):
    """n = 2^24 (L = 2.85e7 > 2^23: past the single-prime limit), m = floor(0.7 n)."""
    from paper_2011_04130_b200 import dist as qd
    n = 1 << 24
    m = 7 * n // 10
    raw = S.adc_samples(24, n // 8)
    seed = S.uniform_bits(24, n + m - 1, tag=7)
    key = qd.extract_block_emulated(dev(raw), n, m, dev(seed), world).cpu().numpy()
    check_rows(oracle_mod, key, raw, seed, n, m, key_seed=world)
    tail = m % 8
    if tail:
        assert key[-1] & ((1 << (8 - tail)) - 1) == 0


def test_single_gpu_large_L_through_api(q, oracle_mod):
    """qrng_toeplitz_extract with 2^23 < L <= 2^26 runs the world-1 four-step
    block by block; two blocks, sampled rows of both, pad bits zero."""
    n = 1 << 24
    m = 7 * n // 10 + 3
    B = 2
    raw = S.adc_samples(25, B * n // 8)
    seed = S.uniform_bits(25, n + m - 1, tag=8)
    key = q.toeplitz_extract(dev(raw), B, n, m, dev(seed)).cpu().numpy()
    check_rows(oracle_mod, key, raw, seed, n, m, B=B, n_rows=200)
    tail = B * m % 8
    if tail:
        assert key[-1] & ((1 << (8 - tail)) - 1) == 0
    n2, m2 = 3 << 24, (1 << 24) + 2  # L = 2^26 + 2^24 + 1 > 2^26
    with pytest.raises(q.QrngError) as ei:
        q.toeplitz_extract(torch.zeros(n2 // 8, dtype=torch.uint8, device="cuda"), 1, n2, m2,
                           torch.zeros((n2 + m2 + 7) // 8, dtype=torch.uint8, device="cuda"))
    assert ei.value.status == q.QRNG_E_UNSUPPORTED


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, qu):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2011_04130_b200 as qq
        from paper_2011_04130_b200 import dist as qd
        qq.load_library()
        torch.cuda.set_device(0)
        n, m = 1 << 20, 734003
        raw = S.adc_samples(26, n // 8)
        seed = torch.zeros((n + m - 1 + 7) // 8, dtype=torch.uint8)
        if rank == 0:
            seed.copy_(torch.from_numpy(S.uniform_bits(26, n + m - 1, tag=9)))
        qd.broadcast_seed(seed)
        key = qd.extract_block_distributed(dev(raw), n, m, seed.cuda())
        qu.put((rank, key.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_two_process_gloo_orchestration(q, oracle_mod):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, qu)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(qu.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    n, m = 1 << 20, 734003
    raw = S.adc_samples(26, n // 8)
    seed = S.uniform_bits(26, n + m - 1, tag=9)
    assert np.array_equal(res[0], res[1])
    check_rows(oracle_mod, res[0], raw, seed, n, m, n_rows=400)
