"""GPU parity of the Karatsuba decomposition over the tcgen05 GEMM path
(DESIGN.md "Karatsuba over the GEMM path"): for every depth the CUDA path
(through the C ABI) is bit-exact to the CPU oracle.

Run on a B200:  python -m pytest tests -m gpu
"""
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
    q.set_debug_path(q.PATH_AUTO)
    q.set_karatsuba(-1)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint8)).cuda()


def kara_extract(q, raw, B, n, m, seed, depth):
    q.set_debug_path(q.PATH_GEMM)
    q.set_karatsuba(depth)
    try:
        with q.Plan(n, m, dev(seed)) as plan:
            info = plan.info()
            out = plan.extract(dev(raw), B)
            torch.cuda.synchronize()
            return out.cpu().numpy(), info
    finally:
        q.set_debug_path(q.PATH_AUTO)
        q.set_karatsuba(-1)


def assert_same(got, ref, m):
    if not np.array_equal(got, ref):
        gb, rb = np.unpackbits(got), np.unpackbits(ref)
        bad = np.nonzero(gb != rb)[0]
        raise AssertionError(f"{bad.size} bits differ; first at bit {bad[0]} "
                             f"(block {bad[0] // m}, i {bad[0] % m})")


CASES = [
    (256, 200, 3), (512, 300, 129), (1024, 716, 17), (1024, 1, 4), (1024, 1023, 130),
    (2048, 1433, 10), (3072, 2100, 7), (4096, 2867, 257), (8192, 5734, 131), (8192, 100, 9),
    (16384, 11468, 3), (16384, 16383, 2), (32768, 22937, 2),
]


@pytest.mark.parametrize("depth", [0, 1, 2, 3, 5, -1])
@pytest.mark.parametrize("n,m,B", CASES)
def test_random(q, oracle_mod, n, m, B, depth):
    key = n * 7919 + m + depth
    raw = S.random_bytes(key, B * n // 8)
    seed = S.random_bytes(key, (n + m - 1 + 7) // 8, tag=2)
    got, info = kara_extract(q, raw, B, n, m, seed, depth)
    if depth >= 0:
        assert info["karatsuba_depth"] <= depth
    assert_same(got, oracle_mod.extract(raw, B, n, m, seed), m)


@pytest.mark.parametrize("depth", [0, 1, 3, -1])
@pytest.mark.parametrize("n,m,B", [(1024, 716, 3), (8192, 5734, 3), (16384, 11468, 2), (65536, 45875, 2)])
def test_all_ones(q, oracle_mod, n, m, B, depth):
    """All-ones seed and raw: every leaf window sum is maximal (n = 2^16 at depth
    0: the S32 sums reach 65536, whose parity survives the epilogue's 16-bit
    packed accumulator reads) and every XOR combination of seed windows / block
    windows is exercised with dense data."""
    raw = np.full(B * n // 8, 0xFF, np.uint8)
    seed = np.full((n + m - 1 + 7) // 8, 0xFF, np.uint8)
    got, _ = kara_extract(q, raw, B, n, m, seed, depth)
    assert_same(got, oracle_mod.extract(raw, B, n, m, seed), m)


@pytest.mark.parametrize("depth", [0, 1, 2, 3, -1])
def test_config2_all_blocks(q, oracle_mod, depth):
    """BASELINE config 2 (what bench.py times), every block, each depth."""
    w = S.CONFIGS[2]
    raw, seed = S.workload_inputs(w)
    ref = oracle_mod.extract(raw, w.n_blocks, w.n, w.m, seed)
    got, info = kara_extract(q, raw, w.n_blocks, w.n, w.m, seed, depth)
    assert_same(got, ref, w.m)
    if depth > 0:
        assert info["karatsuba_depth"] == depth and info["macs_per_block"] < w.n * w.m


def sampled(oracle_mod, got, raw, seed, n, m, B, n_rows=256, key=0):
    rng = np.random.default_rng(key)
    blocks = sorted({0, B - 1, B // 2, *rng.integers(0, B, 5).tolist()})
    bl, rw = [], []
    for b in blocks:
        rows = np.unique(np.concatenate([[0, 1, m - 2, m - 1], rng.integers(0, m, n_rows)]))
        bl += [b] * rows.size
        rw += rows.tolist()
    bl, rw = np.array(bl, np.uint64), np.array(rw, np.uint64)
    ref = oracle_mod.extract_rows(raw, bl, rw, n, m, seed)
    gb = np.unpackbits(got)[(bl * m + rw).astype(np.int64)]
    bad = np.nonzero(gb != ref)[0]
    assert bad.size == 0, f"{bad.size} sampled bits differ, first (block {bl[bad[0]]}, row {rw[bad[0]]})"


@pytest.mark.parametrize("log2n", [15, 16, 17, 18])
def test_large_n_sampled_plus_full_block(q, oracle_mod, log2n):
    """Config 3 (n = 2^16) and sweep points beyond the dense kernel's 2^16 limit
    (the Karatsuba root may exceed it; leaves stay <= 2^16): sampled rows of
    every shape plus one complete block."""
    w = S.sweep_workload(log2n)
    B = 130 if log2n <= 16 else 66
    raw, seed = S.workload_inputs(w, 0, B)
    got, info = kara_extract(q, raw, B, w.n, w.m, seed, -1)
    assert info["karatsuba_depth"] >= 1
    sampled(oracle_mod, got, raw, seed, w.n, w.m, B, key=log2n)
    b = B - 1
    ref = oracle_mod.extract_blocks(raw, [b], w.n, w.m, seed)[0]
    assert np.array_equal(np.unpackbits(got)[b * w.m:(b + 1) * w.m], np.unpackbits(ref)[:w.m])


def test_config3_full_size_sampled(q, oracle_mod):
    w = S.CONFIGS[3]
    raw, seed = S.workload_inputs(w)
    got, info = kara_extract(q, raw, w.n_blocks, w.n, w.m, seed, -1)
    assert info["karatsuba_depth"] >= 1
    sampled(oracle_mod, got, raw, seed, w.n, w.m, w.n_blocks, key=3)


def test_guard_bytes_untouched(q, oracle_mod):
    n, m, B = 2048, 1433, 33  # B*m % 32 != 0: partial final word through the combine kernel
    raw = S.random_bytes(11, B * n // 8)
    seed = S.random_bytes(11, (n + m - 1 + 7) // 8, tag=3)
    q.set_debug_path(q.PATH_GEMM)
    q.set_karatsuba(3)
    try:
        nb = q.out_bytes(B, m)
        d_out = torch.full((nb + 64,), 0xEE, dtype=torch.uint8, device="cuda")
        q.toeplitz_extract(dev(raw), B, n, m, dev(seed), out=d_out[:nb])
        got = d_out.cpu().numpy()
    finally:
        q.set_debug_path(q.PATH_AUTO)
        q.set_karatsuba(-1)
    assert_same(got[:nb], oracle_mod.extract(raw, B, n, m, seed), m)
    assert (got[nb:] == 0xEE).all()


def test_back_to_back_mixed_plans_one_stream(q, oracle_mod):
    """Karatsuba extractions of different shapes queued back to back on one
    stream without synchronisation (the Q-buffer, leaf-GEMM and combine kernels
    are chained with programmatic dependent launch): every key is still exact."""
    shapes = [(8192, 5734, 33), (16384, 11468, 7), (4096, 2867, 65), (8192, 5734, 17), (32768, 22937, 3)]
    jobs = []
    for k, (n, m, B) in enumerate(shapes):
        raw = S.random_bytes(9000 + k, B * n // 8)
        seed = S.random_bytes(9000 + k, (n + m - 1 + 7) // 8, tag=4)
        jobs.append((n, m, B, raw, seed, dev(raw), dev(seed)))
    q.set_debug_path(q.PATH_GEMM)
    try:
        outs = [q.toeplitz_extract(dr, B, n, m, ds) for n, m, B, raw, seed, dr, ds in jobs]
        torch.cuda.synchronize()
    finally:
        q.set_debug_path(q.PATH_AUTO)
    for (n, m, B, raw, seed, _, _), out in zip(jobs, outs):
        assert_same(out.cpu().numpy(), oracle_mod.extract(raw, B, n, m, seed), m)
