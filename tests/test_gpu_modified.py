"""GPU parity of the modified Toeplitz [T | I_m] (SURVEY
NEXT-1) against the oracle: bit-exact on both paths -- fused (P <= 2^15, incl.
two blocks per transform) and multi-pass NTT, and the tensor-core path
(inputs repacked to a multiple of 128 bits, C1 product, XOR of the last m raw
bits) -- full-size configs on sampled outputs."""
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
    return q


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint8)).cuda()


PATHS = ["auto", "ntt", "gemm"]


def gpu_mod(q, raw, B, n, m, seed, path="auto"):
    q.set_debug_path({"auto": q.PATH_AUTO, "ntt": q.PATH_NTT, "gemm": q.PATH_GEMM}[path])
    try:
        out = q.modified_toeplitz_extract(dev(raw), B, n, m, dev(seed))
        torch.cuda.synchronize()
    finally:
        q.set_debug_path(q.PATH_AUTO)
    return out.cpu().numpy()


def assert_same(got, ref, m):
    if not np.array_equal(got, ref):
        bad = np.nonzero(np.unpackbits(got) != np.unpackbits(ref))[0]
        raise AssertionError(f"{bad.size} bits differ; first at block {bad[0] // m}, row {bad[0] % m}")


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("n,m,B", [
    (32, 1, 3), (64, 20, 5), (96, 95, 4), (1024, 716, 9), (1024, 300, 7), (8192, 5734, 5),
    (8192, 2000, 4), (16384, 11468, 3), (32768, 22937, 2), (65536, 45875, 2), (65536, 10000, 2),
    (4096, 3968, 33), (2048, 1, 5), (66592, 1024, 2),
])
def test_modified_random(q, oracle_mod, n, m, B, path):
    if path == "gemm" and n - m > (1 << 16):
        pytest.skip("GEMM path: n - m <= 2^16")
    raw = S.random_bytes(n + 3 * m, B * n // 8)
    seed = S.random_bytes(n + 3 * m, n // 8, tag=7)
    if n * m * B <= 2e8:
        ref = oracle_mod.modified_extract(raw, B, n, m, seed)
        assert_same(gpu_mod(q, raw, B, n, m, seed, path), ref, m)
    else:
        got = gpu_mod(q, raw, B, n, m, seed, path)
        bl = np.repeat(np.arange(B), m)
        rw = np.tile(np.arange(m), B)
        ref = oracle_mod.modified_rows(raw, bl, rw, n, m, seed)
        assert np.array_equal(np.unpackbits(got)[:B * m], ref)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("n,m,B", [(8192, 5734, 3), (65536, 1000, 2)])
def test_modified_all_ones(q, oracle_mod, n, m, B, path):
    """All-ones: the GEMM path's largest sums (n - m = 64536 -> K = 64640 in one accumulator)."""
    raw = np.full(B * n // 8, 0xFF, np.uint8)
    seed = np.full(n // 8, 0xFF, np.uint8)
    assert_same(gpu_mod(q, raw, B, n, m, seed, path), oracle_mod.modified_extract(raw, B, n, m, seed), m)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("cfg", [2, 4])
def test_modified_full_size_sampled(q, oracle_mod, cfg, path):
    """BASELINE configs 2 and 4 with the modified construction (n-bit seed)."""
    w = S.CONFIGS[cfg]
    if path == "gemm" and w.n - w.m > (1 << 16):
        pytest.skip("GEMM path: n - m <= 2^16")
    raw, _ = S.workload_inputs(w)
    seed = S.uniform_bits(w.key, w.n, tag=9)
    got = gpu_mod(q, raw, w.n_blocks, w.n, w.m, seed, path)
    rng = np.random.default_rng(cfg)
    blocks = sorted({0, w.n_blocks - 1, *rng.integers(0, w.n_blocks, 6).tolist()})
    bl, rw = [], []
    for b in blocks:
        rows = np.unique(np.concatenate([[0, w.m - 1], rng.integers(0, w.m, 300)]))
        bl += [b] * rows.size
        rw += rows.tolist()
    bl, rw = np.array(bl, np.uint64), np.array(rw, np.uint64)
    ref = oracle_mod.modified_rows(raw, bl, rw, w.n, w.m, seed)
    assert np.array_equal(np.unpackbits(got)[(bl * w.m + rw).astype(np.int64)], ref)


def test_modified_plan_paths(q, oracle_mod):
    n, m, B = 1024, 716, 6
    raw = S.random_bytes(5, B * n // 8)
    seed = S.random_bytes(5, n // 8, tag=8)
    ref = oracle_mod.modified_extract(raw, B, n, m, seed)
    with q.Plan(n, m, dev(seed), modified=True) as plan:
        assert plan.path == q.PATH_GEMM  # AUTO: n - m far below the crossover
        assert plan.info()["macs_per_block"] == 384 * m  # n - m = 308 rounded up to 3 x 128
        assert_same(plan.extract(dev(raw), B).cpu().numpy(), ref, m)
    q.set_debug_path(q.PATH_NTT)
    try:
        with q.Plan(n, m, dev(seed), modified=True) as plan:
            assert plan.path == q.PATH_NTT
            assert_same(plan.extract(dev(raw), B).cpu().numpy(), ref, m)
    finally:
        q.set_debug_path(q.PATH_AUTO)
    # n - m beyond the tensor-core kernel's 2^16: AUTO takes the NTT, GEMM is refused
    n2, m2 = 140000, 100
    seed2 = dev(S.random_bytes(6, n2 // 8, tag=8))
    with q.Plan(n2, m2, seed2, modified=True) as plan:
        assert plan.path == q.PATH_NTT
    q.set_debug_path(q.PATH_GEMM)
    try:
        with pytest.raises(q.QrngError) as ei:
            q.Plan(n2, m2, seed2, modified=True)
        assert ei.value.status == q.QRNG_E_UNSUPPORTED
    finally:
        q.set_debug_path(q.PATH_AUTO)
