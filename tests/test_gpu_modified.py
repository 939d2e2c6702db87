"""GPU parity of the modified Toeplitz [T | I_m] (SURVEY
NEXT-1) against the oracle: bit-exact, fused (P <= 2^15, incl. two blocks per
transform) and multi-pass NTT, full-size configs on sampled outputs."""
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


def gpu_mod(q, raw, B, n, m, seed):
    out = q.modified_toeplitz_extract(dev(raw), B, n, m, dev(seed))
    torch.cuda.synchronize()
    return out.cpu().numpy()


def assert_same(got, ref, m):
    if not np.array_equal(got, ref):
        bad = np.nonzero(np.unpackbits(got) != np.unpackbits(ref))[0]
        raise AssertionError(f"{bad.size} bits differ; first at block {bad[0] // m}, row {bad[0] % m}")


@pytest.mark.parametrize("n,m,B", [
    (32, 1, 3), (64, 20, 5), (96, 95, 4), (1024, 716, 9), (1024, 300, 7), (8192, 5734, 5),
    (8192, 2000, 4), (16384, 11468, 3), (32768, 22937, 2), (65536, 45875, 2), (65536, 10000, 2),
])
def test_modified_random(q, oracle_mod, n, m, B):
    raw = S.random_bytes(n + 3 * m, B * n // 8)
    seed = S.random_bytes(n + 3 * m, n // 8, tag=7)
    if n * m * B <= 2e8:
        ref = oracle_mod.modified_extract(raw, B, n, m, seed)
        assert_same(gpu_mod(q, raw, B, n, m, seed), ref, m)
    else:
        got = gpu_mod(q, raw, B, n, m, seed)
        bl = np.repeat(np.arange(B), m)
        rw = np.tile(np.arange(m), B)
        ref = oracle_mod.modified_rows(raw, bl, rw, n, m, seed)
        assert np.array_equal(np.unpackbits(got)[:B * m], ref)


def test_modified_all_ones(q, oracle_mod):
    n, m, B = 8192, 5734, 3
    raw = np.full(B * n // 8, 0xFF, np.uint8)
    seed = np.full(n // 8, 0xFF, np.uint8)
    assert_same(gpu_mod(q, raw, B, n, m, seed), oracle_mod.modified_extract(raw, B, n, m, seed), m)


@pytest.mark.parametrize("cfg", [2, 4])
def test_modified_full_size_sampled(q, oracle_mod, cfg):
    """BASELINE configs 2 and 4 with the modified construction (n-bit seed)."""
    w = S.CONFIGS[cfg]
    raw, _ = S.workload_inputs(w)
    seed = S.uniform_bits(w.key, w.n, tag=9)
    got = gpu_mod(q, raw, w.n_blocks, w.n, w.m, seed)
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


def test_modified_plan_and_rejects_gemm(q, oracle_mod):
    n, m, B = 1024, 716, 6
    raw = S.random_bytes(5, B * n // 8)
    seed = S.random_bytes(5, n // 8, tag=8)
    ref = oracle_mod.modified_extract(raw, B, n, m, seed)
    with q.Plan(n, m, dev(seed), modified=True) as plan:
        assert plan.path == q.PATH_NTT
        assert_same(plan.extract(dev(raw), B).cpu().numpy(), ref, m)
    q.set_debug_path(q.PATH_GEMM)
    try:
        with pytest.raises(q.QrngError) as ei:
            q.modified_toeplitz_extract(dev(raw), B, n, m, dev(seed))
        assert ei.value.status == q.QRNG_E_UNSUPPORTED
    finally:
        q.set_debug_path(q.PATH_AUTO)
