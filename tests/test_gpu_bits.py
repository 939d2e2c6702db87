"""GPU parity of the CUDA-core product (QRNG_PATH_BITS, bits.cu) against the
oracle: forced on random shapes (n % 32 == 0, m below / above / not a multiple
of 32, m = 1, ragged batches), one-shot and through plans; AUTO sends small
batches of dense shapes there and large ones to the tensor cores; the output
needs no pre-zeroing (garbage-filled buffers) and bytes past the key stay
untouched.

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


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint8)).cuda()


def inputs(n, m, B, tag=0):
    raw = S.random_bytes(n * 3 + m + tag, B * n // 8)
    seed = S.random_bytes(n * 3 + m + tag, (n + m - 1 + 7) // 8, tag=13)
    return raw, seed


def shapes(seed, count):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        n = int(rng.integers(1, 96)) * 32
        m = int(rng.choice([1, 2, 31, 32, 33, int(rng.integers(1, n)) if n > 1 else 1, n - 1, (7 * n) // 10]))
        m = max(1, min(m, max(1, n - 1)))
        B = int(rng.integers(1, 300))
        out.append((n, m, B))
    return out


CASES = shapes(7, 40) + [(32, 1, 1), (32, 31, 5), (64, 63, 33), (1024, 716, 256), (4096, 2867, 37), (8192, 5734, 9)]


@pytest.mark.parametrize("n,m,B", CASES, ids=[f"{c[0]}-{c[1]}-{c[2]}" for c in CASES])
def test_forced_bits_oneshot(q, oracle_mod, n, m, B):
    if m >= n:
        pytest.skip("needs m < n")
    raw, seed = inputs(n, m, B)
    ref = oracle_mod.extract(raw, B, n, m, seed)
    q.set_debug_path(q.PATH_BITS)
    try:
        got = q.toeplitz_extract(dev(raw), B, n, m, dev(seed)).cpu().numpy()
        assert q.last_path() == q.PATH_BITS
    finally:
        q.set_debug_path(q.PATH_AUTO)
    assert np.array_equal(got, ref), (n, m, B)


@pytest.mark.parametrize("n,m", [(1024, 716), (96, 50), (2048, 33)])
def test_forced_bits_plan_and_garbage_output(q, oracle_mod, n, m):
    """A forced CUDA-core plan, reused for ragged batches, writing into
    0xA5-filled buffers: every key word is overwritten, nothing past the key."""
    q.set_debug_path(q.PATH_BITS)
    try:
        raw, seed = inputs(n, m, 300, tag=1)
        with q.Plan(n, m, dev(seed)) as plan:
            assert plan.path == q.PATH_BITS
            for B in (1, 7, 300):
                ref = oracle_mod.extract(raw[: B * n // 8], B, n, m, seed)
                nbytes = (B * m + 7) // 8
                out = torch.full((nbytes + 64,), 0xA5, dtype=torch.uint8, device="cuda")
                plan.extract(dev(raw[: B * n // 8]), B, out=out)
                o = out.cpu().numpy()
                assert np.array_equal(o[:nbytes], ref), (n, m, B)
                assert (o[nbytes:] == 0xA5).all()
    finally:
        q.set_debug_path(q.PATH_AUTO)


def test_auto_small_batch_runs_on_cuda_cores(q, oracle_mod):
    """Config 1 (256 blocks of n = 1024) goes to the CUDA cores under AUTO, a
    large batch of the same shape to the tensor cores, through one plan."""
    n, m = 1024, 716
    raw, seed = inputs(n, m, 16384, tag=2)
    with q.Plan(n, m, dev(seed)) as plan:
        assert plan.path == q.PATH_GEMM
        for B, want in ((256, q.PATH_BITS), (16384, q.PATH_GEMM)):
            got = plan.extract(dev(raw[: B * n // 8]), B).cpu().numpy()
            assert q.last_path() == want, (B, q.last_path())
            assert np.array_equal(got, oracle_mod.extract(raw[: B * n // 8], B, n, m, seed)), B
    got = q.toeplitz_extract(dev(raw[: 256 * n // 8]), 256, n, m, dev(seed)).cpu().numpy()
    assert q.last_path() == q.PATH_BITS
    assert np.array_equal(got, oracle_mod.extract(raw[: 256 * n // 8], 256, n, m, seed))


def test_config1_full(q, oracle_mod):
    """BASELINE config 1 end to end (ADC samples, its seed), AUTO."""
    w = S.CONFIGS[1]
    raw_np, seed_np = S.workload_inputs(w)
    got = q.toeplitz_extract(dev(raw_np), w.n_blocks, w.n, w.m, dev(seed_np)).cpu().numpy()
    assert q.last_path() == q.PATH_BITS
    assert np.array_equal(got, oracle_mod.extract(raw_np, w.n_blocks, w.n, w.m, seed_np))


def test_bits_rejects_unsupported(q):
    """A seed longer than the kernel's shared-memory window: E_UNSUPPORTED."""
    n, m = 1 << 21, 1 << 20
    q.set_debug_path(q.PATH_BITS)
    try:
        raw = torch.zeros(n // 8, dtype=torch.uint8, device="cuda")
        seed = torch.zeros((n + m - 1 + 7) // 8, dtype=torch.uint8, device="cuda")
        with pytest.raises(q.QrngError) as e:
            q.toeplitz_extract(raw, 1, n, m, seed)
        assert e.value.status == q.QRNG_E_UNSUPPORTED
    finally:
        q.set_debug_path(q.PATH_AUTO)
