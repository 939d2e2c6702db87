"""Randomised parity sweep: many random (n, m, blocks) shapes -- random
multiples of 32 / 128 for n, random m in [1, n), ragged block counts -- on
every path the scheduler can take (AUTO, forced GEMM with the planner's or a
random Karatsuba depth, forced NTT) plus the modified Toeplitz, each compared
with the CPU oracle on the whole key.  Seeds are fixed, so failures reproduce.

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


def shapes(seed, count, nmax_log, mult):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        n = int(rng.integers(1, (1 << nmax_log) // mult + 1)) * mult
        m = int(rng.integers(1, n)) if n > 1 else 1
        if rng.random() < 0.25:  # near the extremes
            m = int(rng.choice([1, n - 1, (7 * n) // 10]))
        m = max(1, min(m, n - 1))
        B = int(rng.integers(1, max(2, min(300, (1 << 21) // n))))
        out.append((n, m, B))
    return out


CASES = ([("auto", s) for s in shapes(1, 64, 14, 32)] + [("gemm", s) for s in shapes(2, 40, 14, 128)] +
         [("ntt", s) for s in shapes(3, 40, 15, 32)] + [("kara", s) for s in shapes(4, 40, 15, 128)])


@pytest.mark.parametrize("mode,shape", CASES, ids=[f"{c[0]}-{c[1][0]}-{c[1][1]}-{c[1][2]}" for c in CASES])
def test_random_shape(q, oracle_mod, mode, shape):
    n, m, B = shape
    if n < 2:
        pytest.skip("n = 1 has no valid m")
    raw = S.random_bytes(n * 7 + m, B * n // 8)
    seed = S.random_bytes(n * 7 + m, (n + m - 1 + 7) // 8, tag=11)
    ref = oracle_mod.extract(raw, B, n, m, seed)
    try:
        if mode == "gemm":
            q.set_debug_path(q.PATH_GEMM)
        elif mode == "ntt":
            q.set_debug_path(q.PATH_NTT)
        elif mode == "kara":
            q.set_debug_path(q.PATH_GEMM)
            q.set_karatsuba(int(np.random.default_rng(n + m).integers(1, 5)))
        try:
            got = q.toeplitz_extract(dev(raw), B, n, m, dev(seed)).cpu().numpy()
        except q.QrngError as e:
            # forced GEMM with a shape its kernel cannot take is a documented E_UNSUPPORTED
            assert mode in ("gemm", "kara") and e.status == q.QRNG_E_UNSUPPORTED
            return
    finally:
        q.set_debug_path(q.PATH_AUTO)
        q.set_karatsuba(-1)
    assert np.array_equal(got, ref), f"{mode} n={n} m={m} B={B}"


MOD_CASES = shapes(5, 32, 14, 32)


@pytest.mark.parametrize("shape", MOD_CASES, ids=[f"{s[0]}-{s[1]}-{s[2]}" for s in MOD_CASES])
def test_random_shape_modified(q, oracle_mod, shape):
    n, m, B = shape
    B = min(B, 40)
    raw = S.random_bytes(n * 3 + m, B * n // 8)
    seed = S.uniform_bits(n * 3 + m, n, tag=12)
    ref = oracle_mod.modified_extract(raw, B, n, m, seed)
    got = q.modified_toeplitz_extract(dev(raw), B, n, m, dev(seed)).cpu().numpy()
    assert np.array_equal(got, ref), f"modified n={n} m={m} B={B}"
