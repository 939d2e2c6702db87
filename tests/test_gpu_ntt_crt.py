"""GPU parity of the NTT path's packed three-prime form (ntt.cu, round 2).

Multi-pass NTT plans with n < 2^21 put G = 4 blocks into one transform per
prime as v = sum_g 2^(k g) x_g (k = bit length of n) and recover each block's
window sums from the CRT value (DESIGN.md 6.3 "Packed three-prime form").  The
exactness argument needs every window sum below 2^k and n sum_g 2^(k g) below
kP kP2 kP3; these tests drive both to their limits and check the grouping
(ragged last groups, single blocks) against the CPU oracle, bit-exact.
"""
import numpy as np
import pytest

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
    q.set_debug_path(q.PATH_NTT)
    yield q
    q.set_debug_path(q.PATH_AUTO)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint8)).cuda()


def run(q, raw, B, n, m, seed):
    out = q.toeplitz_extract(dev(raw), B, n, m, dev(seed))
    torch.cuda.synchronize()
    return out.cpu().numpy()


def plan_form(q, n, m, seed):
    with q.Plan(n, m, dev(seed)) as pl:
        return pl.info()


@pytest.mark.parametrize("n,m,B", [(65536, 45875, 1), (65536, 45875, 3), (65536, 45875, 5), (65536, 45875, 8),
                                   (40960, 30001, 7), (98304, 1, 6), (65536, 65535 - 32, 9), (131072, 90000, 4)])
def test_packed_form_whole_blocks(q, oracle_mod, n, m, B):
    rng = np.random.default_rng(n + 3 * m + B)
    raw = rng.integers(0, 256, B * n // 8, dtype=np.uint8)
    seed = rng.integers(0, 256, (n + m - 1 + 7) // 8, dtype=np.uint8)
    info = plan_form(q, n, m, seed)
    assert info["path"] == q.PATH_NTT and info["log2_transform"] > 15
    assert (info["blocks_per_transform"], info["primes"]) == (4, 3), info
    got = run(q, raw, B, n, m, seed)
    ref = oracle_mod.extract(raw, B, n, m, seed)
    assert np.array_equal(got, ref)


def test_packed_form_max_window_sums(q, oracle_mod):
    # seed all ones: every window of s covers all of x, so y_i = popcount(x_b)
    # mod 2 and every window sum equals popcount(x_b) <= n -- the top of each
    # block's k-bit field.  Block b clears b bits, so the four fields of a
    # group hold n, n - 1, n - 2, n - 3 (distinct parities, v near n 2^(3k)).
    n, m, B = 1 << 20, 1000, 8
    raw = np.full(B * n // 8, 0xFF, np.uint8)
    for b in range(B):
        for j in range(b % 4):
            raw[b * n // 8 + 17 * j] &= 0xFE
    seed = np.full((n + m - 1 + 7) // 8, 0xFF, np.uint8)
    info = plan_form(q, n, m, seed)
    assert (info["blocks_per_transform"], info["primes"]) == (4, 3), info
    got = np.unpackbits(run(q, raw, B, n, m, seed))[:B * m].reshape(B, m)
    for b in range(B):
        assert (got[b] == (b % 4) % 2).all(), f"block {b}"
    ref = np.unpackbits(oracle_mod.extract(raw, B, n, m, seed))[:B * m].reshape(B, m)
    assert np.array_equal(got, ref)


def test_packed_form_config4_sampled(q, oracle_mod):
    # config 4's shape (n = 2^20, m = 734,003) on 6 blocks (a ragged second
    # group), 200 sampled rows per block against the oracle's row form
    import qrng_synth as S
    w = S.CONFIGS[4]
    B = 6
    raw_all, seed = S.workload_inputs(w)
    raw = raw_all[:B * w.n // 8]
    got = np.unpackbits(run(q, raw, B, w.n, w.m, seed))[:B * w.m].reshape(B, w.m)
    rng = np.random.default_rng(4)
    rows = np.concatenate([[0, 1, w.m - 1], rng.integers(0, w.m, 197)]).astype(np.uint64)
    blocks = np.repeat(np.arange(B, dtype=np.uint64), rows.size)
    ref = oracle_mod.extract_rows(raw, blocks, np.tile(rows, B), w.n, w.m, seed)
    assert np.array_equal(got[blocks.astype(int), np.tile(rows, B).astype(int)], ref)


@pytest.mark.parametrize("n,m,B", [(131072, 50000, 5), (1 << 20, 734003, 2)])
def test_packed_form_modified_toeplitz(q, oracle_mod, n, m, B):
    # [T | I_m] (reading A24): the product of the first n - m bits, then the
    # CRT pass XORs raw bit t + 1 of each block of the group; every block's
    # first / last rows and 300 random rows against the oracle's row form
    rng = np.random.default_rng(n + m)
    raw = rng.integers(0, 256, B * n // 8, dtype=np.uint8)
    seed = rng.integers(0, 256, n // 8, dtype=np.uint8)
    with q.Plan(n, m, dev(seed), modified=True) as pl:
        info = pl.info()
        got = pl.extract(dev(raw), B).cpu().numpy()
    assert info["path"] == q.PATH_NTT and (info["blocks_per_transform"], info["primes"]) == (4, 3), info
    bits = np.unpackbits(got)[:B * m].reshape(B, m)
    rows = np.concatenate([[0, 1, m - 2, m - 1], rng.integers(0, m, 300)]).astype(np.uint64)
    bl = np.repeat(np.arange(B, dtype=np.uint64), rows.size)
    rw = np.tile(rows, B)
    ref = oracle_mod.modified_rows(raw, bl, rw, n, m, seed)
    assert np.array_equal(bits[bl.astype(int), rw.astype(int)], ref)


def test_small_transform_keeps_one_prime(q):
    # P = 2^16 measured slower packed: one block per transform
    n, m = 65536, 1
    seed = np.random.default_rng(6).integers(0, 256, (n + m - 1 + 7) // 8, dtype=np.uint8)
    info = plan_form(q, n, m, seed)
    assert info["log2_transform"] == 16 and info["blocks_per_transform"] == 1, info


def test_one_prime_form_above_2_20(q, oracle_mod):
    # n >= 2^21: the k-bit fields no longer fit four blocks under 2^64 / M, so
    # the plan keeps one block per transform
    n, m = 1 << 21, 1000
    seed = np.random.default_rng(5).integers(0, 256, (n + m - 1 + 7) // 8, dtype=np.uint8)
    info = plan_form(q, n, m, seed)
    assert info["blocks_per_transform"] == 1 and info["primes"] == 1, info
