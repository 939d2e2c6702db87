"""GPU edge cases through the C ABI, each against the CPU oracle (bit-exact):

* the packed-accumulator branch of the grouped tcgen05 kernel driven at its
  maximum (N tile 1 sum S1 = 2048 = w, so F = S0 + 2^12 S1 >= 2^23) with an
  ODD low half S0 (gemm_tc.cu packed epilogue; DESIGN.md 6.1 "Packed
  accumulators") -- the one input class that would expose a dropped low bit
  at maximum magnitude;
* AUTO on shapes the Karatsuba planner leaves undecomposed at n > 2^16
  (small m) runs on the NTT path instead of failing;
* the histogram on unaligned sample slices (shard slices samples[lo:hi]);
* the modified Toeplitz with m close to n (seed window larger than the
  tensor-core kernel's shared memory) through AUTO;
* more distinct Karatsuba shapes than the table cache holds, with the first
  plan still extracting correctly after its tables were evicted;
* binding-level size and device checks (short buffers never reach the C ABI).

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


def assert_same(got, ref, m):
    if not np.array_equal(got, ref):
        gb, rb = np.unpackbits(got), np.unpackbits(ref)
        bad = np.nonzero(gb != rb)[0]
        raise AssertionError(f"{bad.size} bits differ; first at bit {bad[0]} "
                             f"(block {bad[0] // m}, i {bad[0] % m})")


def bits_to_bytes(bits):
    return np.packbits(np.asarray(bits, np.uint8))


# ---- packed accumulators at S1 = 2048 with odd S0 ---------------------------------

def adversarial_packed_inputs(B=256):
    """n = 4096, m = 2867 at Karatsuba depth 1: leaf 0 is Q = A (x0 ^ x1), a
    2048 x 2048 Toeplitz product whose seed is d[k] = s[2048 + k] (the host
    planner's table says so; checked below).  Seed: all ones except d[k] = 0
    for odd k < 224.  Blocks with x0 = 1^2048, x1 = 0^2048 feed Q an all-ones
    input, so row i of Q sums S(i) = 2048 - #{odd k in [i, 224)}: every row
    >= 224 (every N tile 1 row of the kernel's 448-row pairs) sums to 2048,
    rows < 224 alternate between odd and even sums."""
    n, m, h = 4096, 2867, 2048
    L = n + m - 1
    s = np.ones(L, np.uint8)
    s[h + np.arange(1, 224, 2)] = 0
    rng = np.random.default_rng(77)
    X = np.zeros((B, n), np.uint8)
    X[:, :h] = 1                        # x0 = ones, x1 = zeros -> x0 ^ x1 = ones
    X[1::4, h:] = 1                     # x0 = x1 = ones -> Q input zero, P2/P3 inputs ones
    X[2::4] = rng.integers(0, 2, (len(X[2::4]), n))   # random blocks in the same M tiles
    return n, m, h, s, X


def test_adversarial_packed_accumulator(q, oracle_mod):
    n, m, h, s, X = adversarial_packed_inputs()
    B = X.shape[0]
    raw, seed = bits_to_bytes(X.reshape(-1)), bits_to_bytes(s)
    ref = oracle_mod.extract(raw, B, n, m, seed)
    q.set_debug_path(q.PATH_GEMM)
    q.set_karatsuba(1)
    try:
        with q.Plan(n, m, dev(seed)) as plan:
            assert plan.info()["karatsuba_depth"] == 1
            got = plan.extract(dev(raw), B).cpu().numpy()
    finally:
        q.set_debug_path(q.PATH_AUTO)
        q.set_karatsuba(-1)
    assert_same(got, ref, m)
    # AUTO (what the bench runs) on the same inputs
    got2 = q.toeplitz_extract(dev(raw), B, n, m, dev(seed)).cpu().numpy()
    assert_same(got2, ref, m)


# ---- AUTO falls back to the NTT path for undecomposed large-n shapes ------------------

@pytest.mark.parametrize("n,m,B", [(131072, 1000, 8), (262144, 4000, 4), (131072, 1, 3)])
def test_auto_small_m_large_n(q, oracle_mod, n, m, B):
    raw = S.random_bytes(n + m, B * n // 8)
    seed = S.random_bytes(n + m, (n + m - 1 + 7) // 8, tag=5)
    with q.Plan(n, m, dev(seed)) as plan:
        path = plan.path
        got = plan.extract(dev(raw), B).cpu().numpy()
    assert path in (q.PATH_GEMM, q.PATH_NTT)
    assert_same(got, oracle_mod.extract(raw, B, n, m, seed), m)


# ---- histogram on unaligned slices ----------------------------------------------------

@pytest.mark.parametrize("lo,hi", [(1, 100), (3, 1 << 16), (15, (1 << 20) + 7), (17, 18), (5, 21)])
def test_hist_unaligned_slices(q, oracle_mod, lo, hi):
    x = S.adc_samples(42, (1 << 20) + 64)
    d = dev(x)
    counts = torch.zeros(256, dtype=torch.int64, device="cuda")
    q.hist256_async(d[lo:hi], counts)
    assert np.array_equal(counts.cpu().numpy().astype(np.uint64), oracle_mod.hist256(x[lo:hi]))
    if hi - lo >= 1000:  # (a fitted sigma needs more than a handful of samples)
        rep = q.minentropy(d[lo:hi], 8, 1024, 0, allow_no_output=True)
        assert np.array_equal(rep.counts, oracle_mod.hist256(x[lo:hi]))


# ---- modified Toeplitz with m close to n ------------------------------------------------

def test_modified_m_close_to_n(q, oracle_mod):
    n, m, B = 1 << 20, 1000000, 2
    raw = S.random_bytes(5, B * n // 8)
    seed = S.uniform_bits(5, n, tag=9)
    got = q.modified_toeplitz_extract(dev(raw), B, n, m, dev(seed)).cpu().numpy()
    rng = np.random.default_rng(5)
    bl = np.repeat(np.arange(B), 300).astype(np.uint64)
    rw = np.concatenate([np.r_[0, 1, m - 2, m - 1, rng.integers(0, m, 296)] for _ in range(B)]).astype(np.uint64)
    ref = oracle_mod.modified_rows(raw, bl, rw, n, m, seed)
    assert np.array_equal(np.unpackbits(got)[(bl * m + rw).astype(np.int64)], ref)
    # forced GEMM: the seed window does not fit the kernel's shared memory
    q.set_debug_path(q.PATH_GEMM)
    try:
        with pytest.raises(q.QrngError) as ei:
            q.modified_toeplitz_extract(dev(raw), B, n, m, dev(seed))
        assert ei.value.status == q.QRNG_E_UNSUPPORTED
    finally:
        q.set_debug_path(q.PATH_AUTO)


# ---- Karatsuba table cache eviction ------------------------------------------------------

def test_table_cache_eviction_keeps_live_plans(q, oracle_mod):
    n, B = 8192, 40
    raw = S.random_bytes(8, B * n // 8)
    seed = S.random_bytes(8, (2 * n) // 8, tag=2)
    first = q.Plan(n, 5734, dev(seed))
    assert first.info()["karatsuba_depth"] > 0
    # 20 more distinct (n, m) shapes than the cache's 16 entries
    for m in range(4000, 4000 + 20 * 37, 37):
        with q.Plan(n, m, dev(seed)) as p:
            got = p.extract(dev(raw), B).cpu().numpy()
        if m % 3 == 0:
            assert_same(got, oracle_mod.extract(raw, B, n, m, seed), m)
    got = first.extract(dev(raw), B).cpu().numpy()
    first.close()
    assert_same(got, oracle_mod.extract(raw, B, n, 5734, seed), 5734)


# ---- binding checks ------------------------------------------------------------------------

def test_binding_rejects_short_buffers(q):
    n, m, B = 1024, 716, 8
    raw = torch.zeros(B * n // 8, dtype=torch.uint8, device="cuda")
    seed = torch.zeros((n + m - 1 + 7) // 8, dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):
        q.toeplitz_extract(raw[:-1], B, n, m, seed)
    with pytest.raises(ValueError):
        q.toeplitz_extract(raw, B, n, m, seed[:-1])
    with pytest.raises(ValueError):
        q.toeplitz_extract(raw, B, n, m, seed, out=torch.zeros(q.out_bytes(B, m) - 1, dtype=torch.uint8,
                                                                device="cuda"))
    with q.Plan(n, m, seed) as p:
        with pytest.raises(ValueError):
            p.extract(raw, B + 1)
    with pytest.raises(ValueError):
        q.modified_toeplitz_extract(raw, B, n, m, seed[:n // 8 - 1])
