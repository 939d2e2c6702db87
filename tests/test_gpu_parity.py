"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle,
bit-exact (integer/bit work: zero tolerance), on seeded synthetic inputs.

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


def gpu_extract(q, raw, B, n, m, seed, path=None):
    if path is not None:
        q.set_debug_path(path)
    try:
        out = q.toeplitz_extract(dev(raw), B, n, m, dev(seed))
        torch.cuda.synchronize()
        return out.cpu().numpy()
    finally:
        if path is not None:
            q.set_debug_path(q.PATH_AUTO)


def assert_same(got, ref, m):
    if not np.array_equal(got, ref):
        gb, rb = np.unpackbits(got), np.unpackbits(ref)
        bad = np.nonzero(gb != rb)[0]
        raise AssertionError(f"{bad.size} bits differ; first at bit {bad[0]} "
                             f"(block {bad[0] // m}, i {bad[0] % m})")


PATHS = ["ntt", "gemm", "bits"]  # bits: the CUDA-core product AUTO uses for small batches


def path_id(q, name):
    return {"ntt": q.PATH_NTT, "gemm": q.PATH_GEMM, "bits": q.PATH_BITS}[name]


SMALL_CASES = [
    (32, 1, 1), (32, 31, 3), (64, 7, 5), (96, 50, 7), (128, 127, 2), (256, 200, 9),
    (512, 300, 33), (1024, 716, 17), (1024, 1, 4), (2048, 1433, 10), (4096, 2867, 5),
    (8192, 5734, 7), (16384, 11468, 3), (16384, 16383, 2), (12288, 8000, 5),
    # odd multiples of 128: the E2M1 kernel's last 256-K stage is half zero-filled
    (384, 300, 7), (1152, 806, 9), (2432, 1702, 5), (65408, 45785, 2),
]


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("n,m,B", SMALL_CASES)
def test_random_small(q, oracle_mod, path, n, m, B):
    if path == "gemm" and n % 128:
        pytest.skip("GEMM path needs n % 128 == 0")
    key = n * 7919 + m
    raw = S.random_bytes(key, B * n // 8)
    seed = S.random_bytes(key, (n + m - 1 + 7) // 8, tag=2)
    ref = oracle_mod.extract(raw, B, n, m, seed)
    assert_same(gpu_extract(q, raw, B, n, m, seed, path_id(q, path)), ref, m)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("n,m,B", [(1024, 716, 3), (8192, 5734, 3), (16384, 11468, 2), (96, 95, 5), (1152, 806, 3)])
def test_all_ones_max_window(q, oracle_mod, path, n, m, B):
    if path == "gemm" and n % 128:
        pytest.skip("GEMM path needs n % 128 == 0")
    """Every window sum equals n (the maximum): exercises p > n and the
    two-blocks-per-transform separation at its worst case."""
    raw = np.full(B * n // 8, 0xFF, np.uint8)
    seed = np.full((n + m - 1 + 7) // 8, 0xFF, np.uint8)
    ref = oracle_mod.extract(raw, B, n, m, seed)
    assert_same(gpu_extract(q, raw, B, n, m, seed, path_id(q, path)), ref, m)
    alt = np.full(B * n // 8, 0xAA, np.uint8)
    assert_same(gpu_extract(q, alt, B, n, m, seed, path_id(q, path)),
                oracle_mod.extract(alt, B, n, m, seed), m)


@pytest.mark.parametrize("cfg", [1, 2])
def test_config_full(q, oracle_mod, cfg):
    """BASELINE configs 1 and 2, every block, through the AUTO path (the launch
    configuration bench.py times) and through each forced path."""
    w = S.CONFIGS[cfg]
    raw, seed = S.workload_inputs(w)
    ref = oracle_mod.extract(raw, w.n_blocks, w.n, w.m, seed)
    assert_same(gpu_extract(q, raw, w.n_blocks, w.n, w.m, seed), ref, w.m)
    for p in PATHS:
        assert_same(gpu_extract(q, raw, w.n_blocks, w.n, w.m, seed, path_id(q, p)), ref, w.m)


@pytest.mark.parametrize("N,K", [(192, 128), (64, 256), (256, 1024), (16, 128)])
def test_umma_probe_layouts(q, N, K):
    """tcgen05 kind::i8 with A in TMEM and the overlapping core-matrix B
    descriptor (SBO 128 B, LBO 256 B) against an int64 numpy matmul."""
    rng = np.random.default_rng(N * 1000 + K)
    for A in (rng.integers(0, 2, (128, K)), rng.integers(0, 256, (128, K))):
        h = rng.integers(0, 256, N + K).astype(np.uint8)
        B = np.array([[h[i + k] for k in range(K)] for i in range(N)], np.int64)
        D = q.umma_probe(dev(A.astype(np.uint8)), dev(h), N, K).cpu().numpy()
        assert np.array_equal(D.astype(np.int64), A.astype(np.int64) @ B.T)


def test_plan_reuse_and_block_slices(q, oracle_mod):
    w = S.CONFIGS[1]
    raw, seed = S.workload_inputs(w)
    ref = oracle_mod.extract(raw, w.n_blocks, w.n, w.m, seed)
    with q.Plan(w.n, w.m, dev(seed)) as plan:
        assert plan.path == q.PATH_GEMM  # AUTO below the measured crossover
        draw = dev(raw)
        for _ in range(2):
            out = plan.extract(draw, w.n_blocks).cpu().numpy()
            assert_same(out, ref, w.m)
        # a shard of 32 blocks starting at block 64 is word aligned (32*m % 32 == 0)
        sub = plan.extract(draw[64 * w.n // 8:96 * w.n // 8], 32).cpu().numpy()
        assert np.array_equal(sub, ref[64 * w.m // 8:96 * w.m // 8])


def test_host_buffers_api(q, oracle_mod):
    w = S.CONFIGS[1]
    raw, seed = S.workload_inputs(w, 0, 40)
    out = np.zeros(q.out_bytes(40, w.m), np.uint8)
    q.toeplitz_extract_host(raw, 40, w.n, w.m, seed, out)
    assert_same(out, oracle_mod.extract(raw, 40, w.n, w.m, seed), w.m)


def test_partial_tail_word_and_pad_bits(q, oracle_mod):
    n, m, B = 64, 13, 3  # 39 output bits: 5 bytes, final 32-bit word partial
    raw = S.random_bytes(5, B * n // 8)
    seed = S.random_bytes(5, (n + m - 1 + 7) // 8, tag=3)
    ref = oracle_mod.extract(raw, B, n, m, seed)
    d_out = torch.full((16,), 0xEE, dtype=torch.uint8, device="cuda")
    q.toeplitz_extract(dev(raw), B, n, m, dev(seed), out=d_out[:5])
    got = d_out.cpu().numpy()
    assert np.array_equal(got[:5], ref)
    assert (got[5:] == 0xEE).all()  # nothing written past ceil(B*m/8)


def test_rejects_misaligned_and_overlap(q):
    buf = torch.zeros(4096, dtype=torch.uint8, device="cuda")
    seed = torch.zeros(256, dtype=torch.uint8, device="cuda")  # L = 1739 bits fit
    with pytest.raises(q.QrngError) as ei:
        q.toeplitz_extract(buf[1:129], 1, 1024, 716, seed, out=buf[1024:1200])
    assert ei.value.status == q.QRNG_E_INVALID
    with pytest.raises(q.QrngError) as ei:
        q.toeplitz_extract(buf[:128], 1, 1024, 716, seed, out=buf[64:256])
    assert ei.value.status == q.QRNG_E_INVALID


@pytest.mark.parametrize("cfg", [1, 2])
def test_minentropy_matches_oracle(q, cfg):
    from oracle import entropy as E
    import oracle
    w = S.CONFIGS[cfg]
    raw, _ = S.workload_inputs(w)
    rep = q.minentropy(dev(raw), 8, w.n, 0)
    assert np.array_equal(rep.counts, oracle.hist256(raw))
    ref = E.report(raw, 8, w.n, 0)
    for f in ("mu", "sigma", "h_min_hist", "h_min_ideal", "stat_dist", "delta_h_m", "h_min_mod"):
        assert getattr(rep, f) == pytest.approx(getattr(ref, f), rel=1e-12, abs=1e-12), f
    assert rep.m == ref.m


def test_hist_sharded_accumulate(q):
    import oracle
    x = S.adc_samples(9, (1 << 20) + 13, 128, 12)
    counts = torch.zeros(256, dtype=torch.int64, device="cuda")
    half = x.size // 2
    q.hist256_async(dev(x[:half]), counts)
    q.hist256_async(dev(x[half:]), counts)
    assert np.array_equal(counts.cpu().numpy().astype(np.uint64), oracle.hist256(x))


# ---- multi-pass NTT (P > 2^15) and full-size configurations -----------------------

@pytest.mark.parametrize("n,m,B", [(32768, 22937, 3), (49152, 30000, 2), (65536, 45875, 3),
                                   (131072, 91750, 2), (65536, 1, 2), (65536, 65535, 1)])
def test_multipass_random(q, oracle_mod, n, m, B):
    key = n * 31 + m
    raw = S.random_bytes(key, B * n // 8)
    seed = S.random_bytes(key, (n + m - 1 + 7) // 8, tag=2)
    ref = oracle_mod.extract(raw, B, n, m, seed)
    assert_same(gpu_extract(q, raw, B, n, m, seed, q.PATH_NTT), ref, m)


def test_multipass_all_ones(q, oracle_mod):
    n, m, B = 131072, 91750, 2  # window sums reach n: p > n at P = 2^18
    raw = np.full(B * n // 8, 0xFF, np.uint8)
    seed = np.full((n + m - 1 + 7) // 8, 0xFF, np.uint8)
    assert_same(gpu_extract(q, raw, B, n, m, seed, q.PATH_NTT), oracle_mod.extract(raw, B, n, m, seed), m)


def sampled_check(oracle_mod, got, raw, seed, n, m, B, n_rows=256, key=0):
    """Sampled outputs at full size: first/last/middle/random blocks, random rows
    plus the first and last rows of each block, against the oracle one by one."""
    rng = np.random.default_rng(key)
    blocks = sorted({0, B - 1, B // 2, *rng.integers(0, B, 5).tolist()})
    bl, rw = [], []
    for b in blocks:
        rows = np.unique(np.concatenate([[0, 1, m - 2, m - 1], rng.integers(0, m, n_rows)]))
        bl += [b] * rows.size
        rw += rows.tolist()
    bl, rw = np.array(bl, np.uint64), np.array(rw, np.uint64)
    ref = oracle_mod.extract_rows(raw, bl, rw, n, m, seed)
    bits = np.unpackbits(got)
    gb = bits[(bl * m + rw).astype(np.int64)]
    bad = np.nonzero(gb != ref)[0]
    assert bad.size == 0, f"{bad.size} sampled bits differ, first (block {bl[bad[0]]}, row {rw[bad[0]]})"
    # pad bits of the last byte
    tail = B * m % 8
    if tail:
        assert got[-1] & ((1 << (8 - tail)) - 1) == 0


@pytest.mark.parametrize("cfg", [3, 4])
def test_config_full_size_sampled(q, oracle_mod, cfg):
    """Configs 3 and 4 at full size through AUTO (what bench.py times), sampled
    outputs vs the oracle, plus two complete blocks."""
    w = S.CONFIGS[cfg]
    raw, seed = S.workload_inputs(w)
    got = gpu_extract(q, raw, w.n_blocks, w.n, w.m, seed)
    sampled_check(oracle_mod, got, raw, seed, w.n, w.m, w.n_blocks, key=cfg)
    for b in (0, w.n_blocks - 1):
        ref = oracle_mod.extract_blocks(raw, [b], w.n, w.m, seed)[0]
        gbits = np.unpackbits(got)[b * w.m:(b + 1) * w.m]
        assert np.array_equal(gbits, np.unpackbits(ref)[:w.m]), b


def test_sweep_max_n_sampled(q, oracle_mod):
    """Config 5's largest point n = 2^22 (P = 2^23, two global passes), 32 blocks."""
    w = S.sweep_workload(22)
    B = 32
    raw, seed = S.workload_inputs(w, 0, B)
    got = gpu_extract(q, raw, B, w.n, w.m, seed)
    sampled_check(oracle_mod, got, raw, seed, w.n, w.m, B, n_rows=128, key=22)


@pytest.mark.parametrize("log2n,B", [(10, 1024), (12, 512), (14, 256), (16, 64)])
def test_gemm_equals_ntt_all_blocks(q, log2n, B):
    """P10: the two independent GPU paths agree bit for bit on every block."""
    w = S.sweep_workload(log2n)
    raw, seed = S.workload_inputs(w, 0, B)
    a = gpu_extract(q, raw, B, w.n, w.m, seed, q.PATH_GEMM)
    b = gpu_extract(q, raw, B, w.n, w.m, seed, q.PATH_NTT)
    assert_same(a, b, w.m)


@pytest.mark.parametrize("n,m,B", [(1024, 179, 100), (8192, 5734, 333), (2048, 1, 65), (96, 50, 70)])
def test_host_buffers_pipelined_chunks(q, oracle_mod, n, m, B):
    """qrng_toeplitz_extract_host splits the batch into 32-block-granule chunks
    (H2D / kernel / D2H overlapped on three streams); odd m and ragged tails."""
    raw = S.random_bytes(n + B, B * n // 8)
    seed = S.random_bytes(n + B, (n + m - 1 + 7) // 8, tag=4)
    out = np.full(q.out_bytes(B, m) + 8, 0xA5, np.uint8)
    q.toeplitz_extract_host(raw, B, n, m, seed, out)
    assert_same(out[:q.out_bytes(B, m)], oracle_mod.extract(raw, B, n, m, seed), m)
    assert (out[q.out_bytes(B, m):] == 0xA5).all()


def test_config4b_m_from_minentropy(q, oracle_mod):
    """Config 4b (reading A8): m from qrng_minentropy on config 4's samples
    (s = 0) equals the oracle's; the extraction with that m is bit-exact on
    sampled outputs and on one complete block."""
    from oracle import entropy as E
    w4 = S.CONFIGS[4]
    raw, _ = S.workload_inputs(w4)
    rep = q.minentropy(dev(raw), 8, w4.n, 0)
    ref = E.report(raw, 8, w4.n, 0)
    assert rep.m == ref.m and 0 < rep.m < w4.m
    w = S.config4b(rep.m)
    raw, seed = S.workload_inputs(w)
    assert seed.size == (w4.n + rep.m - 1 + 7) // 8
    got = gpu_extract(q, raw, w.n_blocks, w.n, w.m, seed)
    sampled_check(oracle_mod, got, raw, seed, w.n, w.m, w.n_blocks, key=41)
    blk = oracle_mod.extract_blocks(raw, [7], w.n, w.m, seed)[0]
    assert np.array_equal(np.unpackbits(got)[7 * w.m:8 * w.m], np.unpackbits(blk)[:w.m])


def test_one_plan_two_streams_concurrently(q, oracle_mod):
    """The header allows one plan on several streams at once: two batches with a
    partial final word each, launched back to back on two streams."""
    n, m = 1024, 179
    seed = S.random_bytes(77, (n + m - 1 + 7) // 8, tag=2)
    raws = [S.random_bytes(78 + k, B * n // 8) for k, B in enumerate((33, 45))]
    refs = [oracle_mod.extract(r, len(r) * 8 // n, n, m, seed) for r in raws]
    for path in (q.PATH_GEMM, q.PATH_NTT):
        q.set_debug_path(path)
        try:
            with q.Plan(n, m, dev(seed)) as plan:
                streams = [torch.cuda.Stream(), torch.cuda.Stream()]
                outs = []
                for r, st in zip(raws, streams):
                    with torch.cuda.stream(st):
                        d = dev(r)
                        outs.append(plan.extract(d, len(r) * 8 // n, stream=st))
                torch.cuda.synchronize()
                for o, ref in zip(outs, refs):
                    assert_same(o.cpu().numpy(), ref, m)
        finally:
            q.set_debug_path(q.PATH_AUTO)


def test_max_seed_length_2_23(q, oracle_mod):
    """L = n + m - 1 = 2^23 exactly: the largest transform (P = 2^23, the 2-adic
    limit of p = 119*2^23 + 1); one bit more moves to the world-1 four-step
    NTT modulo 7*2^26 + 1 (P = 2^24), also bit-exact."""
    n = 5033152  # multiple of 32
    m = (1 << 23) + 1 - n
    B = 2
    raw = S.random_bytes(123, B * n // 8)
    seed = S.random_bytes(123, (n + m - 1 + 7) // 8, tag=3)
    got = gpu_extract(q, raw, B, n, m, seed)
    sampled_check(oracle_mod, got, raw, seed, n, m, B, n_rows=200, key=23)
    seed2 = S.random_bytes(124, (n + m + 7) // 8, tag=3)
    got2 = gpu_extract(q, raw, B, n, m + 1, seed2)
    sampled_check(oracle_mod, got2, raw, seed2, n, m + 1, B, n_rows=200, key=24)


@pytest.mark.parametrize("path", PATHS)
def test_zero_seed_and_zero_raw(q, oracle_mod, path):
    n, m, B = 1024, 716, 40
    raw = S.random_bytes(9, B * n // 8)
    zero_seed = np.zeros((n + m - 1 + 7) // 8, np.uint8)
    assert not gpu_extract(q, raw, B, n, m, zero_seed, path_id(q, path)).any()
    seed = S.random_bytes(9, (n + m - 1 + 7) // 8, tag=2)
    assert not gpu_extract(q, np.zeros_like(raw), B, n, m, seed, path_id(q, path)).any()


@pytest.mark.parametrize("n,m,path", [(1024, 179, "gemm"), (8192, 5734, "gemm"), (2048, 1433, "ntt"),
                                      (131072, 91750, "ntt")])
def test_stream_batches_and_histogram(q, oracle_mod, n, m, path):
    """qrng_stream_*: several host batches of different sizes (ragged, partial
    final words) with three in flight; every key bit-exact, and the streamed
    histogram equals the oracle's over all submitted bytes."""
    seed = S.random_bytes(n + 5, (n + m - 1 + 7) // 8, tag=6)
    sizes = [37, 64, 5, 40, 1] if n < 65536 else [3, 2, 1, 2]
    q.set_debug_path(path_id(q, path))
    try:
        with q.Plan(n, m, dev(seed)) as plan, q.Stream(plan, max(sizes), depth=3, hist=True) as st:
            raws = [S.random_bytes(n * 31 + k, B * n // 8) for k, B in enumerate(sizes)]
            outs = [np.full(q.out_bytes(B, m) + 4, 0xC3, np.uint8) for B in sizes]
            for r, o, B in zip(raws, outs, sizes):
                st.submit(r, B, o)
            st.synchronize()
            for r, o, B in zip(raws, outs, sizes):
                assert_same(o[:q.out_bytes(B, m)], oracle_mod.extract(r, B, n, m, seed), m)
                assert (o[q.out_bytes(B, m):] == 0xC3).all()
            assert np.array_equal(st.counts(), oracle_mod.hist256(np.concatenate(raws)))
    finally:
        q.set_debug_path(q.PATH_AUTO)
