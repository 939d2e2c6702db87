"""Pins for the extraction oracle (oracle/toeplitz_oracle.c) -- CPU only.

Each check ties the oracle to something other than itself: the paper's worked
values / hand-checked fixtures, textbook library routines (np.convolve,
scipy.linalg.toeplitz, Python carry-less integer products), the paper's own
float-FFT method (Listing 2 with the prose window), closed forms and
invariants (BASELINE.json north_star: brute force n <= 16, GF(2) linearity,
Toeplitz shift structure).  A dropped term, wrong sign/index or transposed
operand in the oracle fails at least one of them.
"""
import json
import os

import numpy as np
import pytest
import scipy.linalg

from conftest import GOLDEN
import qrng_synth


def bits_of(buf, count, off=0):
    return np.unpackbits(np.asarray(buf, np.uint8))[off:off + count]


def pack(bits):
    return np.packbits(np.asarray(bits, np.uint8))


def toeplitz_matrix(seed_bits, n, m):
    """T from the paper's displayed matrix: first column
    (a_n, a_{n+1}, ..., a_{n+m-1}) = s[n-1 .. n+m-2], first row
    (a_n, a_{n-1}, ..., a_1) = s[n-1], s[n-2], ..., s[0]; built by scipy."""
    s = np.asarray(seed_bits, np.int64)
    return scipy.linalg.toeplitz(s[n - 1:n + m - 1], s[n - 1::-1])


def keys_by_library(raw_bits_2d, seed_bits, n, m):
    """np.convolve reduction: y_i = conv(s, x)[n-1+i] mod 2."""
    s = np.asarray(seed_bits, np.int64)
    return np.array([np.convolve(s, x.astype(np.int64))[n - 1:n + m - 1] % 2
                     for x in raw_bits_2d], dtype=np.uint8)


def run_oracle(oracle_mod, raw_bits_2d, seed_bits, n, m, mode):
    B = raw_bits_2d.shape[0]
    out = oracle_mod.extract(pack(raw_bits_2d.reshape(-1)), B, n, m, pack(seed_bits), mode)
    return bits_of(out, B * m).reshape(B, m)


@pytest.mark.parametrize("mode", ["scalar", "words"])
def test_golden_p1(oracle_mod, mode):
    g = json.load(open(os.path.join(GOLDEN, "p1_spec_example_rotated.json")))
    y = run_oracle(oracle_mod, np.array([g["raw_bits"]], np.uint8), g["seed_bits"],
                   g["n"], g["m"], mode)
    assert y.tolist() == [g["key_bits"]]


@pytest.mark.parametrize("mode", ["scalar", "words"])
def test_golden_p2_bytes(oracle_mod, mode):
    g = json.load(open(os.path.join(GOLDEN, "p2_byte_level.json")))
    raw = np.frombuffer(bytes.fromhex(g["raw_hex"]), np.uint8)
    seed = np.frombuffer(bytes.fromhex(g["seed_hex"]), np.uint8)
    out = oracle_mod.extract(raw, g["n_blocks"], g["n"], g["m"], seed, mode)
    assert out.tobytes().hex() == g["key_hex"]
    per = oracle_mod.extract_blocks(raw, [0, 1, 2], g["n"], g["m"], seed, mode)
    assert [bits_of(r, g["m"]).tolist() for r in per] == g["block_keys"]


def test_seed_pad_bits_ignored(oracle_mod):
    g = json.load(open(os.path.join(GOLDEN, "p2_byte_level.json")))
    raw = np.frombuffer(bytes.fromhex(g["raw_hex"]), np.uint8)
    seed = np.frombuffer(bytes.fromhex(g["seed_hex"]), np.uint8).copy()
    seed[-1] |= 0x1F  # bits 11..15 are padding
    assert oracle_mod.extract(raw, 3, 8, 4, seed).tobytes().hex() == g["key_hex"]


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 7, 8, 9, 10])
def test_bruteforce_all_blocks_small_n(oracle_mod, n):
    """Exhaustive over x (all 2^n blocks in one stream) for every m < n; seeds:
    every seed when 2n+m-1 <= 14, else all unit seeds plus 8 random seeds.
    Reference: the paper's matrix built by scipy.linalg.toeplitz, times X."""
    X = ((np.arange(1 << n)[:, None] >> np.arange(n - 1, -1, -1)) & 1).astype(np.uint8)
    rng = np.random.default_rng(1000 + n)
    for m in range(1, n):
        L = n + m - 1
        if 2 * n + m - 1 <= 14:
            seeds = ((np.arange(1 << L)[:, None] >> np.arange(L - 1, -1, -1)) & 1)
        else:
            seeds = np.vstack([np.eye(L, dtype=np.int64), rng.integers(0, 2, (8, L))])
        for s in seeds:
            ref = (toeplitz_matrix(s, n, m) @ X.T.astype(np.int64) % 2).T
            for mode in (["words", "scalar"] if n <= 6 else ["words"]):
                got = run_oracle(oracle_mod, X, s, n, m, mode)
                assert np.array_equal(got, ref), (n, m, s, mode)


@pytest.mark.parametrize("n", [11, 13, 16])
def test_bruteforce_n_le_16(oracle_mod, n):
    """n up to 16 (north_star): all 2^n blocks against the library matrix,
    for the two unit seeds at the ends of the seed and 2 random seeds."""
    X = ((np.arange(1 << n)[:, None] >> np.arange(n - 1, -1, -1)) & 1).astype(np.uint8)
    rng = np.random.default_rng(n)
    for m in (1, n // 2, n - 1):
        L = n + m - 1
        seeds = [np.eye(L, dtype=np.int64)[0], np.eye(L, dtype=np.int64)[L - 1],
                 rng.integers(0, 2, L), rng.integers(0, 2, L)]
        for s in seeds:
            ref = (toeplitz_matrix(s, n, m) @ X.T.astype(np.int64) % 2).T
            assert np.array_equal(run_oracle(oracle_mod, X, s, n, m, "words"), ref)


def test_unit_pairs_closed_form(oracle_mod):
    """P3: s = e_k, x = e_j  =>  y_i = [i == k + j - n + 1], every (k, j)."""
    for n, m in [(6, 4), (9, 5), (64, 33), (70, 69)]:
        L = n + m - 1
        X = np.eye(n, dtype=np.uint8)
        for k in range(L):
            s = np.zeros(L, np.uint8)
            s[k] = 1
            got = run_oracle(oracle_mod, X, s, n, m, "words")
            ref = np.zeros((n, m), np.uint8)
            for j in range(n):
                i = k + j - n + 1
                if 0 <= i < m:
                    ref[j, i] = 1
            assert np.array_equal(got, ref), (n, m, k)


def test_special_cases(oracle_mod):
    """P4 closed forms."""
    rng = np.random.default_rng(4)
    for n, m in [(32, 20), (100, 7), (1024, 716)]:
        L = n + m - 1
        X = rng.integers(0, 2, (5, n)).astype(np.uint8)
        e = np.zeros(L, np.uint8)
        e[n - 1] = 1  # identity: y = x[0:m)
        assert np.array_equal(run_oracle(oracle_mod, X, e, n, m, "words"), X[:, :m])
        for d in (1, 3, m - 1):  # shift: s = e_{n-1+d} => y_i = x_{i-d}
            e = np.zeros(L, np.uint8)
            e[n - 1 + d] = 1
            ref = np.zeros((5, m), np.uint8)
            ref[:, d:] = X[:, :m - d]
            assert np.array_equal(run_oracle(oracle_mod, X, e, n, m, "words"), ref)
        ones = np.ones(L, np.uint8)
        par = (X.sum(1) % 2).astype(np.uint8)
        assert np.array_equal(run_oracle(oracle_mod, X, ones, n, m, "words"),
                              np.repeat(par[:, None], m, 1))
        full = np.ones((1, n), np.uint8)  # every window sum equals n
        assert np.array_equal(run_oracle(oracle_mod, full, ones, n, m, "words"),
                              np.full((1, m), n % 2, np.uint8))
        assert not run_oracle(oracle_mod, X, np.zeros(L, np.uint8), n, m, "words").any()
        assert not run_oracle(oracle_mod, np.zeros((2, n), np.uint8), rng.integers(0, 2, L),
                              n, m, "words").any()


@pytest.mark.parametrize("n,m,B", [(1024, 716, 6), (2048, 1500, 3), (4096, 2867, 2), (777 * 8, 4000, 2)])
def test_library_convolution(oracle_mod, n, m, B):
    """P5: np.convolve(s, x)[n-1:n+m-1] % 2, scipy toeplitz @ x, and the GF(2)[z]
    carry-less product of Python ints, coefficients n-1..n+m-2."""
    rng = np.random.default_rng(n + m)
    X = rng.integers(0, 2, (B, n)).astype(np.uint8)
    s = rng.integers(0, 2, n + m - 1).astype(np.uint8)
    ref = keys_by_library(X, s, n, m)
    assert np.array_equal(run_oracle(oracle_mod, X, s, n, m, "words"), ref)
    T = toeplitz_matrix(s, n, m)
    assert np.array_equal((T @ X[0].astype(np.int64)) % 2, ref[0])
    # carry-less product: bit t of S(z)*X(z) over GF(2)
    S = sum(int(b) << k for k, b in enumerate(s))
    x = sum(int(b) << k for k, b in enumerate(X[0]))
    prod = 0
    while x:
        low = x & -x
        prod ^= S << (low.bit_length() - 1)
        x ^= low
    clmul = np.array([(prod >> (n - 1 + i)) & 1 for i in range(m)], np.uint8)
    assert np.array_equal(clmul, ref[0])


def test_scalar_equals_words_random(oracle_mod):
    """Mode (ii) validated against mode (i) on random inputs up to n = 2^12."""
    rng = np.random.default_rng(12)
    for n, m, B in [(64, 63, 3), (65, 2, 4), (127, 90, 3), (1000, 333, 2), (4096, 2867, 1)]:
        X = rng.integers(0, 2, (B, n)).astype(np.uint8)
        s = rng.integers(0, 2, n + m - 1).astype(np.uint8)
        a = run_oracle(oracle_mod, X, s, n, m, "scalar")
        b = run_oracle(oracle_mod, X, s, n, m, "words")
        assert np.array_equal(a, b)


def test_paper_fft_method(oracle_mod):
    """The paper's own O(n log n) method (Listing 2 at
    PAPER.md:402-413): k' = round(ifft(fft(a) * fft(r'))) mod 2 with a = s
    (first column of the circulant A, Def. 1), r' = r zero-padded to L, keeping
    k_n .. k_{n+m-1}.  Double precision is exact at these L."""
    rng = np.random.default_rng(7)
    for n, m in [(1024, 716), (4096, 2867), (3000, 1234)]:
        L = n + m - 1
        X = rng.integers(0, 2, (3, n)).astype(np.uint8)
        s = rng.integers(0, 2, L).astype(np.float64)
        ref = []
        for x in X:
            r = np.zeros(L)
            r[:n] = x
            k = np.fft.ifft(np.fft.fft(s) * np.fft.fft(r)).real
            assert np.max(np.abs(k - np.round(k))) < 0.25
            ref.append((np.round(k).astype(np.int64) % 2)[n - 1:n + m - 1])
        assert np.array_equal(run_oracle(oracle_mod, X, s.astype(np.uint8), n, m, "words"),
                              np.array(ref, np.uint8))


def test_linearity_and_shift(oracle_mod):
    """P6: h(x ^ x') = h(x) ^ h(x'); same in s; shift structure
    x' = (0, x_0..x_{n-2}) => y'_i = y_{i-1} ^ (s[i-1] & x_{n-1}), i >= 1."""
    rng = np.random.default_rng(6)
    n, m = 200, 150
    L = n + m - 1
    x1, x2 = rng.integers(0, 2, (2, n)).astype(np.uint8)
    s1, s2 = rng.integers(0, 2, (2, L)).astype(np.uint8)
    h = lambda x, s: run_oracle(oracle_mod, x[None], s, n, m, "words")[0]
    assert np.array_equal(h(x1 ^ x2, s1), h(x1, s1) ^ h(x2, s1))
    assert np.array_equal(h(x1, s1 ^ s2), h(x1, s1) ^ h(x1, s2))
    xs = np.concatenate([[0], x1[:-1]]).astype(np.uint8)
    y, ys = h(x1, s1), h(xs, s1)
    for i in range(1, m):
        assert ys[i] == y[i - 1] ^ (s1[i - 1] & x1[n - 1])
    # Toeplitz structure of the implied matrix: T[i+1][j+1] == T[i][j]
    T = np.array([run_oracle(oracle_mod, np.eye(n, dtype=np.uint8)[j:j + 1], s1, n, m, "words")[0]
                  for j in range(n)]).T  # column j = h(e_j)
    assert np.array_equal(T[1:, 1:], T[:-1, :-1])


def test_block_independence_and_selection(oracle_mod):
    """Block b of a batch equals the single-block call (P10 host side) and
    extract_blocks on sampled ids equals the corresponding slices."""
    w = qrng_synth.CONFIGS[1]
    raw, seed = qrng_synth.workload_inputs(w, 0, 40)
    full = oracle_mod.extract(raw, 40, w.n, w.m, seed)
    ids = [0, 7, 39]
    per = oracle_mod.extract_blocks(raw, ids, w.n, w.m, seed)
    for q, b in enumerate(ids):
        assert np.array_equal(bits_of(per[q], w.m), bits_of(full, w.m, b * w.m))
        single = oracle_mod.extract(raw[b * w.n // 8:(b + 1) * w.n // 8], 1, w.n, w.m, seed)
        assert np.array_equal(bits_of(single, w.m), bits_of(full, w.m, b * w.m))


def test_output_pad_bits_zero(oracle_mod):
    rng = np.random.default_rng(3)
    n, m, B = 24, 13, 3  # 39 output bits -> 5 bytes, 1 pad bit
    raw = rng.integers(0, 256, n * B // 8).astype(np.uint8)
    seed = rng.integers(0, 256, (n + m - 1 + 7) // 8).astype(np.uint8)
    out = oracle_mod.extract(raw, B, n, m, seed)
    assert out.size == 5 and out[-1] & 1 == 0


def test_rejects_bad_args(oracle_mod):
    raw = np.zeros(16, np.uint8)
    seed = np.zeros(16, np.uint8)
    for n, m, B in [(8, 8, 1), (8, 0, 1), (0, 1, 1), (8, 4, 0)]:
        with pytest.raises(ValueError):
            oracle_mod.extract(raw, B, n, m, seed)
