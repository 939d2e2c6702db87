"""Pins for the modified-Toeplitz oracle (Sec. III.D;
Listing 3 at PAPER.md:415-429), reading A24: the key is
[T | I_m] r with T = the last m rows and first n-m columns of the n x n
circulant A_c whose first column is the n-bit seed a', and the
identity block adds the last m raw bits (k_i = k'_i + r_{i+1}).
"""
import numpy as np
import pytest
import scipy.linalg


def bits_of(buf, count, off=0):
    return np.unpackbits(np.asarray(buf, np.uint8))[off:off + count]


def pack(bits):
    return np.packbits(np.asarray(bits, np.uint8))


def paper_matrix(seed_bits, n, m):
    """[T | I_m] built literally: scipy circulant with first column a' (Def. 1
    pattern of PAPER.md:253), last m rows, first n-m columns, then I_m."""
    Ac = scipy.linalg.circulant(np.asarray(seed_bits, np.int64))
    T = Ac[n - m:, :n - m]
    return np.hstack([T, np.eye(m, dtype=np.int64)])


def run(oracle_mod, X, seed, n, m):
    B = X.shape[0]
    out = oracle_mod.modified_extract(pack(X.reshape(-1)), B, n, m, pack(seed))
    return bits_of(out, B * m).reshape(B, m)


@pytest.mark.parametrize("n", [2, 3, 4, 5, 6, 8, 10])
def test_matrix_form_exhaustive_blocks(oracle_mod, n):
    X = ((np.arange(1 << n)[:, None] >> np.arange(n - 1, -1, -1)) & 1).astype(np.uint8)
    rng = np.random.default_rng(n)
    for m in range(1, n):
        seeds = ((np.arange(1 << n)[:, None] >> np.arange(n - 1, -1, -1)) & 1) if n <= 5 else \
            np.vstack([np.eye(n, dtype=np.int64), rng.integers(0, 2, (6, n))])
        for s in seeds:
            ref = (paper_matrix(s, n, m) @ X.T.astype(np.int64) % 2).T
            assert np.array_equal(run(oracle_mod, X, s, n, m), ref), (n, m, s)


def test_paper_fft_listing3_structure(oracle_mod):
    """Listing 3's computation k' = round(ifft(fft(a') fft(r'))) mod 2 with the
    last m raw bits zeroed in r', keeping the rows the prose names
    (n-m .. n-1, 0-based) and adding the withheld bits."""
    rng = np.random.default_rng(3)
    for n, m in [(1024, 716), (2048, 1000), (777, 300)]:
        X = rng.integers(0, 2, (3, n)).astype(np.uint8)
        a = rng.integers(0, 2, n)
        ref = []
        for x in X:
            r = x.astype(np.float64).copy()
            r[n - m:] = 0
            k = np.round(np.fft.ifft(np.fft.fft(a) * np.fft.fft(r)).real).astype(np.int64) % 2
            ref.append(k[n - m:] ^ x[n - m:])
        assert np.array_equal(run(oracle_mod, X, a, n, m), np.array(ref, np.uint8))


def test_closed_forms(oracle_mod):
    rng = np.random.default_rng(5)
    n, m = 40, 17
    X = rng.integers(0, 2, (4, n)).astype(np.uint8)
    # seed 0: only the identity block survives (the withheld raw bits)
    assert np.array_equal(run(oracle_mod, X, np.zeros(n, np.uint8), n, m), X[:, n - m:])
    for k in (1, 5, n - m, n - 1):
        e = np.zeros(n, np.uint8)
        e[k] = 1
        ref = X[:, n - m:].copy()
        for t in range(m):
            j = n - m + t - k
            if 0 <= j < n - m:
                ref[:, t] ^= X[:, j]
        assert np.array_equal(run(oracle_mod, X, e, n, m), ref), k


def test_equals_standard_on_shortened_block(oracle_mod):
    """Derived identity: [T | I_m] r = (standard C1 extraction of r[0:n-m] with
    n' = n-m and seed a'[1:], n'+m-1 = n-1 bits)  XOR  r[n-m:n].  (The standard
    oracle requires m < n', so only m < n/2 here; the matrix-form and Listing-3
    pins cover m > n/2.)"""
    rng = np.random.default_rng(9)
    for n, m in [(64, 20), (1024, 300), (301, 150)]:
        B = 5
        X = rng.integers(0, 2, (B, n)).astype(np.uint8)
        a = rng.integers(0, 2, n).astype(np.uint8)
        std = oracle_mod.extract(pack(X[:, :n - m].reshape(-1)), B, n - m, m, pack(a[1:]))
        ref = bits_of(std, B * m).reshape(B, m) ^ X[:, n - m:]
        assert np.array_equal(run(oracle_mod, X, a, n, m), ref)


def test_linearity(oracle_mod):
    rng = np.random.default_rng(11)
    n, m = 96, 50
    x1, x2 = rng.integers(0, 2, (2, n)).astype(np.uint8)
    a = rng.integers(0, 2, n).astype(np.uint8)
    h = lambda x: run(oracle_mod, x[None], a, n, m)[0]
    assert np.array_equal(h(x1 ^ x2), h(x1) ^ h(x2))


def test_rows_mode_equals_literal(oracle_mod):
    """The word-parallel sampled-row form equals the literal bit loop."""
    rng = np.random.default_rng(13)
    for n, m, B in [(64, 20, 3), (96, 95, 2), (1024, 716, 3), (800, 1, 2), (256, 200, 4)]:
        X = rng.integers(0, 2, (B, n)).astype(np.uint8)
        a = rng.integers(0, 2, n).astype(np.uint8)
        full = run(oracle_mod, X, a, n, m)
        bl = np.repeat(np.arange(B), m)
        rw = np.tile(np.arange(m), B)
        got = oracle_mod.modified_rows(pack(X.reshape(-1)), bl, rw, n, m, pack(a))
        assert np.array_equal(got.reshape(B, m), full)
