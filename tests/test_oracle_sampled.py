"""Pins for the oracle's sampled entry points -- CPU only.

``oracle_extract_rows`` (y_i of block b for chosen (b, i) pairs) and
``oracle_extract_blocks`` are the checkers of every full-size sampled GPU
test, and ``oracle_hist256`` is the checker of the GPU histogram.  Each is
tied here to something other than itself:

* extract_rows / extract_blocks == the np.convolve reduction of C1
  (y_i = conv(s, x)[n-1+i] mod 2) computed
  from the unpacked bits, and == the literal scalar bit loop
  (``oracle.extract(..., "scalar")``, itself pinned in test_oracle_toeplitz.py);
* shapes with m % 64 != 0, n % 64 != 0, m = 1, m = n - 1, unsorted and
  repeated block ids, 1 thread and all threads;
* hist256 == np.bincount (the empirical distribution P'(x) of PAPER.md:57-61).
"""
import numpy as np
import pytest


def unpack(buf, count, off=0):
    return np.unpackbits(np.asarray(buf, np.uint8))[off:off + count]


def conv_keys(raw, seed, n, m, ids):
    """np.convolve form of C1 for the blocks `ids` (rows: blocks, cols: i)."""
    s = unpack(seed, n + m - 1).astype(np.int64)
    out = []
    for b in ids:
        x = unpack(raw, n, b * n).astype(np.int64)
        out.append(np.convolve(s, x)[n - 1:n + m - 1] % 2)
    return np.array(out, dtype=np.uint8)


SHAPES = [  # (n, m, blocks)
    (64, 1, 5),
    (64, 63, 4),
    (96, 37, 7),
    (128, 127, 4),
    (200, 130, 6),      # n % 64 != 0, m % 64 != 0
    (320, 64, 5),       # m % 64 == 0
    (1024, 716, 6),     # config 1 shape
    (2048, 1433, 3),
]


@pytest.mark.parametrize("n,m,B", SHAPES)
@pytest.mark.parametrize("threads", [1, 0])
def test_extract_rows_equals_convolution(oracle_mod, n, m, B, threads):
    rng = np.random.default_rng(1000 + n + m + B)
    raw = rng.integers(0, 256, (B * n + 7) // 8).astype(np.uint8)
    seed = rng.integers(0, 256, (n + m - 1 + 7) // 8).astype(np.uint8)
    ref = conv_keys(raw, seed, n, m, range(B))                  # (B, m)
    # every (block, row) pair, in a shuffled order with repeats
    bl = np.repeat(np.arange(B), m)
    rw = np.tile(np.arange(m), B)
    perm = rng.permutation(bl.size)
    extra = rng.integers(0, bl.size, bl.size // 3 + 1)
    order = np.concatenate([perm, extra])
    got = oracle_mod.extract_rows(raw, bl[order], rw[order], n, m, seed, threads=threads)
    assert np.array_equal(got, ref[bl[order], rw[order]])
    # and against the literal scalar loop over the whole batch
    lit = unpack(oracle_mod.extract(raw, B, n, m, seed, "scalar", threads), B * m).reshape(B, m)
    assert np.array_equal(lit, ref)


@pytest.mark.parametrize("n,m,B", SHAPES)
@pytest.mark.parametrize("mode", ["scalar", "words"])
def test_extract_blocks_unsorted_repeated(oracle_mod, n, m, B, mode):
    rng = np.random.default_rng(2000 + n + m)
    raw = rng.integers(0, 256, (B * n + 7) // 8).astype(np.uint8)
    seed = rng.integers(0, 256, (n + m - 1 + 7) // 8).astype(np.uint8)
    ids = list(rng.permutation(B)) + [B - 1, 0, B - 1]
    got = oracle_mod.extract_blocks(raw, ids, n, m, seed, mode)
    ref = conv_keys(raw, seed, n, m, ids)
    for q in range(len(ids)):
        assert np.array_equal(unpack(got[q], m), ref[q])
        # pad bits of each row stay 0
        assert not np.any(unpack(got[q], 8 * got.shape[1])[m:])


def test_extract_rows_rejects_bad_rows(oracle_mod):
    raw = np.zeros(16, np.uint8)
    seed = np.zeros(16, np.uint8)
    with pytest.raises(ValueError):
        oracle_mod.extract_rows(raw, [0], [8], 64, 8, seed)


@pytest.mark.parametrize("size", [0, 1, 15, 16, 17, 1000, 1 << 20])
def test_hist256_equals_bincount(oracle_mod, size):
    rng = np.random.default_rng(size)
    x = np.clip(np.rint(rng.normal(128, 20, size)), 0, 255).astype(np.uint8)
    if size > 3:
        x[:3] = [0, 255, 255]  # edge bins
    got = oracle_mod.hist256(x)
    assert got.dtype == np.uint64 and got.size == 256
    assert np.array_equal(got, np.bincount(x, minlength=256).astype(np.uint64))
    assert int(got.sum()) == size
