"""Config 5 (BASELINE.json configs[4]) at FULL size, every point, through AUTO
-- what bench.py and the driver time: one fixed 2^30-bit raw sequence,
n = 2^k for k = 10..22, m = floor(0.7 n), 2^30 / n blocks (2^20 ... 256),
against the CPU oracle bit for bit (Fig. 6 / Table 2: the
block-length sweep).

Per point:
* sampled outputs (oracle_extract_rows, pinned in test_oracle_sampled.py) on
  the first, last and middle blocks, the blocks on both sides of every
  rank boundary of the 2-, 4- and 8-GPU partitions (SURVEY 8(e):
  [floor(rB/W), floor((r+1)B/W))), and random blocks; first/last rows of each;
* one whole block, every row, against the oracle;
* P10 on one GPU: the 8 shards of the 8-GPU partition extracted as separate
  calls (each a self-contained stream, what each rank computes) concatenate
  to the 1-GPU output byte for byte.

Run on a B200:  python -m pytest tests -m gpu
"""
import numpy as np
import pytest

import qrng_synth as S
from paper_2011_04130_b200 import dist as qd

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
    q.set_debug_path(q.PATH_AUTO)
    q.set_karatsuba(-1)
    yield q


@pytest.fixture(scope="module")
def raw_stream():
    """The one fixed 2^30-bit sequence of config 5 (the same bytes at every n)."""
    w = S.sweep_workload(10)
    raw, _ = S.workload_inputs(w)
    assert raw.size * 8 == 1 << 30
    return raw, torch.from_numpy(raw).cuda()


def bits_at(buf: np.ndarray, pos: np.ndarray) -> np.ndarray:
    pos = pos.astype(np.int64)
    return (buf[pos >> 3] >> (7 - (pos & 7))) & 1


def boundary_blocks(B):
    out = {0, B - 1, B // 2}
    for W in (2, 4, 8):
        for r in range(1, W):
            b0 = qd.shard_range(B, r, W)[0]
            out |= {b0 - 1, b0}
    return sorted(out)


@pytest.mark.parametrize("log2n", list(range(10, 23)))
def test_sweep_point_full_size(q, oracle_mod, raw_stream, log2n):
    w = S.sweep_workload(log2n)
    n, m, B = w.n, w.m, w.n_blocks
    raw, d_raw = raw_stream
    _, seed = S.workload_inputs(w, 0, 1)
    d_seed = torch.from_numpy(seed).cuda()
    got = q.toeplitz_extract(d_raw, B, n, m, d_seed).cpu().numpy()
    assert got.size == (B * m + 7) // 8

    # sampled rows
    rng = np.random.default_rng(log2n)
    blocks = sorted(set(boundary_blocks(B)) | set(rng.integers(0, B, 6).tolist()))
    n_rows = 48
    bl, rw = [], []
    for b in blocks:
        rows = np.unique(np.concatenate([[0, 1, m - 2, m - 1], rng.integers(0, m, n_rows)]))
        bl += [b] * rows.size
        rw += rows.tolist()
    bl, rw = np.array(bl, np.uint64), np.array(rw, np.uint64)
    ref = oracle_mod.extract_rows(raw, bl, rw, n, m, seed)
    gb = bits_at(got, bl * m + rw)
    bad = np.nonzero(gb != ref)[0]
    assert bad.size == 0, f"{bad.size} sampled bits differ, first (block {bl[bad[0]]}, row {rw[bad[0]]})"

    # one whole block (a random one), every row
    b = int(rng.integers(0, B))
    rows = np.arange(m, dtype=np.uint64)
    ref_block = oracle_mod.extract_rows(raw, np.full(m, b, np.uint64), rows, n, m, seed)
    assert np.array_equal(bits_at(got, b * m + rows), ref_block), f"block {b}"

    # pad bits of the last byte
    tail = B * m % 8
    if tail:
        assert got[-1] & ((1 << (8 - tail)) - 1) == 0

    # the 8-GPU partition's shards, each its own call, concatenate to the same stream
    W = 8
    for r in range(W):
        b0, b1 = qd.shard_range(B, r, W)
        assert (b0 * m) % 8 == 0 and ((b1 - b0) * m) % 8 == 0  # shard bits are whole bytes here
        part = q.toeplitz_extract(d_raw[b0 * n // 8:b1 * n // 8], b1 - b0, n, m, d_seed).cpu().numpy()
        assert np.array_equal(part, got[b0 * m // 8:b1 * m // 8]), f"rank {r} of {W}"
