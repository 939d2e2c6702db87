"""Host logic of the Karatsuba decomposition (no GPU): the planner's tables,
applied literally, reproduce the CPU oracle's extraction.

The library's host planner (qrng_debug_karatsuba_plan, include/qrng.h) says
which Toeplitz leaf products the tensor cores run -- each leaf seed an XOR of
windows of the seed s, each leaf input an XOR of windows of the block x -- and
which leaf parity words XOR into each output word.  Here every leaf product is
computed from its definition y_l[i] = XOR_j d_l[i-j+w-1] x_l[j] (np.convolve
parity), the leaves are combined as the tables say, and the
result must equal the oracle's key bit for bit (the GF(2) Karatsuba identities
of DESIGN.md "Karatsuba over the GEMM path").  A wrong seed window, a wrong
input window, a wrong combine offset or a dropped term fails this test.
"""
import numpy as np
import pytest

import paper_2011_04130_b200 as q


@pytest.fixture(scope="module", autouse=True)
def lib():
    from paper_2011_04130_b200 import build
    build.build()
    q.load_library()


def bits_of(packed: np.ndarray, nbits: int) -> np.ndarray:
    return np.unpackbits(packed)[:nbits].astype(np.int64)


def apply_plan(kp, s_bits, x_bits, m):
    """Evaluate the decomposition literally (test-side, CPU)."""
    L = s_bits.size
    pad = np.concatenate([s_bits, np.zeros(4 * x_bits.size + 64, np.int64)])  # s is 0 past L
    y_words = max(l[2] + (l[0] + 31) // 32 for l in kp.leaves)
    Y = np.zeros(32 * y_words, np.int64)
    for r, w, out_off, sterms, iterms in kp.leaves:
        d = np.zeros(r + w - 1, np.int64)
        for t in sterms:
            assert t + r + w - 1 <= pad.size
            d ^= pad[t:t + r + w - 1]
        xl = np.zeros(w, np.int64)
        for u in iterms:
            assert u + w <= x_bits.size, "input window past the block"
            xl ^= x_bits[u:u + w]
        yl = np.convolve(d, xl)[w - 1:w - 1 + r] & 1  # y_l[i] = sum_j d[i-j+w-1] x[j]
        Y[32 * out_off:32 * out_off + r] = yl
    words = (m + 31) // 32
    y = np.zeros(32 * words, np.int64)
    for j in range(words):
        acc = np.zeros(32, np.int64)
        for e in kp.comb_idx[kp.comb_ptr[j]:kp.comb_ptr[j + 1]]:
            acc ^= Y[32 * int(e):32 * int(e) + 32]
        y[32 * j:32 * j + 32] = acc
    del L
    return y[:m]


CASES = [
    (256, 200, 1), (512, 300, 2), (1024, 716, 1), (1024, 716, 2), (1024, 1000, 3), (2048, 1433, 3),
    (2048, 5, 3), (2048, 2047, 4), (4096, 2867, -1), (8192, 5734, 1), (8192, 5734, 2), (8192, 5734, 3),
    (8192, 5734, -1), (8192, 100, 4), (3072, 2100, 3), (65536, 45875, -1),
]


@pytest.mark.parametrize("n,m,depth", CASES)
def test_plan_reproduces_oracle(oracle_mod, n, m, depth):
    kp = q.karatsuba_plan(n, m, depth)
    if depth > 0:
        assert kp.depth >= 1
    rng = np.random.default_rng(n * 7 + m * 3 + depth)
    L = n + m - 1
    seed = rng.integers(0, 256, (L + 7) // 8, dtype=np.uint8)
    raw = rng.integers(0, 256, n // 8, dtype=np.uint8)
    ref = bits_of(oracle_mod.extract(raw, 1, n, m, seed), m)
    got = apply_plan(kp, bits_of(seed, L), bits_of(raw, n), m)
    assert np.array_equal(got, ref)


def test_leaf_shapes_and_work():
    """Depth-d splits of a square-ish product: leaves are multiples of 128 wide,
    rows never exceed the leaf width, and each Karatsuba level cuts the
    multiply-accumulates (3 half products instead of 4)."""
    n, m = 8192, 5734
    macs = []
    for d in range(0, 4):
        kp = q.karatsuba_plan(n, m, d)
        for r, w, *_ in kp.leaves:
            assert w % 128 == 0 and 1 <= r <= w
        macs.append(sum(r * w for r, w, *_ in kp.leaves))
    assert macs[0] == n * m
    assert macs[1] < macs[0] and macs[2] < macs[1] and macs[3] < macs[2]


def test_no_decomposition_rejected():
    with pytest.raises(q.QrngError):
        q.karatsuba_plan(8192 + 32, 100, 2)  # n % 128 != 0
    with pytest.raises(q.QrngError):
        q.karatsuba_plan(1024, 1024, 2)      # m >= n


def test_adversarial_packed_precondition():
    """tests/test_gpu_edges.py's packed-accumulator case really drives
    S1 = 2048 next to odd S0 in leaf 0 (CPU arithmetic on the plan's own
    leaf table; the GPU test then checks the kernel against the oracle)."""
    import sys, os
    sys.path.insert(0, os.path.dirname(__file__))
    from test_gpu_edges import adversarial_packed_inputs
    import paper_2011_04130_b200 as q
    n, m, h, s, X = adversarial_packed_inputs()
    plan = q.karatsuba_plan(n, m, 1)
    assert plan.depth == 1
    r, w, _, sterms, iterms = plan.leaves[0]
    assert (r, w, sterms, sorted(iterms)) == (2048, 2048, [h], [0, h])
    d = s[h:h + r + w - 1].astype(np.int64)
    xq = (X[0, :h] ^ X[0, h:]).astype(np.int64)
    # S(i) = sum_j d[i - j + w - 1] x_j
    S0 = np.array([int(np.dot(d[i:i + w][::-1], xq)) for i in range(r)])
    assert np.all(S0[224:] == 2048)
    assert np.sum(S0[:224] % 2 == 1) >= 100
    F = S0[:192] + 4096 * S0[224:224 + 192]     # a packed pair: rows c and 224 + c
    assert np.all(F >= 1 << 23) and np.any(F % 2 == 1)
