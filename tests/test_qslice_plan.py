"""CPU test of the one-pass Q-buffer table (karatsuba.cu qslice_kernel, round 2).

The GEMM path's Karatsuba leaves read their inputs x_l = XOR over input terms u
of x[u, u + w) either straight from the raw block or from a Q buffer (x0 ^ x1 of
a node) in the block's X row.  qslice_kernel forms every Q buffer in one pass
from the block's n / s aligned s-bit slices, as the library's chunk list says
(qrng_debug_qslice_plan).  Here that list is applied literally to random blocks
in numpy and every leaf's input window is compared with the XOR of raw windows
the planner lists for it independently (qrng_debug_karatsuba_plan's input
terms, built by the tree walk in `collect`): a wrong mask, slice index or
destination unit changes some leaf's input for a random block.
"""
import numpy as np
import pytest

import paper_2011_04130_b200 as q

# (n, m, depth): config 2 (auto = depth 2, 4 slices), forced depths 1-4,
# m < n/2 (a column split at the root, Karatsuba below), 2^14 / 2^15 auto (8 / 16 slices)
COVERED = [(8192, 5734, -1), (8192, 5734, 1), (8192, 5734, 3), (4096, 2867, 2), (8192, 3000, 3),
           (16384, 11468, -1), (32768, 22937, -1), (2048, 1500, 4), (8192, 8000, 2)]


def _leaf_inputs_from_slices(n, ns, lsu, ent, xw, leaf_x, leaves, x):
    s = 128 << lsu
    assert s * ns == n
    X = np.zeros(32 * xw, np.uint8)
    written = np.zeros(32 * xw, bool)
    for e in ent:
        mask, unit = e & 0xFFFF, e >> 16
        assert 0 < mask < (1 << ns)
        acc = np.zeros(s, np.uint8)
        for i in range(ns):
            if (mask >> i) & 1:
                acc ^= x[i * s:(i + 1) * s]
        lo = 128 * unit
        assert lo + s <= X.size
        assert not written[lo:lo + s].any(), "two chunks write the same X-row bits"
        X[lo:lo + s] = acc
        written[lo:lo + s] = True
    out = []
    for (src, word), (r, w, off, sterms, iterms) in zip(leaf_x, leaves):
        lo = 32 * word
        if src:
            assert written[lo:lo + w].all(), "leaf reads X-row bits no chunk writes"
            out.append(X[lo:lo + w])
        else:
            assert lo + w <= n
            out.append(x[lo:lo + w])
    return out


@pytest.mark.parametrize("n,m,depth", COVERED)
def test_qslice_chunks_reproduce_leaf_inputs(n, m, depth):
    ns, lsu, ent, xw, leaf_x = q.qslice_plan(n, m, depth)
    plan = q.karatsuba_plan(n, m, depth)
    assert ns in (2, 4, 8, 16), f"expected a covered tree, got {ns} slices (depth {plan.depth})"
    assert len(leaf_x) == len(plan.leaves)
    rng = np.random.default_rng(n * 7 + m + depth)
    for _ in range(3):
        x = rng.integers(0, 2, n, dtype=np.uint8)
        got = _leaf_inputs_from_slices(n, ns, lsu, ent, xw, leaf_x, plan.leaves, x)
        for l, (r, w, off, sterms, iterms) in enumerate(plan.leaves):
            want = np.zeros(w, np.uint8)
            for u in iterms:
                assert u + w <= n
                want ^= x[u:u + w]
            assert np.array_equal(got[l], want), f"leaf {l} (r={r}, w={w}) input differs"


def test_qslice_chunk_count_bound():
    # every Q buffer of width h at tree level l is h / s chunks; a tree of
    # Karatsuba splits down to depth d has at most sum_l 3^l 2^(d-l-1) = 3^d - 2^d
    for n, m, d in [(8192, 5734, 2), (16384, 11468, 3), (32768, 22937, 4)]:
        ns, _, ent, _, _ = q.qslice_plan(n, m, d)
        assert ns == 2 ** d and 0 < len(ent) <= 3 ** d - 2 ** d


def test_qslice_not_covered():
    # 32 slices (depth 5, config 3), no Q buffers (dense plan; column splits
    # only): the generation kernel / no Q-buffer launch, an empty chunk list
    ns, _, ent, _, _ = q.qslice_plan(65536, 45875, -1)
    assert ns == 0 and ent == []
    ns, _, ent, xw, _ = q.qslice_plan(8192, 5734, 0)
    assert ns == 0 and ent == [] and xw == 0
    ns, _, ent, xw, _ = q.qslice_plan(8192, 1000, 3)
    assert ns == 0 and ent == [] and xw == 0
