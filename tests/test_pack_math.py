"""Host check of the index arithmetic the fused combine + pack kernel uses
(karatsuba.cu, csr_stream_pack_kernel, FUSED form) to place key rows at bit
b*m + i of the output (C4): written out here in plain
Python on random rows and compared with the direct bit concatenation.  Pure
host logic, no GPU; it pins the word/shift/straddle rules, not the CUDA code.
"""
import numpy as np
import pytest


def direct(rows, m):
    """Concatenate the m-bit rows MSB-first and cut into 32-bit words."""
    bits = np.concatenate([np.unpackbits(r.astype(">u4").view(np.uint8))[:m] for r in rows])
    pad = (-bits.size) % 32
    bits = np.concatenate([bits, np.zeros(pad, np.uint8)])
    return np.packbits(bits).view(">u4").astype(np.uint32)


def fused(rows, m):
    """The kernel's rule: lane kk of block bl forms output word W = ceil(s0/32) + kk
    from key words R[kk], R[kk+1] with shift d = 32*ceil(s0/32) - s0; the word that
    straddles into block bl+1 takes that block's word 0 (its 'head') shifted."""
    nb = len(rows)
    ywords = (m + 31) // 32
    R = [np.concatenate([r, np.zeros(1, np.uint32)]) for r in rows]  # pad word = 0
    heads = [int(r[0]) for r in R]
    out = np.zeros((nb * m + 31) // 32, np.uint32)
    written = np.zeros(out.size, bool)
    for bl in range(nb):
        s0, s1 = bl * m, bl * m + m
        wf = (s0 + 31) // 32
        d = 32 * wf - s0
        for kk in range(ywords + 1):
            W = wf + kk
            if 32 * W >= s1:
                continue
            r0, r1 = int(R[bl][kk]) if kk <= ywords else 0, int(R[bl][kk + 1]) if kk + 1 <= ywords else 0
            word = ((r0 << d) | (r1 >> (32 - d))) & 0xFFFFFFFF if d else r0
            if 32 * W + 32 > s1:
                len1 = s1 - 32 * W
                word &= ~(0xFFFFFFFF >> len1) & 0xFFFFFFFF
                if bl + 1 < nb:
                    word |= heads[bl + 1] >> len1
            assert not written[W], "two writers for one word"
            out[W], written[W] = word, True
    assert written.all()  # every output word has exactly one writer
    return out


@pytest.mark.parametrize("m", [64, 65, 95, 96, 127, 716, 1433, 5734, 11468])
def test_fused_pack_rule_matches_concatenation(m):
    rng = np.random.default_rng(m)
    ywords = (m + 31) // 32
    bpc = 32
    while bpc > 1 and (bpc // 2) * m % 32 == 0:  # the host's group size rule
        bpc //= 2
    for nb in sorted({1, 2, bpc}):
        rows = []
        for _ in range(nb):
            r = rng.integers(0, 2**32, ywords, dtype=np.uint64).astype(np.uint32)
            if m % 32:  # key bits past m are zero in the combined rows
                r[-1] &= np.uint32((0xFFFFFFFF << (32 - m % 32)) & 0xFFFFFFFF)
            rows.append(r)
        got = fused(rows, m)
        ref = direct(rows, m)
        if nb * m % 32:  # the tail word's bits past the key are not part of the output
            keep = nb * m % 32
            got[-1] &= np.uint32((0xFFFFFFFF << (32 - keep)) & 0xFFFFFFFF)
        assert np.array_equal(got, ref), (m, nb)
