"""CPU pins of the packed three-prime NTT form's arithmetic (ntt.cu).

The GPU path puts G = 4 blocks into one transform as v = sum_g 2^(k g) x_g,
convolves v with the seed modulo three NTT primes and recovers every block's
key bits from the CRT value.  These tests fix, independently of the GPU code:
the primes' properties the transforms rely on (prime, 2-adic order, primitive
root 3), the range bound V < kP kP2 kP3 for every n the plans pack, and the
whole chain -- residues of the packed convolution, Garner recombination
reduced mod 2^64, bits 0, k, 2k, 3k -- against the per-block parities of a
plain convolution (np.convolve, PAPER.md:213, 229 window y_i = c[n-1+i]),
including the all-ones inputs that put every window sum at its maximum.
"""
import math

import numpy as np
import pytest

P0, P1, P2 = 998244353, 469762049, 167772161  # 119*2^23+1, 7*2^26+1, 5*2^25+1


def is_prime(p):
    if p < 2:
        return False
    for d in range(2, math.isqrt(p) + 1):
        if p % d == 0:
            return False
    return True


def prime_factors(x):
    f, d = set(), 2
    while d * d <= x:
        while x % d == 0:
            f.add(d)
            x //= d
        d += 1
    if x > 1:
        f.add(x)
    return f


@pytest.mark.parametrize("p,two_adic", [(P0, 23), (P1, 26), (P2, 25)])
def test_ntt_prime_properties(p, two_adic):
    assert is_prime(p)
    assert (p - 1) % (1 << two_adic) == 0 and ((p - 1) >> two_adic) % 2 == 1
    assert all(pow(3, (p - 1) // q, p) != 1 for q in prime_factors(p - 1))  # 3 generates Z_p^*
    assert 4 * p < 1 << 32  # lazy residues: sums < 4p fit 32 bits


def test_range_bound_for_packed_sizes():
    # the plans pack G = 4 blocks for n < 2^21 (k = bit length of n, 3k <= 63);
    # V <= n sum_g 2^(k g) must stay below M for every such n
    M = P0 * P1 * P2
    assert M > 1 << 86
    for n in list(range(32, 1 << 12, 32)) + [(1 << 21) - 32, (1 << 20), (1 << 20) - 32, 1 << 19]:
        k = n.bit_length()
        assert 3 * k <= 63
        assert n * sum(1 << (k * g) for g in range(4)) < M
    n = 1 << 21  # the first size that is not packed: k = 22, 3k = 66 > 63
    assert 3 * n.bit_length() > 63


def garner_low64(r0, r1, r2):
    """Garner for (P0, P1, P2) as the CRT pass computes it, then V mod 2^64."""
    y1 = (r1 - r0) * pow(P0, -1, P1) % P1
    y2 = (r2 - r0 - P0 * y1) * pow(P0 * P1, -1, P2) % P2
    return (r0 + P0 * y1 + P0 * P1 * y2) % (1 << 64)


def conv_mod(s, v, p):
    """Linear convolution of integer sequences modulo p (exact big-int sums)."""
    out = [0] * (len(s) + len(v) - 1)
    for i, si in enumerate(s):
        if si:
            for j, vj in enumerate(v):
                out[i + j] += si * vj
    return [c % p for c in out]


def packed_keys(s, xs, n, m):
    k = n.bit_length()
    v = [sum(int(x[j]) << (k * g) for g, x in enumerate(xs)) for j in range(n)]
    res = [conv_mod([int(b) for b in s], v, p) for p in (P0, P1, P2)]
    keys = np.zeros((len(xs), m), np.uint8)
    for i in range(m):
        t = n - 1 + i
        V = garner_low64(res[0][t], res[1][t], res[2][t])
        for g in range(len(xs)):
            keys[g, i] = (V >> (k * g)) & 1
    return keys


def direct_keys(s, xs, n, m):
    return np.array([np.convolve(s.astype(np.int64), x.astype(np.int64))[n - 1:n - 1 + m] % 2 for x in xs],
                    np.uint8)


@pytest.mark.parametrize("n,m,seed", [(64, 40, 1), (96, 95, 2), (100, 7, 3), (128, 1, 4), (200, 150, 5)])
def test_packed_chain_matches_direct_parities(n, m, seed):
    rng = np.random.default_rng(seed)
    s = rng.integers(0, 2, n + m - 1, dtype=np.uint8)
    xs = [rng.integers(0, 2, n, dtype=np.uint8) for _ in range(4)]
    assert np.array_equal(packed_keys(s, xs, n, m), direct_keys(s, xs, n, m))


def test_packed_chain_at_maximal_window_sums():
    # all-ones seed: every window sum is popcount(x_g); blocks clear g bits so the
    # four fields sit at n, n-1, n-2, n-3 (distinct parities, V at its maximum)
    n, m = 128, 60
    s = np.ones(n + m - 1, np.uint8)
    xs = []
    for g in range(4):
        x = np.ones(n, np.uint8)
        x[:g] = 0
        xs.append(x)
    got = packed_keys(s, xs, n, m)
    assert np.array_equal(got, direct_keys(s, xs, n, m))
    assert [int(got[g, 0]) for g in range(4)] == [0, 1, 0, 1]


def test_too_narrow_field_is_detected():
    # with one bit less per field (k = bit length of n - 1) the maximal sums
    # carry into the next block's field and the chain is wrong: the bit length
    # of n is the narrowest exact spacing
    n, m = 128, 30
    s = np.ones(n + m - 1, np.uint8)
    xs = [np.ones(n, np.uint8) for _ in range(4)]
    k = n.bit_length() - 1
    v = [sum(int(x[j]) << (k * g) for g, x in enumerate(xs)) for j in range(n)]
    t = n - 1
    V = sum(int(s[t - j]) * v[j] for j in range(n))
    bits = [(V >> (k * g)) & 1 for g in range(4)]
    assert bits != [n % 2] * 4
