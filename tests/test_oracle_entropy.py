"""Pins for the min-entropy oracle (oracle/entropy.py) -- CPU only.

Closed forms of PAPER.md:59, 153, 155, 187; the soundness inequality the
paper's Sec. II.C derivation establishes; and the paper's
printed Sec. II.B numbers (2.99 / 2.94 / 0.05, loose) via a test-only model of
its N=5 attack example.
"""
import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import entropy as E
import qrng_synth


def test_hmin_closed_forms():
    for k in range(0, 9):
        counts = np.zeros(256, np.uint64)
        counts[:1 << k] = 17  # uniform over 2^k values
        assert E.h_min_counts(counts) == pytest.approx(k, abs=1e-12)
    point = np.zeros(256, np.uint64)
    point[200] = 12345
    assert E.h_min_counts(point) == 0.0
    c = np.array([3, 1, 0, 4], np.uint64)
    assert E.h_min_counts(c) == pytest.approx(-math.log2(4 / 8))


def test_gauss_hmin_pins():
    g = json.load(open(os.path.join(GOLDEN, "p8_entropy_closed_forms.json")))
    for sigma, key in [(20.0, "gauss_sigma20_hmin"), (12.0, "gauss_sigma12_hmin")]:
        p = E.ideal_gauss(128.0, sigma, 8)
        assert p.sum() == pytest.approx(1.0, abs=1e-12)
        # centre bin [127.5, 128.5) has probability erf(1 / (2 sqrt 2 sigma))
        closed = -math.log2(math.erf(0.5 / (math.sqrt(2.0) * sigma)))
        assert E.h_min(p) == pytest.approx(closed, abs=1e-9)
        assert E.h_min(p) == pytest.approx(g[key], abs=g["gauss_tol"])
        # symmetry about the integer mean (bins 128-k and 128+k)
        assert np.allclose(p[128 - 100:128], p[128 + 100:128:-1], atol=1e-15)


def test_fit_gauss_closed_form():
    c = np.zeros(256, np.uint64)
    c[100] = c[102] = 5
    mu, sigma = E.fit_gauss(c)
    assert mu == pytest.approx(101.0) and sigma == pytest.approx(1.0)
    c = np.zeros(256, np.uint64)
    c[7] = 9
    assert E.fit_gauss(c) == (7.0, 0.0)


def test_stat_distance_and_delta():
    assert E.stat_distance([0.6, 0.4], [0.5, 0.5]) == pytest.approx(0.1)
    assert E.stat_distance([1, 0], [0, 1]) == 1.0
    p = E.ideal_gauss(128, 20)
    assert E.stat_distance(p, p) == 0.0
    for N in (1, 5, 8):
        assert E.delta_h_m(0.0, N) == 0.0
        assert E.delta_h_m(2.0 ** (-N - 1), N) == pytest.approx(1.0)
    with pytest.raises(ValueError):
        E.delta_h_m(1.5, 8)


def test_output_length_cases():
    g = json.load(open(os.path.join(GOLDEN, "p8_entropy_closed_forms.json")))
    for n, h, N, s, m in g["output_length_cases"]:
        assert E.output_length(n, h, N, s) == m


def test_soundness_property():
    """P9 / PAPER.md:147-159: H_min(P) - Delta H_m(d(P, P')) <= H_min(P') for any
    P, P' over the same bins (the paper's Delta H <= Delta H_m chain)."""
    rng = np.random.default_rng(9)
    for N in (3, 4, 5, 8):
        K = 1 << N
        for _ in range(2500):
            a = rng.dirichlet(np.full(K, rng.uniform(0.05, 5)))
            b = rng.dirichlet(np.full(K, rng.uniform(0.05, 5))) if rng.random() < 0.5 else \
                np.abs(a + rng.normal(0, 0.01, K))
            b = b / b.sum()
            lhs = E.h_min(a) - E.delta_h_m(min(1.0, E.stat_distance(a, b)), N)
            assert lhs <= E.h_min(b) + 1e-12


def test_report_chain_consistency():
    w = qrng_synth.CONFIGS[1]
    samples = qrng_synth.adc_samples(w.key, 1 << 16, w.mu, w.sigma)
    r = E.report(samples, 8, w.n, 0)
    assert r.n_samples == samples.size
    assert r.h_min_mod == pytest.approx(max(0.0, r.h_min_ideal - r.delta_h_m))
    assert r.h_min_mod <= r.h_min_hist + 1e-12  # soundness on real data
    assert r.m == math.floor(w.n * r.h_min_mod / 8)
    assert abs(r.mu - 128) < 0.5 and abs(r.sigma - 20) < 0.5
    with pytest.raises(ValueError):
        E.histogram(np.array([40], np.uint8), 5)


def _attack_distributions(g):
    """Test-only model of the paper's Sec. II.B example:
    V = alpha_0 I, V' = alpha_e (1 - I/(beta_e I_max)) I, I ~ N(0,1), quantised
    by a 5-bit ADC over [lo, hi] with floor bins clamped at the edges.  Bin
    probabilities by deterministic quadrature of the N(0,1) density."""
    I = np.linspace(-10, 10, 4_000_001)
    w = np.exp(-I * I / 2) / math.sqrt(2 * math.pi) * (I[1] - I[0])
    K = 1 << g["bit_depth"]
    width = (g["hi"] - g["lo"]) / K

    def dist(v):
        k = np.clip(np.floor((v - g["lo"]) / width), 0, K - 1).astype(np.int64)
        return np.bincount(k, weights=w, minlength=K) / w.sum()

    V = g["alpha_0"] * I
    Vp = g["alpha_e"] * (1 - I / (g["beta_e"] * g["i_max"])) * I
    return dist(V), dist(Vp)


def test_paper_attack_example_loose():
    g = json.load(open(os.path.join(GOLDEN, "e1_paper_attack_n5.json")))
    pv, pvp = _attack_distributions(g)
    hv, hvp = E.h_min(pv), E.h_min(pvp)
    assert hv == pytest.approx(g["h_min_V"], abs=g["tolerance"])
    assert hvp == pytest.approx(g["h_min_Vprime"], abs=g["tolerance"])
    assert hv - hvp == pytest.approx(g["mutual_info"], abs=g["tolerance"])
    assert hvp < hv  # the attack lowers the min-entropy
    # the corrected value never exceeds what the attacked source really has
    dh = E.delta_h_m(E.stat_distance(pv, pvp), g["bit_depth"])
    assert hv - dh <= hvp
