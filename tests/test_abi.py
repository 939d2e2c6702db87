"""C-ABI checks that need no GPU: the library loads, exports every symbol the
header declares, rejects invalid arguments with the documented codes, refuses
to run without an sm_100 device (no CPU fallback), and its host-side entropy
finalisation (qrng_entropy_from_counts) agrees with the oracle."""
import math
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
import paper_2011_04130_b200 as q
from paper_2011_04130_b200 import build as qbuild
from oracle import entropy as E
import qrng_synth


@pytest.fixture(scope="module")
def lib():
    qbuild.build()
    return q.load_library()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "qrng.h")).read()
    return sorted(set(re.findall(r"\b(qrng_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    declared = header_symbols()
    assert sorted(q.EXPORTS) == declared
    for name in declared:
        assert hasattr(lib, name), name
    assert q.version().startswith("qrng-b200")


def test_library_is_sm100a_only(lib):
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {q.LIB_PATH} 2>&1").read()
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, out


def test_oracle_not_imported_by_product():
    pkg = os.path.join(ROOT, "paper_2011_04130_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "toeplitz_oracle" not in txt, f


def _call_extract(lib, n, m, B, raw=16, seed=16, out=16):
    return lib.qrng_toeplitz_extract_async(raw, B, n, m, seed, out, None)


def test_invalid_arguments_codes(lib):
    # validated before any device work, so these hold on a CPU-only host too
    assert _call_extract(lib, 0, 1, 1) == q.QRNG_E_INVALID
    assert _call_extract(lib, 64, 0, 1) == q.QRNG_E_INVALID
    assert _call_extract(lib, 64, 64, 1) == q.QRNG_E_INVALID        # m >= n
    assert _call_extract(lib, 64, 100, 1) == q.QRNG_E_INVALID
    assert _call_extract(lib, 64, 32, 0) == q.QRNG_E_INVALID        # n_blocks = 0
    assert _call_extract(lib, 64, 32, 1, raw=0) == q.QRNG_E_INVALID  # NULL
    assert _call_extract(lib, 48, 32, 1) == q.QRNG_E_UNSUPPORTED    # n % 32
    assert _call_extract(lib, 1 << 26, (1 << 22), 1) == q.QRNG_E_UNSUPPORTED  # L > 2^26
    # NEXT-4 plans: bad world / rank are rejected before any device work
    h = ctypes.c_void_p()
    assert lib.qrng_dist_plan_create(1 << 24, 1 << 23, 16, 3, 0, None, ctypes.byref(h)) == q.QRNG_E_INVALID
    assert lib.qrng_dist_plan_create(1 << 24, 1 << 23, 16, 4, 4, None, ctypes.byref(h)) == q.QRNG_E_INVALID
    assert lib.qrng_dist_plan_create(1 << 26, 1 << 22, 16, 4, 0, None, ctypes.byref(h)) == q.QRNG_E_UNSUPPORTED
    assert "n=" in q.last_error() or "seed" in q.last_error() or "exceeds" in q.last_error()
    assert lib.qrng_minentropy(16, 0, 8, None, 1024, 0, 16, None) == q.QRNG_E_INVALID
    assert lib.qrng_minentropy(16, 10, 9, None, 1024, 0, 16, None) == q.QRNG_E_INVALID


def test_no_cpu_fallback_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    st = lib.qrng_toeplitz_extract_async(16, 1, 64, 32, 16, 4096, None)
    assert st == q.QRNG_E_CUDA
    assert "device" in q.last_error().lower()


@pytest.mark.parametrize("sigma,n,s", [(20.0, 1024, 0), (12.0, 1 << 20, 0), (20.0, 8192, 100)])
def test_entropy_finalise_matches_oracle(lib, sigma, n, s):
    x = qrng_synth.adc_samples(77, 1 << 18, 128.0, sigma)
    counts = E.histogram(x, 8)
    ref = E.report_from_counts(counts, 8, n, s)
    got = q.entropy_from_counts(counts, 8, n, s)
    for f in ("mu", "sigma", "h_min_hist", "h_min_ideal", "stat_dist", "delta_h_m", "h_min_mod"):
        assert getattr(got, f) == pytest.approx(getattr(ref, f), rel=1e-12, abs=1e-12), f
    assert got.m == ref.m and got.n_samples == ref.n_samples
    # supplied model
    got2 = q.entropy_from_counts(counts, 8, n, s, model=(128.0, sigma))
    ref2 = E.report_from_counts(counts, 8, n, s, model=(128.0, sigma))
    assert got2.h_min_ideal == pytest.approx(ref2.h_min_ideal, abs=1e-12)
    assert got2.m == ref2.m


def test_entropy_finalise_edge_cases(lib):
    c = np.zeros(256, np.uint64)
    c[3] = 10
    with pytest.raises(q.QrngError) as ei:  # point mass: fitted sigma = 0
        q.entropy_from_counts(c, 8, 1024, 0)
    assert ei.value.status == q.QRNG_E_INVALID
    c = np.zeros(256, np.uint64)
    c[40] = 5
    with pytest.raises(q.QrngError):  # value >= 2^5
        q.entropy_from_counts(c, 5, 1024, 0)
    x = qrng_synth.adc_samples(5, 1 << 16)
    counts = E.histogram(x, 8)
    r = q.entropy_from_counts(counts, 8, 64, 1000, allow_no_output=True)
    assert r.status == q.QRNG_E_NO_OUTPUT and r.m <= 0 and r.h_min_mod > 0
    with pytest.raises(q.QrngError):
        q.entropy_from_counts(counts, 8, 64, 1000)
    # uniform 8-bit histogram: H_min of the histogram is exactly 8
    u = np.full(256, 1000, np.uint64)
    assert q.entropy_from_counts(u, 8, 1024, 0, model=(127.5, 74.0), allow_no_output=True).h_min_hist == 8.0
