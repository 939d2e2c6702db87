"""Parity of the tcgen05 kernel under every work distribution: the tile-run
order (QRNG_GEMM_RUNS runs per CTA, QRNG_GEMM_RUNLEN tiles per run; uneven
runs, runs that cross N pairs and leaves, B-chunk reuse across tiles) and the
strided order, on plain (dense) and packed / deferred Karatsuba launches.  The
settings are read once per process, so each one runs in a subprocess.

Run on a B200:  python -m pytest tests -m gpu
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASE = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import qrng_synth as S, oracle, paper_2011_04130_b200 as q
oracle.build(); q.load_library()
q.set_debug_path(q.PATH_GEMM)
bad = []
# (n, m, blocks, karatsuba depth): plain dense (1 and 2 B chunks per tile), packed
# leaves (K <= 2048) at depths 1-3 and deferred leaves (K = 4096), ragged batches
for n, m, B, d in [(1024, 716, 1000, 0), (2048, 1433, 700, 0), (4096, 2867, 300, 1), (8192, 5734, 517, 2),
                   (8192, 4000, 130, 3), (16384, 11468, 257, 2), (16384, 9000, 64, 1), (4096, 100, 900, 1)]:
    q.set_karatsuba(d)
    raw = S.random_bytes(n + m + d, B * n // 8)
    seed = S.random_bytes(n + m + d, (n + m - 1 + 7) // 8, tag=5)
    dv = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint8)).cuda()
    got = q.toeplitz_extract(dv(raw), B, n, m, dv(seed)).cpu().numpy()
    if not np.array_equal(got, oracle.extract(raw, B, n, m, seed)):
        bad.append((n, m, B, d))
print("BAD", bad)
sys.exit(1 if bad else 0)
"""


@pytest.mark.parametrize("runs,runlen", [("", ""), ("0", ""), ("1", ""), ("3", ""), ("7", ""), ("", "5"), ("", "1")])
def test_work_distribution_parity(runs, runlen):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    env = dict(os.environ, QRNG_GEMM_RUNS=runs, QRNG_GEMM_RUNLEN=runlen)
    r = subprocess.run([sys.executable, "-c", CASE, ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
