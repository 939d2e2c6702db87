"""oracle/paper_fft.py (the paper's float-FFT method, Listing 2, PAPER.md:402-413,
used as a timed context row by bench.py) equals the oracle's key bytes."""
import numpy as np
import pytest

import qrng_synth as S


@pytest.mark.parametrize("n,m,B", [(1024, 716, 5), (3000, 1234, 3), (8192, 5734, 2), (96, 37, 7)])
def test_paper_fft_equals_oracle(oracle_mod, n, m, B):
    from oracle import paper_fft
    raw = S.random_bytes(n + m, (B * n + 7) // 8)
    seed = S.random_bytes(n + m, (n + m - 1 + 7) // 8, tag=4)
    assert np.array_equal(paper_fft.extract(raw, B, n, m, seed), oracle_mod.extract(raw, B, n, m, seed))
