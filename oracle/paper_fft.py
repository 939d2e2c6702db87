"""The paper's own post-processing method -- TEST / BASELINE INFRASTRUCTURE ONLY.

Only ``tests/`` and ``bench.py``'s CPU-baseline leg may import this module
(it is a context row, not the oracle and not the product).

PAPER.md:199-241 (Sec. III.B, Def. 1-2) and Listing 2: the
key is a window of the cyclic convolution of the seed a (first column of the
circulant A) with the zero-padded raw block r', computed with a
double-precision FFT, rounded and reduced mod 2:

    k = round(ifft(fft(a) .* fft(r'))) mod 2,   keep k_n .. k_{n+m-1}

(the window of the prose; reading C1 of DESIGN.md).  The
transform length is L = n + m - 1 as in the listing (non-power-of-two sizes
included).  Checked against the oracle by
tests/test_oracle_toeplitz.py::test_paper_fft_method and
tests/test_oracle_paper_fft.py.
"""
from __future__ import annotations

import numpy as np


def extract(raw: np.ndarray, n_blocks: int, n: int, m: int, seed: np.ndarray) -> np.ndarray:
    """Key bytes (C4) of n_blocks blocks by the paper's float-FFT method."""
    L = n + m - 1
    a = np.unpackbits(np.asarray(seed, np.uint8))[:L].astype(np.float64)
    fa = np.fft.rfft(a, L)
    bits = np.unpackbits(np.asarray(raw, np.uint8))[:n_blocks * n].reshape(n_blocks, n).astype(np.float64)
    k = np.fft.irfft(np.fft.rfft(bits, L, axis=1) * fa[None, :], L, axis=1)
    y = (np.rint(k[:, n - 1:n + m - 1]).astype(np.int64) & 1).astype(np.uint8)
    return np.packbits(y.reshape(-1))
