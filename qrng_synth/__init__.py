"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no Toeplitz product, no
entropy formula): it only draws the numbers both sides consume, so that the
oracle (``oracle/``) and the product (``paper_2011_04130_b200``) can be fed
identical bytes without importing each other.

Recipe (reading A18):

* ADC samples stand in for the paper's laser-phase-noise raw data
  (10 Gbit stream at PAPER.md:283):
  ``uint8(clip(rint(N(mu, sigma^2)), 0, 255))`` drawn with numpy PCG64 from
  ``SeedSequence([key, chunk])`` in chunks of 2**20 samples, so any rank can
  regenerate exactly its own shard.  ``np.rint`` rounds half to even.
* Under the MSB-first convention (C2) the uint8 sample array *is* the packed
  raw bitstream: sample q supplies raw bits 8q..8q+7, most significant first.
* The Toeplitz seed is uniform: ``ceil(L/8)`` bytes from PCG64 seeded with
  ``SeedSequence([key, 2**32 - 1, tag])``; pad bits past L are zeroed.
"""
from __future__ import annotations

import dataclasses
import numpy as np

CHUNK = 1 << 20  # samples per independently seeded chunk


@dataclasses.dataclass(frozen=True)
class Workload:
    """One BASELINE.json config: n-bit blocks, m output bits, n_blocks blocks."""
    name: str
    key: int          # SeedSequence key of the config
    n: int
    m: int
    n_blocks: int
    sigma: float
    mu: float = 128.0

    @property
    def seed_bits(self) -> int:
        return self.n + self.m - 1

    @property
    def raw_bits(self) -> int:
        return self.n * self.n_blocks

    @property
    def n_samples(self) -> int:
        return self.raw_bits // 8


# BASELINE.json "configs" (m stated literally there, m = floor(0.7 n)).
CONFIGS = {
    1: Workload("cfg1_n1024", 1, 1024, 716, 256, 20.0),
    2: Workload("cfg2_n8192", 2, 8192, 5734, 16384, 20.0),
    3: Workload("cfg3_n65536", 3, 65536, 45875, 4096, 20.0),
    4: Workload("cfg4a_n1048576", 4, 1048576, 734003, 256, 12.0),
}


def config4b(m: int) -> Workload:
    """Config 4b: config 4's samples with m from the corrected min-entropy
    (qrng_minentropy with s = 0; SURVEY reading A8).  Its seed (L = n + m - 1
    bits) is drawn with tag 1."""
    c4 = CONFIGS[4]
    return Workload("cfg4b_n1048576", 4, c4.n, int(m), c4.n_blocks, c4.sigma)


def sweep_workload(log2n: int) -> Workload:
    """Config 5: fixed 2**30-bit raw sequence, n = 2**log2n, m = floor(0.7 n)."""
    n = 1 << log2n
    return Workload(f"cfg5_n2^{log2n}", 5, n, (7 * n) // 10, (1 << 30) // n, 20.0)


def adc_samples(key: int, count: int, mu: float = 128.0, sigma: float = 20.0,
                start: int = 0) -> np.ndarray:
    """Samples [start, start+count) of stream `key`: uint8 clip(rint(N(mu,sigma^2)))."""
    out = np.empty(count, dtype=np.uint8)
    if count == 0:
        return out
    first, last = start // CHUNK, (start + count - 1) // CHUNK
    pos = 0
    for c in range(first, last + 1):
        rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([key, c])))
        v = rng.normal(mu, sigma, CHUNK)
        lo = max(start - c * CHUNK, 0)
        hi = min(start + count - c * CHUNK, CHUNK)
        seg = np.clip(np.rint(v[lo:hi]), 0, 255).astype(np.uint8)
        out[pos:pos + seg.size] = seg
        pos += seg.size
    return out


def uniform_bits(key: int, nbits: int, tag: int = 0) -> np.ndarray:
    """ceil(nbits/8) uniform bytes, MSB-first bit order, pad bits zeroed."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([key, 2**32 - 1, tag])))
    nbytes = (nbits + 7) // 8
    buf = rng.integers(0, 256, nbytes, dtype=np.uint8)
    pad = nbytes * 8 - nbits
    if pad:
        buf[-1] &= np.uint8((0xFF << pad) & 0xFF)
    return buf


def workload_inputs(w: Workload, first_block: int = 0, n_blocks: int | None = None):
    """(raw bytes for blocks [first_block, first_block+n_blocks), seed bytes)."""
    if n_blocks is None:
        n_blocks = w.n_blocks - first_block
    assert w.n % 8 == 0
    bpb = w.n // 8
    raw = adc_samples(w.key, n_blocks * bpb, w.mu, w.sigma, start=first_block * bpb)
    tag = w.n if w.key == 5 else (1 if w.name.startswith("cfg4b") else 0)
    return raw, uniform_bits(w.key, w.seed_bits, tag)


def random_bytes(key: int, nbytes: int, tag: int = 1) -> np.ndarray:
    """Uniform bytes for small parity cases (raw streams that are not ADC-shaped)."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([key, 2**32 - 2, tag])))
    return rng.integers(0, 256, nbytes, dtype=np.uint8)
