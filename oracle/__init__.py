"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product package ``paper_2011_04130_b200`` never imports it and shares no code
with it.

* :mod:`oracle.toeplitz_oracle.c` -- the extraction y = T x mod 2 written out
  from the definition, scalar and 64-bit word modes.
  Also the modified Toeplitz [T | I_m] of PAPER.md:253-267 (modified_extract).
* :mod:`oracle.entropy` -- H_min, statistical distance, Delta H_m, corrected
  H_min and the output length m.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "toeplitz_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (C11 + OpenMP).  No CUDA anywhere."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-std=c11", "-O2", "-fopenmp", "-fPIC", "-shared",
                               _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        u8p = ctypes.POINTER(ctypes.c_uint8)
        u64 = ctypes.c_uint64
        for name in ("oracle_extract_scalar", "oracle_extract_words"):
            f = getattr(lib, name)
            f.argtypes = [u8p, u64, u64, u64, u8p, u8p, ctypes.c_int]
            f.restype = ctypes.c_int
        lib.oracle_extract_blocks.argtypes = [u8p, ctypes.POINTER(u64), u64, u64, u64, u8p, u8p,
                                              ctypes.c_int, ctypes.c_int]
        lib.oracle_extract_blocks.restype = ctypes.c_int
        lib.oracle_extract_rows.argtypes = [u8p, ctypes.POINTER(u64), ctypes.POINTER(u64), u64, u64, u64,
                                            u8p, u8p, ctypes.c_int]
        lib.oracle_extract_rows.restype = ctypes.c_int
        lib.oracle_modified_extract.argtypes = [u8p, u64, u64, u64, u8p, u8p, ctypes.c_int]
        lib.oracle_modified_extract.restype = ctypes.c_int
        lib.oracle_modified_rows.argtypes = [u8p, ctypes.POINTER(u64), ctypes.POINTER(u64), u64, u64, u64,
                                             u8p, u8p, ctypes.c_int]
        lib.oracle_modified_rows.restype = ctypes.c_int
        lib.oracle_hist256.argtypes = [u8p, u64, ctypes.POINTER(u64)]
        lib.oracle_hist256.restype = None
        lib.oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _p(a: np.ndarray, t=ctypes.c_uint8):
    return a.ctypes.data_as(ctypes.POINTER(t))


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def extract(raw: np.ndarray, n_blocks: int, n: int, m: int, seed: np.ndarray,
            mode: str = "words", threads: int = 0) -> np.ndarray:
    """Concatenated key bytes (C4) for n_blocks blocks of n raw bits (C2, C3)."""
    raw = np.ascontiguousarray(raw, dtype=np.uint8)
    seed = np.ascontiguousarray(seed, dtype=np.uint8)
    if raw.size * 8 < n_blocks * n:
        raise ValueError("raw buffer too short")
    if seed.size * 8 < n + m - 1:
        raise ValueError("seed buffer too short")
    out = np.zeros((n_blocks * m + 7) // 8, dtype=np.uint8)
    fn = {"scalar": _load().oracle_extract_scalar, "words": _load().oracle_extract_words}[mode]
    rc = fn(_p(raw), n_blocks, n, m, _p(seed), _p(out), threads)
    if rc != 0:
        raise ValueError(f"oracle rejected arguments (n={n}, m={m}, n_blocks={n_blocks})")
    return out


def extract_blocks(raw: np.ndarray, ids, n: int, m: int, seed: np.ndarray,
                   mode: str = "words", threads: int = 0) -> np.ndarray:
    """Per-block keys for block ids (rows of ceil(m/8) bytes, MSB-first from bit 0)."""
    raw = np.ascontiguousarray(raw, dtype=np.uint8)
    seed = np.ascontiguousarray(seed, dtype=np.uint8)
    ids = np.ascontiguousarray(np.asarray(ids, dtype=np.uint64))
    if ids.size and raw.size * 8 < (int(ids.max()) + 1) * n:
        raise ValueError("raw buffer too short")
    out = np.zeros((ids.size, (m + 7) // 8), dtype=np.uint8)
    rc = _load().oracle_extract_blocks(_p(raw), _p(ids, ctypes.c_uint64), ids.size, n, m,
                                       _p(seed), _p(out), 0 if mode == "scalar" else 1, threads)
    if rc != 0:
        raise ValueError("oracle rejected arguments")
    return out


def extract_rows(raw: np.ndarray, blocks, rows, n: int, m: int, seed: np.ndarray,
                 threads: int = 0) -> np.ndarray:
    """y_i of block b for each (b, i) pair (0/1 uint8), word-parallel formula."""
    raw = np.ascontiguousarray(raw, dtype=np.uint8)
    seed = np.ascontiguousarray(seed, dtype=np.uint8)
    blocks = np.ascontiguousarray(np.asarray(blocks, dtype=np.uint64))
    rows = np.ascontiguousarray(np.asarray(rows, dtype=np.uint64))
    assert blocks.shape == rows.shape
    if blocks.size and raw.size * 8 < (int(blocks.max()) + 1) * n:
        raise ValueError("raw buffer too short")
    out = np.zeros(blocks.size, dtype=np.uint8)
    rc = _load().oracle_extract_rows(_p(raw), _p(blocks, ctypes.c_uint64), _p(rows, ctypes.c_uint64),
                                     blocks.size, n, m, _p(seed), _p(out), threads)
    if rc != 0:
        raise ValueError("oracle rejected arguments")
    return out


def modified_extract(raw: np.ndarray, n_blocks: int, n: int, m: int, seed: np.ndarray,
                     threads: int = 0) -> np.ndarray:
    """Modified Toeplitz [T | I_m] with an n-bit seed, literal loop."""
    raw = np.ascontiguousarray(raw, dtype=np.uint8)
    seed = np.ascontiguousarray(seed, dtype=np.uint8)
    if raw.size * 8 < n_blocks * n or seed.size * 8 < n:
        raise ValueError("buffer too short")
    out = np.zeros((n_blocks * m + 7) // 8, dtype=np.uint8)
    if _load().oracle_modified_extract(_p(raw), n_blocks, n, m, _p(seed), _p(out), threads) != 0:
        raise ValueError("oracle rejected arguments")
    return out


def modified_rows(raw: np.ndarray, blocks, rows, n: int, m: int, seed: np.ndarray,
                  threads: int = 0) -> np.ndarray:
    """Sampled outputs of the modified Toeplitz (word-parallel form of the same formula)."""
    raw = np.ascontiguousarray(raw, dtype=np.uint8)
    seed = np.ascontiguousarray(seed, dtype=np.uint8)
    blocks = np.ascontiguousarray(np.asarray(blocks, dtype=np.uint64))
    rows = np.ascontiguousarray(np.asarray(rows, dtype=np.uint64))
    out = np.zeros(blocks.size, dtype=np.uint8)
    rc = _load().oracle_modified_rows(_p(raw), _p(blocks, ctypes.c_uint64), _p(rows, ctypes.c_uint64),
                                      blocks.size, n, m, _p(seed), _p(out), threads)
    if rc != 0:
        raise ValueError("oracle rejected arguments")
    return out


def hist256(samples: np.ndarray) -> np.ndarray:
    samples = np.ascontiguousarray(samples, dtype=np.uint8)
    counts = np.zeros(256, dtype=np.uint64)
    _load().oracle_hist256(_p(samples), samples.size, _p(counts, ctypes.c_uint64))
    return counts


def block_bits_from_stream(out: np.ndarray, b: int, m: int) -> np.ndarray:
    """Bits of block b (m values, 0/1 uint8) from a concatenated key stream (C4)."""
    bits = np.unpackbits(out)  # MSB-first, matches C2
    return bits[b * m:(b + 1) * m]
