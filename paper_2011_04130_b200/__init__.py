"""Python binding of libqrng.so (include/qrng.h) -- argument marshalling only.

B200-native Toeplitz-hashing randomness extraction after arXiv 2011.04130:
every step of the hot path runs in the CUDA kernels of ``csrc/``; this module
only turns torch tensors (device memory, streams) into pointers and status
codes into exceptions.  There is no CPU fallback: if ``libqrng.so`` is
missing or the device is not sm_100, calls raise.

Names follow the paper: n (block length, bits), m (output bits per block),
seed a = s (n+m-1 bits), raw r = x, key k = y.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# QRNG_LIB_PATH selects an experiment build (build.py --variant); default: the in-tree library
LIB_PATH = os.environ.get("QRNG_LIB_PATH") or os.path.join(_HERE, "libqrng.so")

QRNG_OK, QRNG_E_INVALID, QRNG_E_UNSUPPORTED, QRNG_E_NO_OUTPUT, QRNG_E_CUDA, QRNG_E_NOMEM = range(6)
PATH_AUTO, PATH_GEMM, PATH_NTT, PATH_BITS = 0, 1, 2, 3
STATUS_NAMES = {0: "QRNG_OK", 1: "QRNG_E_INVALID", 2: "QRNG_E_UNSUPPORTED", 3: "QRNG_E_NO_OUTPUT",
                4: "QRNG_E_CUDA", 5: "QRNG_E_NOMEM"}

# Every symbol include/qrng.h declares (checked by tests/test_abi.py).
EXPORTS = ["qrng_minentropy", "qrng_hist256_async", "qrng_entropy_from_counts",
           "qrng_toeplitz_extract", "qrng_toeplitz_extract_async", "qrng_toeplitz_extract_host",
           "qrng_plan_create", "qrng_plan_extract", "qrng_plan_destroy", "qrng_plan_path", "qrng_debug_last_path",
           "qrng_plan_create_modified", "qrng_modified_toeplitz_extract_async",
           "qrng_last_error", "qrng_version", "qrng_debug_set_path", "qrng_debug_launch_count",
           "qrng_debug_kernel_timing", "qrng_debug_kernel_time_ms", "qrng_debug_umma_probe",
           "qrng_debug_butterfly_rate", "qrng_debug_pass_rate", "qrng_debug_mxf4_probe", "qrng_debug_gemm_operand_bits", "qrng_debug_set_karatsuba", "qrng_plan_info",
           "qrng_debug_karatsuba_plan", "qrng_debug_qslice_plan", "qrng_debug_gemm_trace", "qrng_stream_create", "qrng_stream_submit",
           "qrng_stream_synchronize", "qrng_stream_counts", "qrng_stream_destroy", "qrng_debug_kernel_time_split",
           "qrng_debug_mma_rate", "qrng_dist_plan_create", "qrng_dist_exchange_words", "qrng_dist_local",
           "qrng_dist_finish", "qrng_dist_plan_destroy"]


class QrngError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class _Gauss(ctypes.Structure):
    _fields_ = [("mu", ctypes.c_double), ("sigma", ctypes.c_double)]


class _PlanInfo(ctypes.Structure):
    _fields_ = [("path", ctypes.c_int32), ("karatsuba_depth", ctypes.c_int32), ("leaves", ctypes.c_int32),
                ("log2_transform", ctypes.c_int32), ("blocks_per_transform", ctypes.c_int32),
                ("primes", ctypes.c_int32), ("macs_per_block", ctypes.c_uint64),
                ("x_words", ctypes.c_uint32), ("y_words", ctypes.c_uint32)]


class _Report(ctypes.Structure):
    _fields_ = [("counts", ctypes.c_uint64 * 256), ("n_samples", ctypes.c_uint64),
                ("bit_depth", ctypes.c_uint32), ("reserved", ctypes.c_uint32),
                ("mu", ctypes.c_double), ("sigma", ctypes.c_double),
                ("h_min_hist", ctypes.c_double), ("h_min_ideal", ctypes.c_double),
                ("stat_dist", ctypes.c_double), ("delta_h_m", ctypes.c_double),
                ("h_min_mod", ctypes.c_double), ("m", ctypes.c_int64)]


@dataclasses.dataclass
class EntropyReport:
    counts: np.ndarray
    n_samples: int
    bit_depth: int
    mu: float
    sigma: float
    h_min_hist: float
    h_min_ideal: float
    stat_dist: float
    delta_h_m: float
    h_min_mod: float
    m: int
    status: int


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libqrng.so (build it with ``python -m paper_2011_04130_b200.build``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run `python -m paper_2011_04130_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    vp, u64, u32, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
    sig = {
        "qrng_minentropy": ([vp, u64, u32, vp, u64, u32, vp, vp], i32),
        "qrng_hist256_async": ([vp, u64, vp, vp], i32),
        "qrng_entropy_from_counts": ([vp, u32, vp, u64, u32, vp], i32),
        "qrng_toeplitz_extract": ([vp, u64, u64, u64, vp, vp], i32),
        "qrng_toeplitz_extract_async": ([vp, u64, u64, u64, vp, vp, vp], i32),
        "qrng_toeplitz_extract_host": ([vp, u64, u64, u64, vp, vp, vp], i32),
        "qrng_plan_create": ([u64, u64, vp, vp, ctypes.POINTER(vp)], i32),
        "qrng_plan_extract": ([vp, vp, u64, vp, vp], i32),
        "qrng_plan_create_modified": ([u64, u64, vp, vp, ctypes.POINTER(vp)], i32),
        "qrng_modified_toeplitz_extract_async": ([vp, u64, u64, u64, vp, vp, vp], i32),
        "qrng_plan_destroy": ([vp], None),
        "qrng_plan_path": ([vp], i32),
        "qrng_debug_last_path": ([], i32),
        "qrng_last_error": ([], ctypes.c_char_p),
        "qrng_version": ([], ctypes.c_char_p),
        "qrng_debug_set_path": ([i32], None),
        "qrng_debug_launch_count": ([], u64),
        "qrng_debug_umma_probe": ([vp, vp, vp, i32, i32, vp], i32),
        "qrng_debug_butterfly_rate": ([i32, ctypes.POINTER(u64), vp], i32),
        "qrng_debug_pass_rate": ([i32, ctypes.POINTER(u64), vp], i32),
        "qrng_debug_mxf4_probe": ([vp, vp, vp, i32, i32, i32, vp], i32),
        "qrng_debug_gemm_operand_bits": ([], i32),
        "qrng_debug_kernel_timing": ([i32], None),
        "qrng_debug_kernel_time_ms": ([ctypes.POINTER(u64)], ctypes.c_double),
        "qrng_debug_set_karatsuba": ([i32], None),
        "qrng_debug_gemm_trace": ([vp, i32], i32),
        "qrng_debug_mma_rate": ([i32, i32, i32, ctypes.POINTER(u64), vp], i32),
        "qrng_stream_create": ([vp, u64, u32, u32, ctypes.POINTER(vp)], i32),
        "qrng_debug_kernel_time_split": ([ctypes.POINTER(ctypes.c_double), ctypes.POINTER(u64), ctypes.POINTER(u64)],
                                         ctypes.c_double),
        "qrng_stream_submit": ([vp, vp, u64, vp], i32),
        "qrng_stream_synchronize": ([vp], i32),
        "qrng_stream_counts": ([vp, vp], i32),
        "qrng_stream_destroy": ([vp], None),
        "qrng_plan_info": ([vp, vp], i32),
        "qrng_debug_karatsuba_plan": ([u64, u64, i32, vp, u32, vp, u32, vp, u32, vp], i32),
        "qrng_debug_qslice_plan": ([u64, u64, i32, vp, u32, vp, u32, vp], i32),
        "qrng_dist_plan_create": ([u64, u64, vp, u32, u32, vp, ctypes.POINTER(vp)], i32),
        "qrng_dist_exchange_words": ([vp], u64),
        "qrng_dist_local": ([vp, vp, vp, vp], i32),
        "qrng_dist_finish": ([vp, vp, vp, vp], i32),
        "qrng_dist_plan_destroy": ([vp], None),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def _check(status: int):
    if status != QRNG_OK:
        raise QrngError(status, load_library().qrng_last_error().decode())


def _stream_handle(stream) -> Optional[int]:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def _ptr(t) -> int:
    return t.data_ptr()


def _need_cuda_u8(t, name):
    import torch
    if not isinstance(t, torch.Tensor) or t.device.type != "cuda" or t.dtype != torch.uint8 \
            or not t.is_contiguous():
        raise TypeError(f"{name} must be a contiguous uint8 CUDA tensor")


def out_bytes(n_blocks: int, m: int) -> int:
    return (n_blocks * m + 7) // 8


def _need_bytes(t, nbytes: int, name: str):
    """The C ABI cannot see buffer sizes: refuse short buffers before any
    device read or write past their end (tensor numel or numpy size)."""
    size = t.numel() if hasattr(t, "numel") and not isinstance(t, np.ndarray) else t.size
    if size < nbytes:
        raise ValueError(f"{name} holds {size} bytes, needs at least {nbytes}")


def _same_device(*ts):
    devs = {t.device for t in ts}
    if len(devs) != 1:
        raise ValueError(f"tensors on different devices: {sorted(map(str, devs))}")


def _check_extract_buffers(raw, n_blocks: int, n: int, m: int, seed, seed_bits: int, out):
    """raw >= n_blocks*n/8 bytes, seed >= ceil(seed_bits/8), out >= ceil(n_blocks*m/8)."""
    if n_blocks < 0 or n < 0 or m < 0:
        raise ValueError("negative size")
    _need_bytes(raw, (n_blocks * n + 7) // 8, "raw")
    if seed is not None:
        _need_bytes(seed, (seed_bits + 7) // 8, "seed")
    _need_bytes(out, out_bytes(n_blocks, m), "out")


def version() -> str:
    return load_library().qrng_version().decode()


def last_error() -> str:
    return load_library().qrng_last_error().decode()


def set_debug_path(path: int) -> None:
    """TEST ONLY: force QRNG_PATH_GEMM / QRNG_PATH_NTT / QRNG_PATH_BITS for plans created afterwards."""
    load_library().qrng_debug_set_path(int(path))


def set_karatsuba(max_depth: int) -> None:
    """TEST/BENCH ONLY: Karatsuba depth of GEMM-path plans created afterwards
    (-1 = cost model, 0 = one dense product, d > 0 = split down to depth d)."""
    load_library().qrng_debug_set_karatsuba(int(max_depth))


@dataclasses.dataclass
class KaratsubaPlan:
    """Host planner output (qrng_debug_karatsuba_plan): see include/qrng.h."""
    depth: int
    leaves: list   # (r, w, out_off, seed_terms, input_terms)
    comb_ptr: np.ndarray
    comb_idx: np.ndarray


def karatsuba_plan(n: int, m: int, max_depth: int) -> KaratsubaPlan:
    """TEST ONLY (no GPU): the decomposition the library would run for (n, m)."""
    lib = load_library()
    counts = (ctypes.c_uint32 * 4)()
    _check(lib.qrng_debug_karatsuba_plan(n, m, max_depth, None, 0, None, 0, None, 0, counts))
    nl, nt, nc, depth = counts[0], counts[1], counts[2], counts[3]
    words = (m + 31) // 32
    leaf = np.zeros(6 * nl, np.uint32)
    terms = np.zeros(max(nt, 1), np.uint32)
    comb = np.zeros(words + 1 + nc, np.uint32)
    _check(lib.qrng_debug_karatsuba_plan(n, m, max_depth, leaf.ctypes.data, nl, terms.ctypes.data, nt,
                                         comb.ctypes.data, comb.size, counts))
    leaves = []
    for l in range(nl):
        r, w, off, t0, ns, ni = (int(v) for v in leaf[6 * l:6 * l + 6])
        leaves.append((r, w, off, [int(v) for v in terms[t0:t0 + ns]], [int(v) for v in terms[t0 + ns:t0 + ns + ni]]))
    return KaratsubaPlan(depth, leaves, comb[:words + 1].copy(), comb[words + 1:].copy())


def qslice_plan(n: int, m: int, max_depth: int):
    """TEST ONLY (no GPU): the one-pass Q-buffer chunk list of the plan for (n, m)
    (qrng_debug_qslice_plan): (slices, log2(s/128), chunks[], X-row words, leaf_x[l] = (src, word))."""
    lib = load_library()
    info = (ctypes.c_uint32 * 5)()
    _check(lib.qrng_debug_qslice_plan(n, m, max_depth, None, 0, None, 0, info))
    ns, lsu, ne, xw, nl = (int(v) for v in info)
    ent = np.zeros(max(ne, 1), np.uint32)
    lx = np.zeros(2 * max(nl, 1), np.uint32)
    _check(lib.qrng_debug_qslice_plan(n, m, max_depth, ent.ctypes.data, ne, lx.ctypes.data, nl, info))
    return ns, lsu, [int(v) for v in ent[:ne]], xw, [(int(lx[2 * l]), int(lx[2 * l + 1])) for l in range(nl)]


def gemm_trace(reset: bool = True) -> np.ndarray:
    """PROFILING ONLY (-DQRNG_GEMM_TIMELINE builds): the MMA-issue timeline,
    512 x (tag, t_start, t_info, t_acc, t_b, t_a, t_issued, 0), then one row
    per CTA (< 256): globaltimer ns at entry, first A stage ready, last MMA
    commit, exit, then the CTA's tile count."""
    c = np.zeros(8 * 768, np.uint64)
    _check(load_library().qrng_debug_gemm_trace(c.ctypes.data, 1 if reset else 0))
    return c.reshape(-1, 8)


def last_path() -> int:
    """BENCH/TEST ONLY: product path (PATH_*) of the most recent extraction."""
    return int(load_library().qrng_debug_last_path())


def launch_count() -> int:
    """Kernels launched by libqrng.so in this process (bench/test instrumentation)."""
    return int(load_library().qrng_debug_launch_count())


def kernel_timing(enable, aux: bool = True) -> None:
    """Time the main extraction kernel(s) with CUDA events (and, with aux, the auxiliary kernels)."""
    load_library().qrng_debug_kernel_timing((2 if aux else 1) if enable else 0)


def kernel_time_ms() -> tuple[float, int]:
    """(summed device ms, launches) of the main extraction kernel since the last read."""
    n = ctypes.c_uint64()
    ms = load_library().qrng_debug_kernel_time_ms(ctypes.byref(n))
    return float(ms), int(n.value)


def kernel_time_split() -> tuple[float, int, float, int]:
    """(main ms, main launches, auxiliary ms, auxiliary launches) since the last read."""
    aux, n, na = ctypes.c_double(), ctypes.c_uint64(), ctypes.c_uint64()
    ms = load_library().qrng_debug_kernel_time_split(ctypes.byref(aux), ctypes.byref(n), ctypes.byref(na))
    return float(ms), int(n.value), float(aux.value), int(na.value)


def mma_rate(form: int, n: int, iters: int = 20000, stream=None) -> float:
    """PROFILING ONLY: MAC/s of back-to-back MMAs of one form (see qrng.h)."""
    import torch
    macs = ctypes.c_uint64()
    s = torch.cuda.current_stream() if stream is None else stream
    _check(load_library().qrng_debug_mma_rate(form, 100, n, ctypes.byref(macs), s.cuda_stream))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    _check(load_library().qrng_debug_mma_rate(form, iters, n, ctypes.byref(macs), s.cuda_stream))
    b.record(s)
    b.synchronize()
    return macs.value / (a.elapsed_time(b) * 1e-3)


def butterfly_rate(iters: int = 2000, stream=None, with_twiddles: bool = False) -> float:
    """Achievable modular-butterfly rate (butterflies/s) of the NTT butterfly code
    (with_twiddles: each DFT followed by the inter-pass twiddle, qrng_debug_pass_rate)."""
    import torch
    n = ctypes.c_uint64()
    s = torch.cuda.current_stream() if stream is None else stream
    fn = load_library().qrng_debug_pass_rate if with_twiddles else load_library().qrng_debug_butterfly_rate
    _check(fn(8, ctypes.byref(n), s.cuda_stream))  # warm-up
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    _check(fn(iters, ctypes.byref(n), s.cuda_stream))
    b.record(s)
    b.synchronize()
    return n.value / (a.elapsed_time(b) * 1e-3)


def gemm_operand_bits() -> int:
    """4: the tensor-core path runs kind::mxf4 (E2M1, FP32 accumulate); 8: kind::i8."""
    return int(load_library().qrng_debug_gemm_operand_bits())


def mxf4_probe(A, h, N: int, K: int, hi_first: bool = False, stream=None):
    """TEST ONLY: D = A @ B^T on kind::mxf4 (E2M1 0/1, unit scales, FP32 accumulate), B[i][k] = h[i + k]."""
    import torch
    _need_cuda_u8(A, "A")
    _need_cuda_u8(h, "h")
    D = torch.empty((128, N), dtype=torch.float32, device=A.device)
    s = torch.cuda.current_stream() if stream is None else stream
    _check(load_library().qrng_debug_mxf4_probe(A.data_ptr(), h.data_ptr(), D.data_ptr(), N, K, 1 if hi_first else 0,
                                                s.cuda_stream))
    return D


def umma_probe(A, h, N: int, K: int, stream=None):
    """TEST ONLY: D = A @ B^T on the tcgen05 path, B[i][k] = h[i + k] (see qrng.h)."""
    import torch
    _need_cuda_u8(A, "A")
    _need_cuda_u8(h, "h")
    D = torch.empty((128, N), dtype=torch.int32, device=A.device)
    _check(load_library().qrng_debug_umma_probe(_ptr(A), _ptr(h), _ptr(D), N, K, _stream_handle(stream)))
    return D


def toeplitz_extract(raw, n_blocks: int, n: int, m: int, seed, out=None, stream=None):
    """Key bytes (C4) of n_blocks blocks: qrng_toeplitz_extract_async on `stream`."""
    import torch
    _need_cuda_u8(raw, "raw")
    _need_cuda_u8(seed, "seed")
    if out is None:
        out = torch.empty(out_bytes(n_blocks, m), dtype=torch.uint8, device=raw.device)
    _need_cuda_u8(out, "out")
    _same_device(raw, seed, out)
    _check_extract_buffers(raw, n_blocks, n, m, seed, n + m - 1, out)
    _check(load_library().qrng_toeplitz_extract_async(_ptr(raw), n_blocks, n, m, _ptr(seed), _ptr(out),
                                                      _stream_handle(stream)))
    return out


def modified_toeplitz_extract(raw, n_blocks: int, n: int, m: int, seed, out=None, stream=None):
    """Modified Toeplitz [T | I_m] with an n-bit seed (tensor-core path for n - m <= 2^16, else NTT)."""
    import torch
    _need_cuda_u8(raw, "raw")
    _need_cuda_u8(seed, "seed")
    if out is None:
        out = torch.empty(out_bytes(n_blocks, m), dtype=torch.uint8, device=raw.device)
    _need_cuda_u8(out, "out")
    _same_device(raw, seed, out)
    _check_extract_buffers(raw, n_blocks, n, m, seed, n, out)
    _check(load_library().qrng_modified_toeplitz_extract_async(_ptr(raw), n_blocks, n, m, _ptr(seed), _ptr(out),
                                                               _stream_handle(stream)))
    return out


def toeplitz_extract_host(raw: np.ndarray, n_blocks: int, n: int, m: int, seed: np.ndarray,
                          out: np.ndarray, stream=None) -> np.ndarray:
    """End-to-end call with HOST buffers (numpy views; pinned memory recommended)."""
    for a in (raw, seed, out):
        if not (isinstance(a, np.ndarray) and a.dtype == np.uint8 and a.flags.c_contiguous):
            raise TypeError("host buffers must be contiguous uint8 numpy arrays")
    _check_extract_buffers(raw, n_blocks, n, m, seed, n + m - 1, out)
    _check(load_library().qrng_toeplitz_extract_host(raw.ctypes.data, n_blocks, n, m, seed.ctypes.data,
                                                     out.ctypes.data, _stream_handle(stream)))
    return out


class Plan:
    """Seed preparation once per (seed, n, m); extract many batches."""

    def __init__(self, n: int, m: int, seed, stream=None, modified: bool = False):
        _need_cuda_u8(seed, "seed")
        _need_bytes(seed, ((n if modified else n + m - 1) + 7) // 8, "seed")
        self.n, self.m = n, m
        self.device = seed.device
        h = ctypes.c_void_p()
        create = load_library().qrng_plan_create_modified if modified else load_library().qrng_plan_create
        _check(create(n, m, _ptr(seed), _stream_handle(stream), ctypes.byref(h)))
        self._h = h

    @property
    def path(self) -> int:
        return load_library().qrng_plan_path(self._h)

    def info(self) -> dict:
        """qrng_plan_info: path, Karatsuba depth / leaves / MACs per block, NTT length."""
        i = _PlanInfo()
        _check(load_library().qrng_plan_info(self._h, ctypes.byref(i)))
        return {k: getattr(i, k) for k, _ in _PlanInfo._fields_ if k != "reserved"}

    def extract(self, raw, n_blocks: int, out=None, stream=None):
        import torch
        _need_cuda_u8(raw, "raw")
        if out is None:
            out = torch.empty(out_bytes(n_blocks, self.m), dtype=torch.uint8, device=raw.device)
        _need_cuda_u8(out, "out")
        if raw.device != self.device or out.device != self.device:
            raise ValueError(f"plan lives on {self.device}; raw on {raw.device}, out on {out.device}")
        _check_extract_buffers(raw, n_blocks, self.n, self.m, None, 0, out)
        _check(load_library().qrng_plan_extract(self._h, _ptr(raw), n_blocks, _ptr(out),
                                                _stream_handle(stream)))
        return out

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            load_library().qrng_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class DistPlan:
    """NEXT-4: this rank's share of ONE block's extraction across `world` GPUs
    (qrng_dist_*, the distributed four-step NTT; see include/qrng.h).  The
    collectives between local() and finish() are the caller's
    (paper_2011_04130_b200.dist.extract_block_distributed)."""

    def __init__(self, n: int, m: int, seed, world: int, rank: int, stream=None):
        _need_cuda_u8(seed, "seed")
        _need_bytes(seed, (n + m - 1 + 7) // 8, "seed")
        self.n, self.m, self.world, self.rank = n, m, world, rank
        self.device = seed.device
        h = ctypes.c_void_p()
        _check(load_library().qrng_dist_plan_create(n, m, _ptr(seed), world, rank, _stream_handle(stream),
                                                     ctypes.byref(h)))
        self._h = h
        self.exchange_words = int(load_library().qrng_dist_exchange_words(self._h))

    def new_buffer(self):
        import torch
        return torch.empty(self.exchange_words, dtype=torch.int32, device=self.device)

    def local(self, block, buf, stream=None):
        """Spectrum slice k1 = rank of the block, * seed slice, inverse, twist -> buf (send chunks)."""
        import torch
        _need_cuda_u8(block, "block")
        _need_bytes(block, (self.n + 7) // 8, "block")
        if buf.dtype != torch.int32 or buf.numel() != self.exchange_words or not buf.is_contiguous():
            raise TypeError("buf must be a contiguous int32 tensor of exchange_words elements")
        _same_device(block, buf)
        _check(load_library().qrng_dist_local(self._h, _ptr(block), _ptr(buf), _stream_handle(stream)))
        return buf

    def finish(self, recv, key, stream=None):
        """ORs this rank's key bits into key (uint8, ceil(m/8) bytes, zeroed by the caller)."""
        import torch
        if recv.dtype != torch.int32 or recv.numel() != self.exchange_words or not recv.is_contiguous():
            raise TypeError("recv must be a contiguous int32 tensor of exchange_words elements")
        _need_cuda_u8(key, "key")
        _need_bytes(key, out_bytes(1, self.m), "key")
        _same_device(recv, key)
        _check(load_library().qrng_dist_finish(self._h, _ptr(recv), _ptr(key), _stream_handle(stream)))
        return key

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            load_library().qrng_dist_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


STREAM_HIST = 1


class Stream:
    """Streaming ingest (qrng_stream_*): host batches extracted with a reused
    plan, `depth` batches in flight (H2D / extraction / D2H overlap).  Host
    buffers (numpy uint8, pinned for overlap) must stay alive until the batch
    completes (synchronize(), or `depth` further submits)."""

    def __init__(self, plan: "Plan", max_blocks: int, depth: int = 3, hist: bool = False):
        h = ctypes.c_void_p()
        _check(load_library().qrng_stream_create(plan._h, max_blocks, depth, STREAM_HIST if hist else 0,
                                                 ctypes.byref(h)))
        self._h, self.plan = h, plan

    def submit(self, raw: np.ndarray, n_blocks: int, out: np.ndarray):
        for a in (raw, out):
            if not (isinstance(a, np.ndarray) and a.dtype == np.uint8 and a.flags.c_contiguous):
                raise TypeError("host buffers must be contiguous uint8 numpy arrays")
        if raw.size * 8 < n_blocks * self.plan.n or out.size < out_bytes(n_blocks, self.plan.m):
            raise ValueError("buffer too small")
        _check(load_library().qrng_stream_submit(self._h, raw.ctypes.data, n_blocks, out.ctypes.data))

    def synchronize(self):
        _check(load_library().qrng_stream_synchronize(self._h))

    def counts(self) -> np.ndarray:
        c = np.zeros(256, np.uint64)
        _check(load_library().qrng_stream_counts(self._h, c.ctypes.data))
        return c

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            load_library().qrng_stream_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def _report(rep: _Report, status: int) -> EntropyReport:
    return EntropyReport(np.array(rep.counts[:], dtype=np.uint64), rep.n_samples, rep.bit_depth, rep.mu,
                         rep.sigma, rep.h_min_hist, rep.h_min_ideal, rep.stat_dist, rep.delta_h_m,
                         rep.h_min_mod, rep.m, status)


def minentropy(samples, bit_depth: int = 8, n: int = 0, s: int = 0, model=None, stream=None,
               allow_no_output: bool = False) -> EntropyReport:
    """qrng_minentropy: device histogram + host H_min / Delta H_m / m (synchronous)."""
    _need_cuda_u8(samples, "samples")
    rep = _Report()
    g = _Gauss(*model) if model is not None else None
    st = load_library().qrng_minentropy(_ptr(samples), samples.numel(), bit_depth,
                                        ctypes.byref(g) if g is not None else None, n, s,
                                        ctypes.byref(rep), _stream_handle(stream))
    if not (st == QRNG_OK or (allow_no_output and st == QRNG_E_NO_OUTPUT)):
        _check(st)
    return _report(rep, st)


def hist256_async(samples, counts, stream=None):
    """Accumulate the shard's histogram into counts (uint64[256] CUDA tensor, caller-zeroed)."""
    import torch
    _need_cuda_u8(samples, "samples")
    if counts.dtype not in (torch.int64, torch.uint64) or counts.numel() != 256 or counts.device.type != "cuda":
        raise TypeError("counts must be a 256-element 64-bit CUDA tensor")
    _same_device(samples, counts)
    _check(load_library().qrng_hist256_async(_ptr(samples), samples.numel(), _ptr(counts),
                                             _stream_handle(stream)))
    return counts


def entropy_from_counts(counts: np.ndarray, bit_depth: int = 8, n: int = 0, s: int = 0, model=None,
                        allow_no_output: bool = False) -> EntropyReport:
    c = np.ascontiguousarray(np.asarray(counts, dtype=np.uint64))
    if c.size != 256:
        raise ValueError("counts must have 256 entries")
    rep = _Report()
    g = _Gauss(*model) if model is not None else None
    st = load_library().qrng_entropy_from_counts(c.ctypes.data, bit_depth,
                                                 ctypes.byref(g) if g is not None else None, n, s,
                                                 ctypes.byref(rep))
    if not (st == QRNG_OK or (allow_no_output and st == QRNG_E_NO_OUTPUT)):
        _check(st)
    return _report(rep, st)
