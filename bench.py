#!/usr/bin/env python
"""Benchmark: Toeplitz-extraction raw Gbit/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]
                    [--scaling weak|strong] [--configs all|none|LIST] [--dry-run]

One step = one pass of the whole hot path over one
batch: the one-shot C-ABI call qrng_toeplitz_extract_async on the rank's
blocks (seed preparation, output clear, extraction kernel(s), tail fix-up),
with raw bits and seed already resident in HBM.  The headline workload is
BASELINE.json configs[1] (config 2: n = 8192, m = 5734, 16384 blocks), the
configuration the metric is quoted on; the default line also carries a
`configs` object with every other config (1, 3, 4a, 4b and the config-5
block-length sweep points over the full 2^30-bit stream), each timed the same
way, checked against the oracle and with its own roofline and CPU baseline.

Multi-GPU: `--gpus N` without torchrun re-launches this script under
`torch.distributed.run` with N local ranks (NCCL; gloo when the box has fewer
GPUs than ranks, and for --dry-run).  Under torchrun it reads
RANK/LOCAL_RANK/WORLD_SIZE.  Blocks are independent, so a
fixed stream of B_total blocks is split into contiguous ranges, rank r owning
[floor(r B_total / W), floor((r+1) B_total / W)) (SURVEY 8(e),
paper_2011_04130_b200.dist.shard_range):
  * weak   (default for configs 1-4): B_total = W x the config's blocks
           (per-GPU work fixed);
  * strong (default for config 5):    B_total = the config's blocks (the one
           fixed 2^30-bit sequence cut W ways).
The seed is broadcast once from rank 0 (NCCL), nothing is exchanged in the
timed loop, and the time is the max over ranks of the summed CUDA-event step
times; every rank checks its own shard against the oracle afterwards.
L2 is flushed (256 MiB write) between timed steps, outside the events.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import qrng_synth as S  # noqa: E402

METRIC = "Toeplitz extraction raw Gbit/s (1/2/4/8 B200), fraction of roofline"
# the default line's `configs` object: (label, --config code)
EXTRA_CONFIGS = [("cfg1", 1), ("cfg3", 3), ("cfg4a", 4), ("cfg4b", 41),
                 ("cfg5_n2^10", 10), ("cfg5_n2^13", 13), ("cfg5_n2^16", 16), ("cfg5_n2^18", 18),
                 ("cfg5_n2^19", 19), ("cfg5_n2^22", 22), ("next4_n2^24", 124)]


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback"


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def workload(cfg: int) -> S.Workload:
    if cfg == 41:  # config 4b: m from qrng_minentropy, resolved at run time
        return S.CONFIGS[4]
    if cfg in S.CONFIGS:
        return S.CONFIGS[cfg]
    if cfg >= 10:  # sweep point: --config 10..22 means config 5 at n = 2^cfg
        return S.sweep_workload(cfg)
    raise SystemExit(f"unknown config {cfg}")


def default_scaling(cfg: int) -> str:
    return "strong" if cfg >= 10 else "weak"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    # nvidia-smi's start-up (NVML initialisation) can stall this process's CUDA
    # calls for tens of ms -- measured as a single 36 ms step inside config 4's
    # timed region (tools/oneshot_jitter.py --smi 1), the "one-shot swing" of
    # round 1.  So the sampler is started before the warm-up, has delivered its
    # first sample before the timed region begins, and the summary keeps the
    # samples taken between mark_start() and mark_end().

    def __init__(self, gpu_index: int):
        self.idx, self.rows, self.proc = gpu_index, [], None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            deadline = time.monotonic() + 5.0
            while not self.rows and time.monotonic() < deadline:
                time.sleep(0.02)
            time.sleep(0.2)  # past nvidia-smi's start-up
        except Exception:
            self.proc = None
        return self

    def mark_start(self):
        self.t0 = time.monotonic()

    def mark_end(self):
        self.t1 = time.monotonic()
        if self.proc:  # one more sample period after a short timed region
            time.sleep(0.25)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append((time.monotonic(), parts))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()
            self.proc = None

    def summary(self):
        rows = self.rows
        if self.t0 is not None and self.t1 is not None:
            inside = [r for r in rows if self.t0 <= r[0] <= self.t1]
            # short regions hold no sample: the nearest ones within 0.3 s
            rows = inside or [r for r in rows if self.t0 - 0.3 <= r[0] <= self.t1 + 0.3]
        rows = [r[1] for r in rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[3 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


PATH_NAMES = {1: "gemm", 2: "ntt", 3: "bits"}


def algorithmic_work(q, path: int, w: S.Workload, n_blocks: int, pack: bool, modified: bool = False,
                     macs_per_block: int = 0, blocks_per_transform: int = 0, primes: int = 1):
    """Roofline numerators, per step of the main kernel(s)."""
    if path == q.PATH_GEMM:
        # tensor-core ops (E2M1 or int8): 2 x the leaf MACs of the Karatsuba
        # decomposition (= 2 m n per block for the dense product, depth 0)
        return 2.0 * (macs_per_block or w.m * w.n) * n_blocks, "tensor", "TOPS"
    if path == q.PATH_BITS:
        # the CUDA-core product: m n bit-MACs (AND + XOR) per block
        return float(w.m) * w.n * n_blocks, "alu", "Tbit-MAC/s"
    L = (w.n - 1) if modified else (w.n + w.m - 1)
    P = 1 << max(5, math.ceil(math.log2(L)))
    if blocks_per_transform:  # the plan says: groups of blocks_per_transform blocks, `primes` transforms each
        transforms = -(-n_blocks // blocks_per_transform) * max(1, primes)
    else:
        transforms = (n_blocks + 1) // 2 if pack else n_blocks
    # fwd + inv radix-2 butterflies (P/2 log P each) + P products per transform
    # (the packed three-prime form: 3 transforms per 4 blocks, CRT not counted)
    bfly = transforms * (P * math.log2(P) + P)
    return bfly, "alu", "Gbutterfly/s"


def ncu_traffic(workload_name: str, path_name: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel from a committed ncu --set full capture (profiles/ncu_traffic.json)."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        e = t.get(f"{workload_name}/{path_name}", {})
        return e.get("bytes_per_launch"), e.get("source")
    except Exception:
        return None, None


def ntt_two_blocks(w: S.Workload, modified: bool) -> bool:
    """Whether the fused NTT kernel packs two blocks per transform (ntt.cu
    choose_pack_shift): window sums <= n_len < 2^k and n_len (2^k + 1) < p, P <= 2^15."""
    n_len = w.n - w.m if modified else w.n
    L = (w.n - 1) if modified else (w.n + w.m - 1)
    k = n_len.bit_length()
    return L <= (1 << 15) and n_len * ((1 << k) + 1) < 998244353


def bits_peak_tmacs(pk):
    # the CUDA-core product's bound: bits.cu's unrolled loop issues 2 LDS.32
    # (seed window word, block word), 1 SHF, 1 LOP3 + 1.25 of loop overhead per
    # 32 bit-MACs per lane; the two shared-memory loads (one wavefront each: the
    # lanes read at most a few distinct words) at 1 per clock per SM bind before
    # the issue slots: 32 lanes x 32 MACs / 2 clocks per SM, 148 SMs, max SM clock
    return 148 * pk.get("sm_max_mhz", 1965.0) * 1e6 * 32 * 32 / 2 / 1e12


def alu_peak_gbfly(pk):
    # 148 SMs x 4 SMSP x 32 lanes issue per clock at the max SM clock, over the
    # 7 integer instructions of one lazy Shoup butterfly.
    return 148 * 128 * pk.get("sm_max_mhz", 1965.0) * 1e6 / 7 / 1e9


# ---------------------------------------------------------------------------
# process group
# ---------------------------------------------------------------------------

class Ctx:
    def __init__(self, args):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.dry = args.dry_run
        self.backend = None
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist
            self.dist = dist
            self.backend = os.environ.get("QRNG_BENCH_BACKEND", "gloo" if self.dry else "nccl")
        if not self.dry:
            import torch
            # one process per GPU; with QRNG_BENCH_BACKEND=gloo several ranks may
            # share a GPU (plumbing check) -- ranks never wait on each other in a kernel
            self.local = self.local % max(1, torch.cuda.device_count())
            torch.cuda.set_device(self.local)
        if self.world > 1:
            import torch
            if self.backend == "nccl":
                self.dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                self.dist.init_process_group(self.backend)

    @property
    def coll_device(self):
        return "cuda" if self.backend == "nccl" else "cpu"

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def allreduce(self, vals, op="max"):
        """All-reduce a list of floats (max or sum) over ranks."""
        if self.world == 1:
            return list(vals)
        import torch
        t = torch.tensor(vals, dtype=torch.float64, device=self.coll_device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX if op == "max" else self.dist.ReduceOp.SUM)
        return [float(v) for v in t.cpu().tolist()]

    def broadcast_seed(self, seed_np):
        """The seed drawn on rank 0 reaches every rank by one broadcast (N1)."""
        import torch
        dev = "cuda" if not self.dry else "cpu"
        seed = torch.empty(seed_np.size, dtype=torch.uint8, device=dev)
        if self.rank == 0:
            seed.copy_(torch.from_numpy(seed_np))
        if self.world > 1:
            from paper_2011_04130_b200 import dist as qd
            if self.coll_device == "cpu" and seed.device.type != "cpu":
                tmp = seed.cpu()
                qd.broadcast_seed(tmp, 0)
                seed.copy_(tmp)
            else:
                qd.broadcast_seed(seed, 0)
        return seed

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def launch_ranks(args) -> int:
    """--gpus N outside torchrun: re-run this script under torch.distributed.run
    with N local ranks on 127.0.0.1 (one process per GPU)."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    if args.dry_run:
        env["QRNG_BENCH_BACKEND"] = "gloo"
    else:
        try:
            import torch
            if torch.cuda.device_count() < args.gpus:
                env.setdefault("QRNG_BENCH_BACKEND", "gloo")
                print(f"bench: {torch.cuda.device_count()} GPU(s) for {args.gpus} ranks: gloo process group, "
                      "ranks share GPUs (no rank waits on another in a kernel)", file=sys.stderr)
        except Exception:
            pass
    env.setdefault("NCCL_DEBUG", "INFO")           # rank count visible in the NCCL init log
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("OMP_NUM_THREADS", "1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def head_start(stream, cycles: int = 4_000_000):
    """A ~2 ms device spin before the first timed step (outside every event):
    the host enqueues the timed steps while it runs, so a host-side stall at
    the start of the region (nvidia-smi's NVML queries take a driver lock,
    measured at 10 ms) is not counted as device time of step 0."""
    import torch
    with torch.cuda.stream(stream):
        torch.cuda._sleep(cycles)


# ---------------------------------------------------------------------------
# one workload
# ---------------------------------------------------------------------------

_RAW_CACHE: dict = {}


def shard_samples(w: S.Workload, b0: int, b1: int) -> np.ndarray:
    key = (w.key, w.mu, w.sigma, b0 * w.n // 8, (b1 - b0) * w.n // 8)
    if key not in _RAW_CACHE:
        _RAW_CACHE.clear()  # one stream at a time (config 5's points share theirs)
        _RAW_CACHE[key] = S.adc_samples(w.key, (b1 - b0) * w.n // 8, w.mu, w.sigma, start=b0 * w.n // 8)
    return _RAW_CACHE[key]


def parity_check(q, out_np: np.ndarray, raw_np: np.ndarray, seed_np: np.ndarray, w: S.Workload, B: int,
                 b_first: int, modified: bool, rows_per_block: int = 64, seed: int = 0):
    """The keys produced by the timed steps against the CPU oracle (after the
    timed region): first / last / middle / random blocks of this rank's shard,
    first and last rows plus random rows of each, bit for bit.  Returns
    (checked bits, mismatches, description)."""
    import oracle
    oracle.build()
    rng = np.random.default_rng(seed)
    blocks = sorted({0, B - 1, B // 2, *rng.integers(0, B, 3).tolist()})
    bl, rw = [], []
    for b in blocks:
        rows = np.unique(np.concatenate([[0, w.m - 1], rng.integers(0, w.m, rows_per_block)]))
        bl += [b] * rows.size
        rw += rows.tolist()
    bl, rw = np.array(bl, np.uint64), np.array(rw, np.uint64)
    if modified:
        ref = oracle.modified_rows(raw_np, bl, rw, w.n, w.m, seed_np)
    else:
        ref = oracle.extract_rows(raw_np, bl, rw, w.n, w.m, seed_np)
    pos = (bl * w.m + rw).astype(np.int64)
    got = (out_np[pos >> 3] >> (7 - (pos & 7))) & 1
    bad = int(np.count_nonzero(got != ref))
    gblocks = [b_first + b for b in blocks]
    return int(pos.size), bad, f"{pos.size} sampled key bits of blocks {gblocks}"


def measure(q, ctx: Ctx, args, cfg: int, *, headline: bool, cpu_budget: float):
    """Time one workload on this rank's shard; returns the JSON-able dict
    (rank 0's view, times max-reduced over ranks)."""
    import torch
    w = workload(cfg)
    scaling = args.scaling or default_scaling(cfg)
    W, r = ctx.world, ctx.rank
    from paper_2011_04130_b200 import dist as qd
    entropy_info = None
    if cfg == 41:
        # config 4b: m from the corrected min-entropy of config 4's
        # samples (s = 0); each rank histograms its share, the counts are summed
        c4 = S.CONFIGS[4]
        lo, hi = qd.shard_range(c4.n_blocks, r, W)
        samples = torch.from_numpy(shard_samples(c4, lo, hi)).cuda()
        counts = torch.zeros(256, dtype=torch.int64, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        q.hist256_async(samples, counts)
        e1.record()
        torch.cuda.synchronize()
        if W > 1:
            c = counts.to(ctx.coll_device)
            qd.allreduce_counts(c)
            counts.copy_(c)
        rep = q.entropy_from_counts(counts.cpu().numpy().astype(np.uint64), 8, c4.n, 0)
        w = S.config4b(rep.m)
        entropy_info = {"m_from_minentropy": int(rep.m), "h_min_hist": rep.h_min_hist,
                        "h_min_ideal": rep.h_min_ideal, "stat_dist": rep.stat_dist,
                        "delta_h_m": rep.delta_h_m, "h_min_mod": rep.h_min_mod,
                        "hist_ms": e0.elapsed_time(e1)}
        del samples
    B_total = w.n_blocks * W if scaling == "weak" else w.n_blocks
    b0, b1 = qd.shard_range(B_total, r, W)
    B = b1 - b0
    modified = args.variant == "modified"
    raw_np = shard_samples(w, b0, b1)
    seed_np = S.uniform_bits(w.key, w.n, tag=9) if modified else S.workload_inputs(w, 0, 1)[1]
    seed = ctx.broadcast_seed(seed_np)
    raw = torch.from_numpy(raw_np).cuda()
    out = torch.empty(q.out_bytes(B, w.m), dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        if modified:  # [T | I_m] with an n-bit seed
            q.modified_toeplitz_extract(raw, B, w.n, w.m, seed, out=out, stream=stream)
        else:
            q.toeplitz_extract(raw, B, w.n, w.m, seed, out=out, stream=stream)

    clk = ClockSampler(ctx.local).start()  # before the warm-up (see ClockSampler)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    oneshot_path = q.last_path()  # the product path the one-shot step ran (small batches: CUDA cores)
    with q.Plan(w.n, w.m, seed, modified=modified) as pl:
        path = pl.path
        pinfo = pl.info()
    if oneshot_path == q.PATH_BITS:
        path = q.PATH_BITS
    pack = ntt_two_blocks(w, modified)

    def timed_pass(kernel_events):
        """K steps, L2 flushed between them outside the step events.  With
        kernel_events the main extraction kernel(s) are also bracketed by CUDA
        event records on their own launching stream inside libqrng; those
        records sit between the chained kernels of a step (Q buffers -> leaf
        GEMM -> combine, programmatic dependent launch) and cost the chain its
        overlap (measured +9 us per config-2 step), so the headline pass runs
        without them and an identical second pass times the kernel."""
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        q.kernel_timing(kernel_events, aux=False)
        q.kernel_time_ms()  # clear
        ctx.barrier()
        torch.cuda.synchronize()
        head_start(stream)
        l0 = q.launch_count()
        for i in range(args.steps):
            flush.zero_()  # L2 flush, outside the events
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize()
        nl = q.launch_count() - l0
        ctx.barrier()
        per = [s.elapsed_time(e) for s, e in zip(starts, ends)]
        km, kn, _, _ = q.kernel_time_split()
        q.kernel_timing(False)
        return sum(per), per, nl, km, kn

    # timed region
    clk.mark_start()
    ms_total, per_step, launches, _, _ = timed_pass(False)
    clk.mark_end()
    clk.stop()
    out_np = out.cpu().numpy()  # the keys of the last timed step (checked below)
    # the same K steps again with the main kernel(s) timed live (roofline)
    ms_total_kt, _, _, kern_ms, kern_n = timed_pass(True)
    ms_max, = ctx.allreduce([ms_total], "max")
    bits_all = float(B_total) * w.n * args.steps
    value = bits_all / (ms_max * 1e-3) / 1e9

    # ---- steady state: the plan (seed preparation) reused ----
    with q.Plan(w.n, w.m, seed, modified=modified) as pl:
        for _ in range(args.warmup):
            pl.extract(raw, B, out=out, stream=stream)
        ss0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ss1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ctx.barrier()
        torch.cuda.synchronize()
        head_start(stream)
        for i in range(args.steps):
            flush.zero_()
            ss0[i].record(stream)
            pl.extract(raw, B, out=out, stream=stream)
            ss1[i].record(stream)
        torch.cuda.synchronize()
    t_ss, = ctx.allreduce([sum(a.elapsed_time(b) for a, b in zip(ss0, ss1))], "max")
    steady = {"value": bits_all / (t_ss * 1e-3) / 1e9, "unit": "Gbit/s", "ms_per_step": t_ss / args.steps,
              "step": "qrng_plan_extract with the plan created once (seed preparation excluded)"}

    # auxiliary kernels (Karatsuba Q buffers + combine/pack, modified repack/XOR):
    # timed in their own pass of the same steps, outside the timed region
    q.kernel_timing(True, aux=True)
    q.kernel_time_split()  # clear
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    _, _, aux_ms, aux_n = q.kernel_time_split()
    q.kernel_timing(False)

    # ---- the keys of the timed steps against the oracle (every rank, own shard) ----
    parity = None
    if not args.no_parity:
        t0 = time.perf_counter()
        nbits, bad, what = parity_check(q, out_np, raw_np, seed_np, w, B, b0, modified, seed=cfg * 131 + r)
        tot_bits, tot_bad = ctx.allreduce([nbits, bad], "sum")
        parity = {"status": "bit-exact" if tot_bad == 0 else f"MISMATCH ({int(tot_bad)} bits)",
                  "checked_bits": int(tot_bits), "mismatches": int(tot_bad),
                  "what": (f"every rank: {what.split(' of blocks')[0]} of its own shard (rank 0: "
                           f"{what.split('sampled key bits of ')[1]}) from the last timed step, "
                           "vs oracle_extract_rows" + (" (modified)" if modified else "")),
                  "check_s": time.perf_counter() - t0}

    # ---- end to end from pinned HOST buffers through the public API (headline) ----
    e2e = None
    if headline and not args.no_e2e and not modified:
        e2e = measure_e2e(q, ctx, args, w, B, raw_np, seed, bits_all, flush, stream)

    # ---- roofline of the dominant kernel ----
    roof = roofline(q, args, w, B, path, pack, modified, pinfo, kern_ms, kern_n, ms_total_kt, aux_ms, aux_n)

    res = {
        "value": value, "unit": "Gbit/s", "ms_per_step": ms_max / args.steps,
        "ms_per_step_median_rank0": statistics.median(per_step), "ms_per_step_min_rank0": min(per_step),
        "ms_per_step_max_rank0": max(per_step),
        "steady_state": steady, "roofline": roof, "parity": parity, "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "dtype": "u8 bits; int32 mod-p NTT" if path == q.PATH_NTT else
                 "u8 bits; 32-bit AND / XOR / popcount on the CUDA cores" if path == q.PATH_BITS else (
            "u8 bits; E2M1 0/1 x E2M1 -> fp32 tensor core (kind::mxf4, unit scales, exact)"
            if q.gemm_operand_bits() == 4 else "u8 bits; int8 x int8 -> int32 tensor core"),
        "config": {"workload": w.name, "n": w.n, "m": w.m, "blocks_total": B_total,
                   "blocks_per_gpu": w.n_blocks if scaling == "weak" else f"~{w.n_blocks / W:g}",
                   "blocks_rank0": B, "seed_bits": w.n if modified else w.seed_bits,
                   "raw_bits_total": B_total * w.n, "path": PATH_NAMES[path],
                   "two_blocks_per_transform": bool(pack and path == q.PATH_NTT),
                   "blocks_per_transform": pinfo["blocks_per_transform"] if path == q.PATH_NTT else None,
                   "ntt_primes": pinfo["primes"] if path == q.PATH_NTT else None,
                   "karatsuba_depth": pinfo["karatsuba_depth"] if path == q.PATH_GEMM else None,
                   "karatsuba_leaves": pinfo["leaves"] if path == q.PATH_GEMM else None,
                   "ntt_log2_transform": pinfo["log2_transform"] if path == q.PATH_NTT else None,
                   "l2": "flushed between timed steps (256 MiB write, outside events)",
                   "variant": args.variant,
                   "step": ("one-shot qrng_modified_toeplitz_extract_async" if modified else
                            "one-shot qrng_toeplitz_extract_async") + " (seed prep + clear + extract)",
                   "scaling": scaling,
                   "partition": (f"rank r of {W} owns blocks [floor(r*{B_total}/{W}), floor((r+1)*{B_total}/{W})) "
                                 f"of one {B_total}-block stream"),
                   "parallelism": f"block-sharded x{W}"},
        "e2e": e2e,
    }
    if entropy_info:
        res["config"]["minentropy"] = entropy_info
    if ctx.rank == 0 and ctx.world == 1 and cpu_budget > 0:
        res["cpu_baseline"] = cpu_baseline(w, budget_s=cpu_budget, modified=modified)
        if headline and not modified:
            res["cpu_baseline"]["paper_method"] = paper_method_baseline(w, budget_s=min(5.0, cpu_budget))
    del raw, out, flush
    torch.cuda.empty_cache()
    return res


def measure_e2e(q, ctx, args, w, B, raw_np, seed, bits_all, flush, stream):
    """Streaming ingest (qrng_stream_*, the continuous-stream use of the paper):
    every step copies its batch host->device, extracts it with the plan and
    copies the key back; three steps in flight on their own streams.  Timed
    on the host clock with full synchronisation on both sides (the work runs
    on the library's internal streams), max over ranks.  Also reported: the
    one-shot synchronous call (plan creation + chunked pipeline per step)."""
    import torch
    h_raw = torch.from_numpy(raw_np).pin_memory()
    h_seed = seed.cpu().pin_memory()
    depth = 3
    h_outs = [torch.empty(q.out_bytes(B, w.m), dtype=torch.uint8).pin_memory() for _ in range(depth)]
    hr, hs = h_raw.numpy(), h_seed.numpy()
    hos = [h.numpy() for h in h_outs]
    with q.Plan(w.n, w.m, seed) as splan, q.Stream(splan, B, depth=depth) as qs:
        for i in range(depth + 1):
            qs.submit(hr, B, hos[i % depth])
        qs.synchronize()
        torch.cuda.synchronize()
        ctx.barrier()
        t0 = time.perf_counter()
        for i in range(args.steps):
            qs.submit(hr, B, hos[i % depth])
        qs.synchronize()
        t_stream = time.perf_counter() - t0
    torch.cuda.synchronize()
    for _ in range(2):
        q.toeplitz_extract_host(hr, B, w.n, w.m, hs, hos[0], stream=stream)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a, b in ev:
        flush.zero_()
        a.record(stream)
        q.toeplitz_extract_host(hr, B, w.n, w.m, hs, hos[0], stream=stream)
        b.record(stream)
    torch.cuda.synchronize()
    t_s, t_o = ctx.allreduce([t_stream * 1e3, sum(a.elapsed_time(b) for a, b in ev)], "max")
    return {"value": bits_all / (t_s * 1e-3) / 1e9, "unit": "Gbit/s",
            "h2d_bytes_per_step": int(h_raw.numel()), "d2h_bytes_per_step": int(h_outs[0].numel()),
            "api": f"qrng_stream_submit (pinned host buffers, plan reused, {depth} batches in flight; "
                   "host clock, synchronised)",
            "oneshot_value": bits_all / (t_o * 1e-3) / 1e9,
            "oneshot_api": "qrng_toeplitz_extract_host per step (plan incl. seed prep, chunked pipeline; "
                           "CUDA events)",
            "oneshot_h2d_bytes_per_step": int(h_raw.numel() + h_seed.numel())}


def roofline(q, args, w, B, path, pack, modified, pinfo, kern_ms, kern_n, ms_total_kt, aux_ms, aux_n):
    pk, pk_kind = peaks()
    work, bound, unit = algorithmic_work(q, path, w, B, pack, modified, pinfo["macs_per_block"],
                                         pinfo.get("blocks_per_transform", 0), pinfo.get("primes", 1))
    if not kern_n:
        return None
    # the path's extraction kernel(s) of one step (GEMM and fused NTT: one
    # launch; multi-pass NTT: passes + segment kernels), CUDA events on the
    # launching stream inside libqrng
    per_step_s = kern_ms / args.steps * 1e-3
    if bound == "tensor":
        achieved = work / per_step_s / 1e12
        fp4 = q.gemm_operand_bits() == 4
        # the contraction's own dtype: E2M1 dense = 4 x bf16, int8 = 2 x bf16
        # (nominal ratios 9 / 4.5 / 2.25 PFLOP/s)
        ratio = 4.0 if fp4 else 2.0
        peak = pk["bf16_tflops"] * ratio
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOPS",
                "peak_kind": f"{pk_kind} bf16 x {ratio:g} ({'E2M1 kind::mxf4' if fp4 else 'int8'} nominal ratio)"}
        clk_mhz = pk.get("sm_max_mhz", 1965.0)
        macs_per_clk = 16384 if fp4 else 8192
        roof["peak_at_sm_max_clock"] = 148 * macs_per_clk * 2 * clk_mhz * 1e6 / 1e12
        # the tensor pipe measured live in the kernel's own stage shape (2 N tiles
        # of 192 per elected issue, back to back, no data movement)
        roof["peak_mma_microbench"] = 2 * q.mma_rate(5 if fp4 else 3, 192 | (192 << 9)) / 1e12
        roof["frac_of_clock_peak"] = achieved / roof["peak_at_sm_max_clock"]
        roof["frac_of_mma_microbench"] = achieved / roof["peak_mma_microbench"]
        roof["ops_per_step"] = work
        roof["dense_ops_per_step"] = 2.0 * w.m * w.n * B  # the O(mn) product without Karatsuba
        roof["dense_equivalent_frac"] = roof["dense_ops_per_step"] / per_step_s / 1e12 / peak
    elif path == q.PATH_BITS:
        achieved = work / per_step_s / 1e12
        roof = {"bound": "alu", "achieved": achieved, "peak": bits_peak_tmacs(pk), "unit": unit,
                "peak_kind": "derived shared-memory load bound of bits.cu's loop (2 LDS.32 per 32 bit-MACs "
                             "per lane, 1 LDS per clock per SM, 148 SMs at the max SM clock)",
                "note": "a small batch: latency-bound (launch, seed staging, one pass), not issue-bound"}
    else:
        # multi-pass batches overlap on two streams: the summed per-launch
        # times then exceed the step, so the butterflies are divided by the
        # device time of the whole step instead
        share = (kern_ms / args.steps) / (ms_total_kt / args.steps)
        if share > 1.0:
            per_step_s = ms_total_kt / args.steps * 1e-3
        achieved = work / per_step_s / 1e9
        peak = q.butterfly_rate() / 1e9
        roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": unit,
                "peak_kind": "measured live: register-resident radix-32 fwd+inv modular butterflies on all SMs "
                             "(qrng_debug_butterfly_rate, the kernels' own butterfly code)",
                "peak_derived_issue_bound": alu_peak_gbfly(pk)}
        roof["pass_rate_peak"] = q.butterfly_rate(with_twiddles=True) / 1e9
        roof["frac_of_pass_rate"] = achieved / roof["pass_rate_peak"]
        bpt, primes = pinfo.get("blocks_per_transform", 1), pinfo.get("primes", 1)
        if primes > 1:  # packed three-prime form: the same time credited with one transform per block
            roof["one_block_per_transform_equivalent_frac"] = achieved * bpt / primes / peak
            roof["work_note"] = (f"{primes} transforms per {bpt} blocks (packed three-prime form); "
                                 "butterflies counted as run, the CRT not counted")
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"], roof["traffic_source"] = ncu_traffic(w.name, PATH_NAMES[path])
    roof["kernel_ms_per_step"] = kern_ms / args.steps  # summed per-launch device times
    roof["kernel_launches_per_step"] = kern_n / args.steps
    roof["kernel_share_of_step"] = (kern_ms / args.steps) / (ms_total_kt / args.steps)
    roof["kernel_timing"] = ("CUDA events on the kernel's launching stream, in a second pass of the same "
                             "K steps (same inputs, same L2 flushes) right after the timed region")
    roof["ms_per_step_with_kernel_events"] = ms_total_kt / args.steps
    hbm_bytes = B * w.n / 8 + B * w.m / 8
    roof["hbm_gbs_algorithmic"] = hbm_bytes / per_step_s / 1e9
    if aux_n:
        aux_s = aux_ms / args.steps * 1e-3
        if modified:  # repack (n'/8 in, K/8 out) + XOR tail (m/8 raw, m/8 key read and written)
            kprod = (w.n - w.m + 127) // 128 * 128
            aux_bytes = B * ((w.n - w.m) / 8 + kprod / 8 + 3 * w.m / 8)
            aux_kernels = "modified_repack_kernel + modified_xor_tail_kernel"
        else:
            aux_bytes = B * (3 * 4.0 * pinfo["x_words"] + 4.0 * pinfo["y_words"] + w.m / 8)
            aux_kernels = "qbuf_kernel + combine/pack kernel"
        roof["aux"] = {"kernels": aux_kernels + " (own pass, outside the timed region)",
                       "ms_per_step": aux_ms / args.steps,
                       "launches_per_step": aux_n / args.steps, "bytes_per_step": aux_bytes,
                       "achieved_gbs": aux_bytes / aux_s / 1e9,
                       "frac_of_hbm": aux_bytes / aux_s / 1e9 / pk["hbm_gbs"]}
    return roof


def cpu_baseline(w: S.Workload, budget_s: float = 15.0, threads: int = 0, modified: bool = False):
    """The oracle as it stands (word mode, OpenMP over blocks; the modified
    variant: its literal loop) on a bounded sample of the same workload:
    consecutive blocks until ~budget_s."""
    import oracle
    oracle.build()
    cores = threads or host_cores()
    # word-mode cost ~ m*n/64 word operations per block at ~1e9 per core-second:
    # when even one block per core would blow the budget (config 5 at n >= 2^20:
    # 1.9e11 word operations per block at 2^22), time a subset of the rows of one
    # block (OpenMP over rows) and extrapolate to whole blocks -- labelled so
    est_batch_s = w.m * w.n / 64 / 1e9
    if not modified and est_batch_s > budget_s / 2:
        return cpu_baseline_rows(w, budget_s, cores)
    sample_blocks = min(w.n_blocks, 4096)
    raw, seed = S.workload_inputs(w, 0, sample_blocks)
    if modified:
        seed = S.uniform_bits(w.key, w.n, tag=9)
    blocks_done, t_total, nb, pos = 0, 0.0, max(1, min(cores, sample_blocks)), 0
    while t_total < budget_s:
        if pos + nb > sample_blocks:  # cycle over the sample
            pos = 0
        chunk = raw[pos * w.n // 8:(pos + nb) * w.n // 8]
        t0 = time.perf_counter()
        if modified:
            oracle.modified_extract(chunk, nb, w.n, w.m, seed, cores)
        else:
            oracle.extract(chunk, nb, w.n, w.m, seed, "words", cores)
        t_total += time.perf_counter() - t0
        blocks_done += nb
        pos += nb
        if t_total < budget_s / 8:
            nb = min(nb * 2, sample_blocks)
    return {"value": blocks_done * w.n / t_total / 1e9, "unit": "Gbit/s", "cores": cores,
            "cpu_model": cpu_model(), "kind": "oracle",
            "sample": f"{blocks_done} blocks (cycling over the first {sample_blocks} of "
                      f"{w.n_blocks}) of {w.name}, {t_total:.1f} s, "
                      + ("modified Toeplitz literal loop" if modified else "word-parallel mode")
                      + ", OpenMP over blocks"}


def paper_method_baseline(w: S.Workload, budget_s: float = 5.0):
    """Context row: the paper's own method (double-precision FFT, round, mod 2;
    Listing 2) in numpy on the host (oracle/paper_fft.py,
    checked against the oracle by tests/test_oracle_paper_fft.py), on a
    bounded sample of the workload -- like for like with the paper's Matlab
    figure (about 0.05 Gbit/s)."""
    from oracle import paper_fft
    nb = max(1, min(w.n_blocks, 64))
    raw, seed = S.workload_inputs(w, 0, nb)
    done, t = 0, 0.0
    while t < budget_s:
        t0 = time.perf_counter()
        paper_fft.extract(raw, nb, w.n, w.m, seed)
        t += time.perf_counter() - t0
        done += nb
    return {"value": done * w.n / t / 1e9, "unit": "Gbit/s", "kind": "paper float-FFT method (numpy rfft, "
            "Listing 2 with the prose window)", "threads": "numpy FFT (one core)",
            "sample": f"{done} blocks of {w.name} in {t:.1f} s"}


def cpu_baseline_rows(w: S.Workload, budget_s: float, cores: int):
    """Oracle timing for blocks too large to finish within the budget: rows
    [0, R) of block 0 (oracle_extract_rows, the same word-parallel formula,
    OpenMP over rows), extrapolated to m rows per block."""
    import oracle
    raw, seed = S.workload_inputs(w, 0, 1)
    R, t = max(cores, 64), 0.0
    while True:
        rows = np.arange(R, dtype=np.uint64)
        t0 = time.perf_counter()
        oracle.extract_rows(raw, np.zeros(R, np.uint64), rows, w.n, w.m, seed, cores)
        t = time.perf_counter() - t0
        if t > budget_s / 4 or R * 2 > w.m:
            break
        R *= 2
    per_block_s = t * w.m / R
    return {"value": w.n / per_block_s / 1e9, "unit": "Gbit/s", "cores": cores, "cpu_model": cpu_model(),
            "kind": "oracle", "extrapolated": True,
            "sample": f"rows [0, {R}) of block 0 of {w.name} in {t:.2f} s (word-parallel oracle_extract_rows, "
                      f"OpenMP over rows), EXTRAPOLATED to the block's {w.m} rows"}


def measure_next4(q, ctx, args, cpu_budget: float, n: int = 1 << 24, blocks: int = 4):
    """NEXT-4: ONE block across all ranks -- the distributed
    four-step NTT (qrng_dist_local, one all_to_all_single of N2 words per rank,
    qrng_dist_finish, an OR all-reduce of the key bytes) for `blocks` blocks of
    n = 2^24 bits per step (m = floor(0.7 n), L > 2^23: past the single-GPU
    prime's limit).  The exchange is a real data-path collective inside the
    timed region (NCCL); at N = 1 it is the single-GPU world-1 four-step.
    Block bits are replicated (2 MiB each); the seed is broadcast once."""
    import torch
    from paper_2011_04130_b200 import dist as qd
    m = 7 * n // 10
    W = ctx.world
    raw_np = S.adc_samples(24, blocks * n // 8)
    seed_np = S.uniform_bits(24, n + m - 1, tag=7)
    seed = ctx.broadcast_seed(seed_np)
    raw = torch.from_numpy(raw_np).cuda()
    stream = torch.cuda.current_stream()
    plan = q.DistPlan(n, m, seed, W, ctx.rank)
    send = plan.new_buffer()
    recv = torch.empty_like(send)
    kbytes = q.out_bytes(1, m)
    keys = torch.zeros(blocks, (kbytes + 3) // 4 * 4, dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    gloo = ctx.backend == "gloo"

    out1 = torch.empty(q.out_bytes(blocks, m), dtype=torch.uint8, device="cuda")

    def step():
        if W == 1:  # one GPU: the single-GPU API (multi-pass NTT mod 7*2^26+1 for L > 2^23)
            q.toeplitz_extract(raw, blocks, n, m, seed, out=out1, stream=stream)
            return
        keys.zero_()
        for b in range(blocks):
            plan.local(raw[b * n // 8:(b + 1) * n // 8], send, stream=stream)
            if W > 1:
                if gloo:
                    r_ = torch.empty(send.numel(), dtype=torch.int32)
                    ctx.dist.all_to_all_single(r_, send.cpu())
                    recv.copy_(r_)
                else:
                    ctx.dist.all_to_all_single(recv, send)
            plan.finish(recv if W > 1 else send, keys[b], stream=stream)
        if W > 1:
            k = keys.cpu() if gloo else keys
            ctx.dist.all_reduce(k, op=ctx.dist.ReduceOp.SUM)  # disjoint bits: SUM == OR
            if gloo:
                keys.copy_(k)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    q.kernel_timing(True, aux=False)
    q.kernel_time_split()
    ctx.barrier()
    torch.cuda.synchronize()
    head_start(stream)
    l0 = q.launch_count()
    t_wall0 = time.perf_counter()
    for i in range(args.steps):
        flush.zero_()
        starts[i].record(stream)
        step()
        ends[i].record(stream)
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall0
    launches = q.launch_count() - l0
    ctx.barrier()
    km, kn, _, _ = q.kernel_time_split()
    q.kernel_timing(False)
    ms = sum(a.elapsed_time(b) for a, b in zip(starts, ends))
    ms_max, = ctx.allreduce([ms], "max")
    bits = float(blocks) * n * args.steps
    value = bits / (ms_max * 1e-3) / 1e9
    if W == 1:  # the last block's key from the batched output stream
        allbits = np.unpackbits(out1.cpu().numpy())[(blocks - 1) * m:blocks * m]
        key_np = np.packbits(allbits)
    else:
        key_np = keys[-1, :kbytes].cpu().numpy()
    parity = None
    if not args.no_parity:
        import oracle
        oracle.build()
        rng = np.random.default_rng(124)
        rows = np.unique(np.concatenate([[0, 1, m - 2, m - 1], rng.integers(0, m, 256)])).astype(np.uint64)
        b = blocks - 1
        ref = oracle.extract_rows(raw_np, np.full(rows.size, b, np.uint64), rows, n, m, seed_np)
        pos = rows.astype(np.int64)
        got = (key_np[pos >> 3] >> (7 - (pos & 7))) & 1
        bad, = ctx.allreduce([float(np.count_nonzero(got != ref))], "sum")
        parity = {"status": "bit-exact" if bad == 0 else f"MISMATCH ({int(bad)} bits)",
                  "checked_bits": int(rows.size) * W, "mismatches": int(bad),
                  "what": f"{rows.size} sampled key bits of the last block on every rank, vs oracle_extract_rows"}
    # ALU roofline: every rank runs one local length-N2 convolution transform per block
    N2 = plan.exchange_words  # W = 1: the full transform length P
    bfly = blocks * (N2 * math.log2(N2) + N2)
    per_step_s = (km / args.steps * 1e-3) if kn else ms_max / args.steps * 1e-3
    peak = q.butterfly_rate() / 1e9
    roof = {"bound": "alu", "achieved": bfly / per_step_s / 1e9, "peak": peak, "unit": "Gbutterfly/s per GPU",
            "kernel_ms_per_step": km / args.steps, "kernel_share_of_step": (km / args.steps) / (ms / args.steps),
            "exchange_bytes_per_rank_per_block": N2 * 4 * (W - 1) / W if W > 1 else 0}
    roof["frac"] = roof["achieved"] / peak
    roof["traffic"], roof["traffic_source"] = ncu_traffic(f"next4_n2^{n.bit_length() - 1}", "ntt")
    plan.close()
    res = {"value": value, "unit": "Gbit/s", "ms_per_step": ms_max / args.steps, "roofline": roof,
           "parity": parity, "gpu_launches": int(launches), "wall_ms_per_step_rank0": t_wall / args.steps * 1e3,
           "dtype": "u8 bits; int32 mod-p NTT (p = 7*2^26+1)",
           "config": {"workload": f"next4_n2^{n.bit_length() - 1}", "n": n, "m": m, "blocks_per_step": blocks,
                      "log2_transform": int(math.log2(N2 * W)), "world": W,
                      "scaling": "strong (each block's transform split across the ranks)",
                      "step": ("one-shot qrng_toeplitz_extract_async on the batch (multi-pass NTT mod 7*2^26+1)"
                               if W == 1 else
                               "per block: qrng_dist_local -> all_to_all_single (N2 words per rank) -> "
                               "qrng_dist_finish; then one OR all-reduce of the keys"),
                      "backend": ctx.backend or "single GPU"}}
    if ctx.rank == 0 and ctx.world == 1 and cpu_budget > 0:
        res["cpu_baseline"] = cpu_baseline_rows(S.Workload("next4", 24, n, m, blocks, 20.0), cpu_budget, host_cores())
    del raw, keys, flush, send, recv, out1
    torch.cuda.empty_cache()
    return res


def run_ours(args):
    ctx = Ctx(args)
    if ctx.dry:
        return dry_run(ctx, args)
    import paper_2011_04130_b200 as q
    q.load_library()
    if args.path != "auto":
        q.set_debug_path({"gemm": q.PATH_GEMM, "ntt": q.PATH_NTT, "bits": q.PATH_BITS}[args.path])
    q.set_karatsuba(args.karatsuba)
    head = measure(q, ctx, args, args.config, headline=True,
                   cpu_budget=0 if args.no_cpu_baseline else args.cpu_budget)
    line = {"metric": METRIC, "value": head["value"], "unit": "Gbit/s", "n_gpus": ctx.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": head["config"]["scaling"], "vs_baseline": None,
            "dtype": head["dtype"],
            "data": "synthetic: uint8 ADC samples clip(rint(N(128,sigma^2))) from PCG64 (qrng_synth); "
                    "seeded uniform seed",
            "headline": (f"{head['config']['workload']} (BASELINE.json configs[1], the configuration the metric "
                         "is quoted on)" if args.config == 2 else head["config"]["workload"]),
            "config": head["config"]}
    for k in ("steady_state", "roofline", "e2e", "parity", "gpu_launches", "clocks", "cpu_baseline",
              "ms_per_step_median_rank0", "ms_per_step_min_rank0", "ms_per_step_max_rank0"):
        if k in head:
            line[k] = head[k]
    extra = []
    if args.configs == "all":
        extra = [c for c in EXTRA_CONFIGS if c[1] != args.config]
    elif args.configs not in ("none", ""):
        want = args.configs.split(",")
        extra = [c for c in EXTRA_CONFIGS if c[0] in want or str(c[1]) in want]
    if extra:
        t0 = time.perf_counter()
        line["configs"] = {}
        for label, code in extra:
            t1 = time.perf_counter()
            if code == 124:
                d = measure_next4(q, ctx, args, cpu_budget=0 if args.no_cpu_baseline else args.cpu_budget_extra)
            else:
                d = measure(q, ctx, args, code, headline=False,
                            cpu_budget=0 if args.no_cpu_baseline else args.cpu_budget_extra)
            d["wall_s"] = time.perf_counter() - t1
            line["configs"][label] = d
        line["configs_wall_s"] = time.perf_counter() - t0
    pars = [line.get("parity")] + [d.get("parity") for d in line.get("configs", {}).values()]
    if all(p is not None for p in pars):
        bad = sum(p["mismatches"] for p in pars)
        line["parity_all"] = ("bit-exact" if bad == 0 else f"MISMATCH ({bad} bits)") + \
            f" ({sum(p['checked_bits'] for p in pars)} sampled key bits over {len(pars)} workloads, every rank)"
    if ctx.rank == 0:
        print(json.dumps(line))
    ctx.close()


def dry_run(ctx: Ctx, args):
    """--dry-run: the multi-rank plumbing without CUDA work (CPU test): shard
    ranges, the seed broadcast and the max-over-ranks reduction."""
    from paper_2011_04130_b200 import dist as qd
    w = workload(args.config)
    scaling = args.scaling or default_scaling(args.config)
    B_total = w.n_blocks * ctx.world if scaling == "weak" else w.n_blocks
    b0, b1 = qd.shard_range(B_total, ctx.rank, ctx.world)
    seed_np = S.workload_inputs(w, 0, 1)[1]
    seed = ctx.broadcast_seed(seed_np if ctx.rank == 0 else np.zeros_like(seed_np))
    seed_ok = bool(np.array_equal(seed.numpy(), seed_np))
    shard_all = ctx.allreduce([0.0] * (2 * ctx.rank) + [b0, b1] + [0.0] * (2 * (ctx.world - ctx.rank - 1)), "sum")
    ok, = ctx.allreduce([1.0 if seed_ok else 0.0], "sum")
    t, = ctx.allreduce([float(ctx.rank + 1)], "max")
    if ctx.rank == 0:
        print(json.dumps({"metric": METRIC, "dry_run": True, "n_gpus": ctx.world, "backend": ctx.backend,
                          "scaling": scaling, "config": {"workload": w.name, "blocks_total": B_total},
                          "shards": [[int(shard_all[2 * i]), int(shard_all[2 * i + 1])] for i in range(ctx.world)],
                          "seed_broadcast_ok_ranks": int(ok), "max_over_ranks": t}))
    ctx.close()


def run_reference(args):
    """--impl reference: the CPU oracle (this tier's reference arm), rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import oracle
    oracle.build()
    w = workload(args.config)
    if args.config == 41:
        from oracle import entropy as E
        w = S.config4b(E.report(S.workload_inputs(w)[0], 8, w.n, 0).m)
    # all host cores (torchrun sets OMP_NUM_THREADS=1 for its workers)
    cores = host_cores()
    if w.m * w.n / 64 / 1e9 > 10.0:
        # blocks too large for whole-block steps (config 5 at n >= 2^20): each
        # step times a subset of one block's rows, extrapolated (labelled)
        ts, cb = [], None
        for _ in range(args.steps):
            t0 = time.perf_counter()
            cb = cpu_baseline_rows(w, 8.0, cores)
            ts.append(time.perf_counter() - t0)
        value = cb["value"]
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": value, "unit": "Gbit/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": w.n / (value * 1e9) * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64 bit words",
            "data": "synthetic (qrng_synth)", "config": {"workload": w.name, "n": w.n, "m": w.m},
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": "Gbit/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return
    per_step_blocks = max(cores, min(w.n_blocks, int(os.environ.get("QRNG_REF_BLOCKS", "0")) or
                                     _ref_blocks(w, cores)))
    per_step_blocks = min(per_step_blocks, w.n_blocks)
    raw, seed = S.workload_inputs(w, 0, per_step_blocks)
    for _ in range(args.warmup):
        nb = min(cores, per_step_blocks)
        oracle.extract(raw[:nb * w.n // 8], nb, w.n, w.m, seed, "words", cores)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.extract(raw, per_step_blocks, w.n, w.m, seed, "words", cores)
        ts.append(time.perf_counter() - t0)
    total = sum(ts)
    value = per_step_blocks * w.n * args.steps / total / 1e9
    sample = f"{per_step_blocks} of {w.n_blocks} blocks of {w.name} per step (word-parallel oracle, OpenMP)"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Gbit/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64 bit words",
        "data": "synthetic (qrng_synth)", "config": {"workload": w.name, "n": w.n, "m": w.m,
                                                     "blocks_per_step": per_step_blocks},
        "cpu_baseline": {"value": value, "unit": "Gbit/s", "cores": cores, "cpu_model": cpu_model(),
                         "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "Gbit/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def _ref_blocks(w: S.Workload, cores: int) -> int:
    # ~ m*n/64 word ops per block at ~1e9 word-ops/s per core; aim for ~5 s per step
    per_block_s = w.m * w.n / 64 / 1.0e9
    return int(max(1, min(w.n_blocks, 5.0 * cores / per_block_s)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2,
                    help="1..4 = BASELINE configs, 41 = config 4b, 10..22 = config 5 at n = 2^k")
    ap.add_argument("--configs", default="all",
                    help="extra workloads in the line's `configs` object: all | none | comma list "
                         "(labels or codes, e.g. cfg3,22)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default=None,
                    help="multi-GPU partition (default: weak for configs 1-4, strong for config 5)")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--path", choices=["auto", "gemm", "ntt", "bits"], default="auto")
    ap.add_argument("--variant", choices=["standard", "modified"], default="standard",
                    help="modified = [T | I_m] with an n-bit seed (PAPER.md:253-267, NEXT-1)")
    ap.add_argument("--karatsuba", type=int, default=-1,
                    help="GEMM path: GF(2) Karatsuba depth (-1 = the library's cost model, 0 = dense)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--cpu-budget-extra", type=float, default=3.0,
                    help="oracle seconds per workload of the `configs` object")
    ap.add_argument("--dry-run", action="store_true", help="multi-rank plumbing only, no CUDA work")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args))
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
