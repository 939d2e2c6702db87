#!/usr/bin/env python
"""Benchmark: Toeplitz-extraction raw Gbit/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

One step = one pass of the whole hot path over one
batch: the one-shot C-ABI call qrng_toeplitz_extract_async on the rank's
blocks (seed preparation, output clear, extraction kernel, tail fix-up), with
raw bits and seed already resident in HBM.  The default workload is
BASELINE.json configs[1] (n = 8192, m = 5734, 16384 blocks).

Multi-GPU (torchrun, one process per GPU, NCCL): blocks are independent, so
each rank extracts its own batch of the config's size ("scaling": "weak"); the
seed is broadcast once from rank 0 (NCCL), nothing is exchanged in the timed
loop, and the time is the max over ranks of the summed CUDA-event step times.
L2 is flushed (256 MiB write) between timed steps, outside the events.

Also reported: the dominant kernel's roofline (CUDA events on its own stream
inside libqrng), the end-to-end number through the host-buffer C-ABI call,
the CPU oracle as cpu_baseline (rank 0, N=1), clocks sampled during the timed
region, and the number of libqrng kernel launches in the timed region.
"""
from __future__ import annotations

import argparse
import json
import math
import os
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


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback"


def workload(cfg: int) -> S.Workload:
    if cfg == 41:  # config 4b: m from qrng_minentropy, resolved in run_ours / run_reference
        return S.CONFIGS[4]
    if cfg in S.CONFIGS:
        return S.CONFIGS[cfg]
    if cfg >= 10:  # sweep point: --config 10..22 means config 5 at n = 2^cfg
        return S.sweep_workload(cfg)
    raise SystemExit(f"unknown config {cfg}")


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx, self.rows, self.proc = gpu_index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[3 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def algorithmic_work(path: int, w: S.Workload, n_blocks: int, pack: bool, modified: bool = False,
                     macs_per_block: int = 0):
    """Roofline numerators, per step of the main kernel(s)."""
    import paper_2011_04130_b200 as q
    if path == q.PATH_GEMM:
        # tensor-core ops (E2M1 or int8): 2 x the leaf MACs of the Karatsuba
        # decomposition (= 2 m n per block for the dense product, depth 0)
        return 2.0 * (macs_per_block or w.m * w.n) * n_blocks, "tensor", "TOPS"
    L = (w.n - 1) if modified else (w.n + w.m - 1)
    P = 1 << max(5, math.ceil(math.log2(L)))
    transforms = (n_blocks + 1) // 2 if pack else n_blocks
    bfly = transforms * (P * math.log2(P) + P)  # fwd + inv radix-2 butterflies (P/2 log P each) + P products
    return bfly, "alu", "Gbutterfly/s"


def ncu_traffic(workload_name: str, path_name: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel from the committed ncu --set full capture (profiles/ncu_traffic.json)."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        return t.get(f"{workload_name}/{path_name}", {}).get("bytes_per_launch")
    except Exception:
        return None


def ntt_two_blocks(w: S.Workload, modified: bool) -> bool:
    """Whether the fused NTT kernel packs two blocks per transform (ntt.cu
    choose_pack_shift): window sums <= n_len < 2^k and n_len (2^k + 1) < p, P <= 2^15."""
    n_len = w.n - w.m if modified else w.n
    L = (w.n - 1) if modified else (w.n + w.m - 1)
    k = n_len.bit_length()
    return L <= (1 << 15) and n_len * ((1 << k) + 1) < 998244353


def alu_peak_gbfly(pk):
    # 148 SMs x 4 SMSP x 32 lanes issue per clock at the max SM clock, over the
    # 7 integer instructions of one lazy Shoup butterfly.
    return 148 * 128 * pk.get("sm_max_mhz", 1965.0) * 1e6 / 7 / 1e9


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2011_04130_b200 as q

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; QRNG_BENCH_BACKEND=gloo lets the multi-rank plumbing be
    # smoke-tested with fewer GPUs than ranks (ranks never wait on each other)
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("QRNG_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    q.load_library()
    w = workload(args.config)
    B = w.n_blocks
    # rank r owns blocks [r*B, (r+1)*B) of a world*B-block stream (weak scaling)
    raw_np = S.adc_samples(w.key, B * w.n // 8, w.mu, w.sigma, start=rank * B * w.n // 8)
    entropy_info = None
    if args.config == 41:
        # config 4b: m from the corrected min-entropy of the samples,
        # s = 0; under torchrun the 256 counts of every rank's shard are summed
        counts = torch.zeros(256, dtype=torch.int64, device="cuda")
        samples = torch.from_numpy(raw_np).cuda()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        q.hist256_async(samples, counts)
        e1.record()
        if world > 1:
            from paper_2011_04130_b200 import dist as qd
            qd.allreduce_counts(counts)
        rep = q.entropy_from_counts(counts.cpu().numpy().astype(np.uint64), 8, w.n, 0)
        torch.cuda.synchronize()
        w = S.config4b(rep.m)
        entropy_info = {"m_from_minentropy": int(rep.m), "h_min_hist": rep.h_min_hist,
                        "h_min_ideal": rep.h_min_ideal, "stat_dist": rep.stat_dist,
                        "delta_h_m": rep.delta_h_m, "h_min_mod": rep.h_min_mod,
                        "hist_ms": e0.elapsed_time(e1)}
        del samples
    modified = args.variant == "modified"
    seed_np = S.uniform_bits(w.key, w.n, tag=9) if modified else S.workload_inputs(w, 0, 1)[1]
    seed = torch.empty(seed_np.size, dtype=torch.uint8, device="cuda")
    if rank == 0:
        seed.copy_(torch.from_numpy(seed_np))
    if world > 1:
        from paper_2011_04130_b200 import dist as qd
        qd.broadcast_seed(seed, 0)  # N1: the one collective, outside the timed loop
    raw = torch.from_numpy(raw_np).cuda()
    out = torch.empty(q.out_bytes(B, w.m), dtype=torch.uint8, device="cuda")
    if args.path != "auto":
        q.set_debug_path({"gemm": q.PATH_GEMM, "ntt": q.PATH_NTT}[args.path])
    q.set_karatsuba(args.karatsuba)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        if modified:  # [T | I_m] with an n-bit seed
            q.modified_toeplitz_extract(raw, B, w.n, w.m, seed, out=out, stream=stream)
        else:
            q.toeplitz_extract(raw, B, w.n, w.m, seed, out=out, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    with q.Plan(w.n, w.m, seed, modified=modified) as pl:
        path = pl.path
        pinfo = pl.info()
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
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = q.launch_count()
        for i in range(args.steps):
            flush.zero_()  # L2 flush, outside the events
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize()
        nl = q.launch_count() - l0
        if world > 1:
            dist.barrier()
        ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
        km, kn, _, _ = q.kernel_time_split()
        q.kernel_timing(False)
        return ms, nl, km, kn

    # timed region
    with ClockSampler(local) as clk:
        ms_total, launches, _, _ = timed_pass(False)
    # the same K steps again with the main kernel(s) timed live (roofline)
    ms_total_kt, _, kern_ms, kern_n = timed_pass(True)
    t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    bits_all = float(w.raw_bits) * world * args.steps
    value = bits_all / (ms_max * 1e-3) / 1e9

    # ---- steady state: the plan (seed preparation) reused ----
    with q.Plan(w.n, w.m, seed, modified=modified) as pl:
        for _ in range(args.warmup):
            pl.extract(raw, B, out=out, stream=stream)
        ss0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ss1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.zero_()
            ss0[i].record(stream)
            pl.extract(raw, B, out=out, stream=stream)
            ss1[i].record(stream)
        torch.cuda.synchronize()
    t_ss = torch.tensor([sum(a.elapsed_time(b) for a, b in zip(ss0, ss1))], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_ss, op=dist.ReduceOp.MAX)
    steady = {"value": bits_all / (float(t_ss.item()) * 1e-3) / 1e9, "unit": "Gbit/s",
              "ms_per_step": float(t_ss.item()) / args.steps,
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

    # ---- end to end from pinned HOST buffers through the public API ----
    # Streaming ingest (qrng_stream_*, the continuous-stream use of the paper):
    # every step copies its batch host->device, extracts it with the plan and
    # copies the key back; three steps in flight on their own streams.  Timed
    # on the host clock with full synchronisation on both sides (the work runs
    # on the library's internal streams), max over ranks.  Also reported: the
    # one-shot synchronous call (plan creation + chunked pipeline per step).
    e2e = None
    if not args.no_e2e and not modified:
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
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            for i in range(args.steps):
                qs.submit(hr, B, hos[i % depth])
            qs.synchronize()
            t_stream = time.perf_counter() - t0
        torch.cuda.synchronize()
        # one-shot synchronous host-buffer call (plan + chunked H2D/extract/D2H per step)
        for _ in range(2):
            q.toeplitz_extract_host(hr, B, w.n, w.m, hs, hos[0], stream=stream)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        for a, b in ev:
            flush.zero_()
            a.record(stream)
            q.toeplitz_extract_host(hr, B, w.n, w.m, hs, hos[0], stream=stream)
            b.record(stream)
        torch.cuda.synchronize()
        e_t = torch.tensor([t_stream * 1e3, sum(a.elapsed_time(b) for a, b in ev)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(e_t, op=dist.ReduceOp.MAX)
        e2e = {"value": bits_all / (float(e_t[0].item()) * 1e-3) / 1e9, "unit": "Gbit/s",
               "h2d_bytes_per_step": int(h_raw.numel()), "d2h_bytes_per_step": int(h_outs[0].numel()),
               "api": f"qrng_stream_submit (pinned host buffers, plan reused, {depth} batches in flight; "
                      "host clock, synchronised)",
               "oneshot_value": bits_all / (float(e_t[1].item()) * 1e-3) / 1e9,
               "oneshot_api": "qrng_toeplitz_extract_host per step (plan incl. seed prep, chunked pipeline; "
                              "CUDA events)",
               "oneshot_h2d_bytes_per_step": int(h_raw.numel() + h_seed.numel())}

    # ---- roofline of the dominant kernel ----
    pk, pk_kind = peaks()
    work, bound, unit = algorithmic_work(path, w, B, pack, modified, pinfo["macs_per_block"])
    roof = None
    if kern_n:
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
            # the measured bf16 x nominal-ratio peak undershoots what the E2M1 pipe
            # sustains (frac can exceed 1 on long-K leaves); against the pipe's own
            # live rate in the kernel's stage shape:
            roof["frac_of_mma_microbench"] = achieved / roof["peak_mma_microbench"]
            roof["ops_per_step"] = work
            roof["dense_ops_per_step"] = 2.0 * w.m * w.n * B  # the O(mn) product without Karatsuba
            # the same kernel time credited with the dense product's ops (> 1 = the
            # Karatsuba decomposition saved tensor work)
            roof["dense_equivalent_frac"] = roof["dense_ops_per_step"] / per_step_s / 1e12 / peak
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
            # the same butterflies with the inter-pass twiddle chains included
            # (the passes' whole register-resident instruction mix): the part of
            # the gap to `peak` the twiddles explain; the rest is shared-memory /
            # global traffic, barriers and occupancy
            roof["pass_rate_peak"] = q.butterfly_rate(with_twiddles=True) / 1e9
            roof["frac_of_pass_rate"] = achieved / roof["pass_rate_peak"]
        roof["frac"] = roof["achieved"] / roof["peak"]
        roof["traffic"] = ncu_traffic(w.name, {1: "gemm", 2: "ntt"}[path])
        roof["kernel_ms_per_step"] = kern_ms / args.steps  # summed per-launch device times
        roof["kernel_launches_per_step"] = kern_n / args.steps
        roof["kernel_share_of_step"] = (kern_ms / args.steps) / (ms_total_kt / args.steps)
        roof["kernel_timing"] = ("CUDA events on the kernel's launching stream, in a second pass of the same "
                                 "K steps (same inputs, same L2 flushes) right after the timed region")
        roof["ms_per_step_with_kernel_events"] = ms_total_kt / args.steps
        hbm_bytes = B * w.n / 8 + B * w.m / 8
        roof["hbm_gbs_algorithmic"] = hbm_bytes / per_step_s / 1e9
        if aux_n:
            # Karatsuba auxiliary stages (HBM/L2-bound): Q buffers (each reads its
            # two halves and writes itself: 3 x the X workspace) and combine +
            # pack (leaf parities in, packed key out)
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

    line = {
        "metric": METRIC, "value": value, "unit": "Gbit/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8 bits; int32 mod-p NTT" if path == 2 else (
            "u8 bits; E2M1 0/1 x E2M1 -> fp32 tensor core (kind::mxf4, unit scales, exact)"
            if q.gemm_operand_bits() == 4 else "u8 bits; int8 x int8 -> int32 tensor core"),
        "data": "synthetic: uint8 ADC samples clip(rint(N(128,sigma^2))) from PCG64 (qrng_synth); seeded uniform seed",
        "config": {"workload": w.name, "n": w.n, "m": w.m, "blocks_per_gpu": B,
                   "seed_bits": w.n if modified else w.seed_bits,
                   "raw_bits_per_gpu": w.raw_bits, "path": {1: "gemm", 2: "ntt"}[path],
                   "two_blocks_per_transform": bool(pack and path == 2),
                   "karatsuba_depth": pinfo["karatsuba_depth"] if path == 1 else None,
                   "karatsuba_leaves": pinfo["leaves"] if path == 1 else None,
                   "l2": "flushed between timed steps (256 MiB write, outside events)",
                   "variant": args.variant,
                   "step": ("one-shot qrng_modified_toeplitz_extract_async" if modified else
                            "one-shot qrng_toeplitz_extract_async") + " (seed prep + clear + extract)",
                   "parallelism": f"block-sharded x{world}"},
        "steady_state": steady,
        "roofline": roof, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk.summary(),
    }
    if entropy_info:
        line["config"]["minentropy"] = entropy_info
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w, budget_s=args.cpu_budget, modified=modified)
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline(w: S.Workload, budget_s: float = 15.0, threads: int = 0, modified: bool = False):
    """The oracle as it stands (word mode, OpenMP over blocks; the modified
    variant: its literal loop) on a bounded sample of the same workload:
    consecutive blocks until ~budget_s."""
    import oracle
    oracle.build()
    if threads == 0:
        threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else oracle.max_threads()
    cores = threads
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
            oracle.modified_extract(chunk, nb, w.n, w.m, seed, threads)
        else:
            oracle.extract(chunk, nb, w.n, w.m, seed, "words", threads)
        t_total += time.perf_counter() - t0
        blocks_done += nb
        pos += nb
        if t_total < budget_s / 8:
            nb = min(nb * 2, sample_blocks)
    return {"value": blocks_done * w.n / t_total / 1e9, "unit": "Gbit/s", "cores": cores,
            "kind": "oracle", "sample": f"{blocks_done} blocks (cycling over the first {sample_blocks} of "
                                        f"{w.n_blocks}) of {w.name}, {t_total:.1f} s, "
                                        + ("modified Toeplitz literal loop" if modified else "word-parallel mode")
                                        + ", OpenMP over blocks"}


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
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else oracle.max_threads()
    per_step_blocks = max(cores, min(w.n_blocks, int(os.environ.get("QRNG_REF_BLOCKS", "0")) or
                                     _ref_blocks(w, cores)))
    raw, seed = S.workload_inputs(w, 0, per_step_blocks)
    for _ in range(args.warmup):
        oracle.extract(raw[:cores * w.n // 8], cores, w.n, w.m, seed, "words", cores)
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
        "cpu_baseline": {"value": value, "unit": "Gbit/s", "cores": cores, "kind": "oracle", "sample": sample},
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
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--path", choices=["auto", "gemm", "ntt"], default="auto")
    ap.add_argument("--variant", choices=["standard", "modified"], default="standard",
                    help="modified = [T | I_m] with an n-bit seed (PAPER.md:253-267, NEXT-1)")
    ap.add_argument("--karatsuba", type=int, default=-1,
                    help="GEMM path: GF(2) Karatsuba depth (-1 = the library's cost model, 0 = dense)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
