#!/usr/bin/env python
"""Config 5: block-length sweep over a fixed 2^30-bit raw sequence (PAPER.md:273-289,
Fig. 6 / Table 2 analogue), both GPU paths, one process.  Prints one JSON line per
(n, path) and the measured crossover.  Timing: CUDA events on the launching stream,
L2 flushed between steps, one-shot C-ABI call (seed prep included) per step.

    python tools/sweep.py [--steps K] [--warmup W] [--min 10] [--max 22] [--step 1]
"""
import argparse, json, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import qrng_synth as S
import paper_2011_04130_b200 as q


def time_path(path, raw, seed, w, steps, warmup, flush):
    q.set_debug_path(path)
    out = torch.empty(q.out_bytes(w.n_blocks, w.m), dtype=torch.uint8, device="cuda")
    try:
        for _ in range(warmup):
            q.toeplitz_extract(raw, w.n_blocks, w.n, w.m, seed, out=out)
        torch.cuda.synchronize()
        tot = 0.0
        for _ in range(steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            q.toeplitz_extract(raw, w.n_blocks, w.n, w.m, seed, out=out)
            b.record()
            torch.cuda.synchronize()
            tot += a.elapsed_time(b)
        return tot / steps, out
    finally:
        q.set_debug_path(q.PATH_AUTO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--min", type=int, default=10)
    ap.add_argument("--max", type=int, default=22)
    ap.add_argument("--step", type=int, default=1)
    ap.add_argument("--gemm-max", type=int, default=20, help="largest log2 n timed on the GEMM path")
    args = ap.parse_args()
    q.load_library()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    samples = torch.from_numpy(S.adc_samples(5, (1 << 30) // 8, 128.0, 20.0)).cuda()
    best = {}
    for k in range(args.min, args.max + 1, args.step):
        w = S.sweep_workload(k)
        seed = torch.from_numpy(S.workload_inputs(w, 0, 1)[1]).cuda()
        raw = samples[: w.n_blocks * w.n // 8]
        res = {}
        outs = {}
        for name, path in (("gemm", q.PATH_GEMM), ("ntt", q.PATH_NTT)):
            if name == "gemm" and w.n > (1 << args.gemm_max):
                continue
            ms, out = time_path(path, raw, seed, w, args.steps, args.warmup, flush)
            res[name] = ms
            outs[name] = out
            rec = {"n": w.n, "m": w.m, "blocks": w.n_blocks, "path": name, "ms": ms, "gbit_s": w.raw_bits / ms / 1e6}
            if name == "gemm":
                q.set_debug_path(path)
                with q.Plan(w.n, w.m, seed) as pl:
                    rec["karatsuba_depth"] = pl.info()["karatsuba_depth"]
                q.set_debug_path(q.PATH_AUTO)
            print(json.dumps(rec), flush=True)
        if len(outs) == 2:
            assert torch.equal(outs["gemm"], outs["ntt"]), f"paths disagree at n={w.n}"
        best[w.n] = min(res, key=res.get)
    print(json.dumps({"best_path_by_n": best}))


if __name__ == "__main__":
    main()
