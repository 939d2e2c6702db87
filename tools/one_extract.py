#!/usr/bin/env python
"""Run a few one-shot extractions of one workload (for ncu captures).

    python tools/one_extract.py --config 2 [--karatsuba D] [--path gemm|ntt|auto] [--reps 2]
"""
import argparse, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import qrng_synth as S
import paper_2011_04130_b200 as q


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--karatsuba", type=int, default=-1)
    ap.add_argument("--path", default="auto")
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    q.load_library()
    if args.config == 124:  # NEXT-4's block length on one GPU: n = 2^24, 4 blocks (multi-pass NTT mod 7*2^26+1)
        w = S.Workload("next4_n2^24", 24, 1 << 24, 7 * (1 << 24) // 10, 4, 20.0)
    elif args.config == 41:  # config 4b: m of the bench's qrng_minentropy run (s = 0)
        w = S.config4b(594060)
    else:
        w = S.CONFIGS[args.config] if args.config in S.CONFIGS else S.sweep_workload(args.config)
    raw_np, seed_np = S.workload_inputs(w)
    raw, seed = torch.from_numpy(raw_np).cuda(), torch.from_numpy(seed_np).cuda()
    if args.path != "auto":
        q.set_debug_path({"gemm": q.PATH_GEMM, "ntt": q.PATH_NTT}[args.path])
    q.set_karatsuba(args.karatsuba)
    out = None
    for _ in range(args.reps):
        out = q.toeplitz_extract(raw, w.n_blocks, w.n, w.m, seed, out=out)
    torch.cuda.synchronize()
    print(f"{w.name}: {args.reps} extractions ok, {q.launch_count()} launches")


if __name__ == "__main__":
    main()
