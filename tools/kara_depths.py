#!/usr/bin/env python
"""Karatsuba-over-GEMM calibration: for each workload and depth, the one-shot
step time (CUDA events, L2 flushed), the grouped tcgen05 kernel time (events
inside libqrng), leaves, and leaf MACs vs the dense m*n.  One JSON line each.

    python tools/kara_depths.py [--configs 2,3] [--log2n 14,17] [--depths 0,1,2,3,4,-1]
"""
import argparse, json, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import qrng_synth as S
import paper_2011_04130_b200 as q


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3")
    ap.add_argument("--log2n", default="")
    ap.add_argument("--depths", default="0,1,2,3,4,-1")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    q.load_library()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    wls = [S.CONFIGS[int(c)] for c in args.configs.split(",") if c]
    wls += [S.sweep_workload(int(k)) for k in args.log2n.split(",") if k]
    for w in wls:
        raw_np, seed_np = S.workload_inputs(w)
        raw, seed = torch.from_numpy(raw_np).cuda(), torch.from_numpy(seed_np).cuda()
        out = torch.empty(q.out_bytes(w.n_blocks, w.m), dtype=torch.uint8, device="cuda")
        ref = None
        for d in [int(x) for x in args.depths.split(",")]:
            if d == 0 and w.n > (1 << 16):
                continue
            q.set_debug_path(q.PATH_GEMM)
            q.set_karatsuba(d)
            try:
                with q.Plan(w.n, w.m, seed) as pl:
                    info = pl.info()
                for _ in range(args.warmup):
                    q.toeplitz_extract(raw, w.n_blocks, w.n, w.m, seed, out=out)
                torch.cuda.synchronize()
                q.kernel_timing(True)
                q.kernel_time_ms()
                tot = 0.0
                for _ in range(args.steps):
                    flush.zero_()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    q.toeplitz_extract(raw, w.n_blocks, w.n, w.m, seed, out=out)
                    b.record()
                    torch.cuda.synchronize()
                    tot += a.elapsed_time(b)
                kms, kn = q.kernel_time_ms()
                q.kernel_timing(False)
            finally:
                q.set_debug_path(q.PATH_AUTO)
                q.set_karatsuba(-1)
            o = out.cpu()
            same = None
            if ref is None:
                ref = o
            else:
                same = bool(torch.equal(o, ref))
            ms = tot / args.steps
            kms /= args.steps
            macs = info["macs_per_block"] * w.n_blocks
            print(json.dumps({"workload": w.name, "n": w.n, "m": w.m, "depth_req": d,
                              "depth": info["karatsuba_depth"], "leaves": info["leaves"],
                              "mac_ratio": info["macs_per_block"] / (w.n * w.m),
                              "step_ms": ms, "gbit_s": w.raw_bits / ms / 1e6,
                              "kernel_ms": kms, "kernel_tops": 2 * macs / (kms * 1e-3) / 1e12 if kms else None,
                              "kernel_share": kms / ms, "same_as_first": same}), flush=True)


if __name__ == "__main__":
    main()
