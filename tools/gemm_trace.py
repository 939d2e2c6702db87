#!/usr/bin/env python
"""Per-role cycle breakdown of the tcgen05 kernel (needs a -DQRNG_GEMM_TRACE
build loaded through QRNG_LIB_PATH).  Prints per-CTA averages in cycles.

    QRNG_LIB_PATH=.../libqrng_trace.so python tools/gemm_trace.py --config 2 [--karatsuba D]
"""
import argparse, json, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import qrng_synth as S
import paper_2011_04130_b200 as q

NAMES = ["mma_wait_a_full", "mma_wait_b_full", "mma_wait_acc_empty", "mma_total", "xf_wait_a_empty",
         "xf_expand_st", "xf_total", "bgen_wait_b_empty", "bgen_total", "epi_wait_acc_full", "epi_total",
         "stages", "mma_wait_acc_empty_nt1", "prologue", "", "", "mma_issue_blocks", "mma_tile_setup"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--karatsuba", type=int, default=0)
    args = ap.parse_args()
    q.load_library()
    w = S.CONFIGS[args.config] if args.config in S.CONFIGS else S.sweep_workload(args.config)
    raw_np, seed_np = S.workload_inputs(w)
    raw, seed = torch.from_numpy(raw_np).cuda(), torch.from_numpy(seed_np).cuda()
    q.set_debug_path(q.PATH_GEMM)
    q.set_karatsuba(args.karatsuba)
    out = q.toeplitz_extract(raw, w.n_blocks, w.n, w.m, seed)
    torch.cuda.synchronize()
    q.gemm_trace(True)
    q.kernel_timing(True)
    q.kernel_time_ms()
    out = q.toeplitz_extract(raw, w.n_blocks, w.n, w.m, seed, out=out)
    torch.cuda.synchronize()
    kms, _ = q.kernel_time_ms()
    q.kernel_timing(False)
    c = q.gemm_trace(True)
    ctas = 148
    res = {"workload": w.name, "karatsuba": args.karatsuba, "gemm_kernel_ms": kms}
    for i, n in enumerate(NAMES):
        if n:
            res[n] = int(c[i]) / (1 if n == "stages" else ctas)
    res["cta_span_us"] = (int(c[14]) - (~int(c[15]) & (2**64 - 1))) / 1e3
    # SM clock during the kernel: MMA-role cycles per CTA over the global span (a lower bound)
    res["sm_ghz_est"] = res["mma_total"] / (res["cta_span_us"] * 1e3) if res["cta_span_us"] > 0 else None
    # per-warp normalisation: xform counters are summed over 4*XF_PAR warps, b-gen 3, epilogue 8
    print(json.dumps(res))


if __name__ == "__main__":
    main()
