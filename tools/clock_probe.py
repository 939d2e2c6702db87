#!/usr/bin/env python
"""SM clock under the tcgen05 kernel's sustained load, two ways: the in-kernel
estimate (clock64 cycles of the MMA role per CTA over the globaltimer span of
the grid, -DQRNG_GEMM_TRACE build via QRNG_LIB_PATH) and nvidia-smi samples
taken while the same extraction runs back to back.

    QRNG_LIB_PATH=.../libqrng_trace.so python tools/clock_probe.py --config 3 [--karatsuba 0] [--seconds 3]
"""
import argparse, json, os, subprocess, sys, threading, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import qrng_synth as S
import paper_2011_04130_b200 as q


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--karatsuba", type=int, default=0)
    ap.add_argument("--seconds", type=float, default=3.0)
    args = ap.parse_args()
    q.load_library()
    w = S.CONFIGS[args.config] if args.config in S.CONFIGS else S.sweep_workload(args.config)
    raw_np, seed_np = S.workload_inputs(w)
    raw, seed = torch.from_numpy(raw_np).cuda(), torch.from_numpy(seed_np).cuda()
    q.set_debug_path(q.PATH_GEMM)
    q.set_karatsuba(args.karatsuba)
    out = q.toeplitz_extract(raw, w.n_blocks, w.n, w.m, seed)
    torch.cuda.synchronize()
    samples, stop = [], threading.Event()

    def sampler():
        while not stop.is_set():
            r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                                "--format=csv,noheader,nounits", "-i", "0"], capture_output=True, text=True)
            samples.append(r.stdout.strip())
            time.sleep(0.05)
    th = threading.Thread(target=sampler)
    th.start()
    est = []
    t_end = time.time() + args.seconds
    while time.time() < t_end:
        q.gemm_trace(True)
        for _ in range(4):
            out = q.toeplitz_extract(raw, w.n_blocks, w.n, w.m, seed, out=out)
        torch.cuda.synchronize()
        c = q.gemm_trace(True)
        span_ns = int(c[14]) - (~int(c[15]) & (2**64 - 1))
        est.append(int(c[3]) / 148 / 4 / (span_ns / 4) if span_ns > 0 else None)  # cycles per CTA per launch / ns
    stop.set()
    th.join()
    print(json.dumps({"workload": w.name, "karatsuba": args.karatsuba,
                      "sm_ghz_in_kernel": est[len(est) // 2:][:5], "nvidia_smi": samples[len(samples) // 2:][:8]}))


if __name__ == "__main__":
    main()
