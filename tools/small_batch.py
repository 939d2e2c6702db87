#!/usr/bin/env python
"""Latency of small batches (config 1 and friends): device-event time per
one-shot step and per plan-reused step, on the GEMM and NTT paths, for a few
block counts (256 MiB L2 flush between steps, outside the events)."""
import json, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import qrng_synth as S
import paper_2011_04130_b200 as q

q.load_library()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()


def timed(fn, steps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for s, e in ev:
        flush.zero_()
        s.record(st)
        fn()
        e.record(st)
    torch.cuda.synchronize()
    t = sorted(s.elapsed_time(e) * 1e3 for s, e in ev)
    return round(t[len(t) // 2], 2)


for n, m, B in [(1024, 716, 256), (1024, 716, 1024), (1024, 716, 4096), (2048, 1433, 256), (4096, 2867, 256)]:
    raw_np = S.random_bytes(1, B * n // 8)
    seed_np = S.random_bytes(2, (n + m - 1 + 7) // 8)
    raw, seed = torch.from_numpy(raw_np).cuda(), torch.from_numpy(seed_np).cuda()
    out = torch.empty(q.out_bytes(B, m), dtype=torch.uint8, device="cuda")
    res = {"n": n, "m": m, "B": B}
    for name, path in (("auto", q.PATH_AUTO), ("gemm", q.PATH_GEMM), ("ntt", q.PATH_NTT)):
        q.set_debug_path(path)
        res[f"{name}_oneshot_us"] = timed(lambda: q.toeplitz_extract(raw, B, n, m, seed, out=out, stream=st))
        with q.Plan(n, m, seed) as pl:
            res[f"{name}_steady_us"] = timed(lambda: pl.extract(raw, B, out=out, stream=st))
        q.kernel_timing(True, aux=True)
        q.kernel_time_split()
        for _ in range(20):
            q.toeplitz_extract(raw, B, n, m, seed, out=out, stream=st)
        torch.cuda.synchronize()
        km, kn, am, an = q.kernel_time_split()
        q.kernel_timing(False)
        res[f"{name}_kernel_us"] = round(km / 20 * 1e3, 2)
    q.set_debug_path(q.PATH_AUTO)
    print(json.dumps(res), flush=True)
