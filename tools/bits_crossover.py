#!/usr/bin/env python
"""Small-batch crossover between the CUDA-core product (QRNG_PATH_BITS) and the
dense tcgen05 kernel (QRNG_PATH_GEMM): device-event time per one-shot step
(256 MiB L2 flush between steps, outside the events) over block counts, for
the dense-GEMM block lengths.  Prints one JSON line per (n, B) with the
bit-MACs n m B: the AUTO threshold (api.cu bits_max_macs) sits where the
two times cross."""
import json, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import qrng_synth as S
import paper_2011_04130_b200 as q

q.load_library()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()


def timed(fn, steps=40):
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


for n in (1024, 2048, 4096):
    m = (7 * n) // 10
    for B in (16, 64, 256, 1024, 2048, 4096, 16384):
        raw_np = S.random_bytes(n + B, B * n // 8)
        seed_np = S.random_bytes(n + 1, (n + m - 1 + 7) // 8)
        raw, seed = torch.from_numpy(raw_np).cuda(), torch.from_numpy(seed_np).cuda()
        out = torch.empty(q.out_bytes(B, m), dtype=torch.uint8, device="cuda")
        res = {"n": n, "m": m, "B": B, "bit_macs": n * m * B}
        for name, path in (("bits", q.PATH_BITS), ("gemm", q.PATH_GEMM), ("auto", q.PATH_AUTO)):
            q.set_debug_path(path)
            res[f"{name}_us"] = timed(lambda: q.toeplitz_extract(raw, B, n, m, seed, out=out, stream=st))
            res[f"{name}_ran"] = {1: "gemm", 2: "ntt", 3: "bits"}.get(q.last_path())
        q.set_debug_path(q.PATH_AUTO)
        print(json.dumps(res), flush=True)
