#!/usr/bin/env python
"""Streaming-ingest throughput vs batch count and depth (config 2): host-clock
time of N qrng_stream_submit calls + synchronize, pinned host buffers."""
import json, os, sys, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import qrng_synth as S
import paper_2011_04130_b200 as q

q.load_library()
w = S.CONFIGS[2]
raw_np, seed_np = S.workload_inputs(w)
seed = torch.from_numpy(seed_np).cuda()
hr = torch.from_numpy(raw_np).pin_memory().numpy()
B = w.n_blocks
for depth in (2, 3, 4):
    hos = [torch.empty(q.out_bytes(B, w.m), dtype=torch.uint8).pin_memory().numpy() for _ in range(depth)]
    with q.Plan(w.n, w.m, seed) as pl, q.Stream(pl, B, depth=depth) as qs:
        for i in range(depth + 2):
            qs.submit(hr, B, hos[i % depth])
        qs.synchronize()
        for steps in (20, 100):
            t0 = time.perf_counter()
            for i in range(steps):
                qs.submit(hr, B, hos[i % depth])
            qs.synchronize()
            t = time.perf_counter() - t0
            print(json.dumps({"depth": depth, "steps": steps, "gbit_s": w.raw_bits * steps / t / 1e9,
                              "ms_per_batch": 1e3 * t / steps}), flush=True)
