#!/usr/bin/env python
"""Host-buffer path probe: PCIe copy rates and qrng_toeplitz_extract_host time (config 2)."""
import os, sys, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import qrng_synth as S
import paper_2011_04130_b200 as q


def ev_time(fn, reps=10):
    s = torch.cuda.current_stream()
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    b.synchronize()
    return a.elapsed_time(b) / reps


w = S.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
raw, seed = S.workload_inputs(w)
h_raw = torch.from_numpy(raw).pin_memory()
d_raw = torch.empty_like(h_raw, device="cuda")
ob = q.out_bytes(w.n_blocks, w.m)
h_out = torch.empty(ob, dtype=torch.uint8).pin_memory()
d_out = torch.empty(ob, dtype=torch.uint8, device="cuda")
t_h2d = ev_time(lambda: d_raw.copy_(h_raw, non_blocking=True))
t_d2h = ev_time(lambda: h_out.copy_(d_out, non_blocking=True))
print(f"H2D {raw.nbytes/1e6:.1f} MB {t_h2d:.3f} ms = {raw.nbytes/t_h2d/1e6:.1f} GB/s; D2H {ob/1e6:.1f} MB {t_d2h:.3f} ms = {ob/t_d2h/1e6:.1f} GB/s")
hs = torch.from_numpy(seed).pin_memory().numpy()
hr, ho = h_raw.numpy(), h_out.numpy()
t = ev_time(lambda: q.toeplitz_extract_host(hr, w.n_blocks, w.n, w.m, hs, ho), reps=10)
print(f"extract_host {t:.3f} ms = {w.raw_bits/t/1e6:.1f} Gbit/s  (QRNG_HOST_CHUNKS={os.environ.get('QRNG_HOST_CHUNKS', '8')})")
