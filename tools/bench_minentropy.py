#!/usr/bin/env python
"""Row a7: device histogram (qrng_hist256_async) and the full qrng_minentropy call
on uint8 ADC samples; CUDA events after warm-up; HBM roofline (1 B read per sample)."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_04130_b200 as q
import qrng_synth as S

q.load_library()
pk = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
for count, sigma in [(1 << 25, 12.0), (1 << 27, 20.0)]:
    x = torch.from_numpy(S.adc_samples(4, count, 128, sigma)).cuda()
    counts = torch.zeros(256, dtype=torch.int64, device="cuda")
    for _ in range(5):
        q.hist256_async(x, counts)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    a.record()
    for _ in range(reps):
        q.hist256_async(x, counts)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    gbs = count / (ms * 1e-3) / 1e9
    import time
    t0 = time.perf_counter()
    rep = q.minentropy(x, 8, 1 << 20, 0)
    t1 = time.perf_counter()
    print(json.dumps({"samples": count, "hist_ms": ms, "hist_GBps": gbs, "frac_of_hbm": gbs / pk["hbm_gbs"],
                      "minentropy_call_ms_wall": (t1 - t0) * 1e3, "m": rep.m}))
