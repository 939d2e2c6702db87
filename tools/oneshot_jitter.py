#!/usr/bin/env python
"""Per-step device time and host enqueue time of one-shot calls (config 4 by
default): finds the occasional slow step and says whether the host call (an
allocation, a lazy load) or the device work took the time."""
import argparse, json, os, sys, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import qrng_synth as S
import paper_2011_04130_b200 as q

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--steps", type=int, default=100)
ap.add_argument("--flush", type=int, default=1)
ap.add_argument("--smi", type=int, default=0, help="1: start `nvidia-smi -lms 100` right before the timed loop")
a = ap.parse_args()
q.load_library()
w = S.CONFIGS[a.config] if a.config in S.CONFIGS else S.sweep_workload(a.config)
raw_np, seed_np = S.workload_inputs(w)
raw, seed = torch.from_numpy(raw_np).cuda(), torch.from_numpy(seed_np).cuda()
out = torch.empty(q.out_bytes(w.n_blocks, w.m), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
for _ in range(5):
    q.toeplitz_extract(raw, w.n_blocks, w.n, w.m, seed, out=out, stream=st)
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
host = []
smi = None
if a.smi:
    import subprocess
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "100"],
                           stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
for s0, s1 in ev:
    if a.flush:
        flush.zero_()
    s0.record(st)
    t0 = time.perf_counter()
    q.toeplitz_extract(raw, w.n_blocks, w.n, w.m, seed, out=out, stream=st)
    host.append((time.perf_counter() - t0) * 1e3)
    s1.record(st)
torch.cuda.synchronize()
if smi:
    smi.terminate()
dev = [s0.elapsed_time(s1) for s0, s1 in ev]
med = sorted(dev)[len(dev) // 2]
slow = [(i, round(d, 3), round(h, 3)) for i, (d, h) in enumerate(zip(dev, host)) if d > 1.3 * med]
print(json.dumps({"workload": w.name, "smi": a.smi, "median_ms": med, "max_ms": max(dev), "host_median_ms": sorted(host)[len(host) // 2],
                  "host_max_ms": max(host), "slow_steps(idx,dev_ms,host_ms)": slow}))
