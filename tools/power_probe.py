#!/usr/bin/env python
"""SM clock, power and throttle reasons while one workload's one-shot
extraction runs back to back for a few seconds (nvidia-smi every 50 ms),
plus the device time per call in that sustained regime.

    python tools/power_probe.py --config 2 --seconds 3
"""
import argparse, json, os, statistics, subprocess, sys, threading, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import qrng_synth as S
import paper_2011_04130_b200 as q

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--seconds", type=float, default=3.0)
a = ap.parse_args()
q.load_library()
w = S.CONFIGS[a.config] if a.config in S.CONFIGS else S.sweep_workload(a.config)
raw_np, seed_np = S.workload_inputs(w)
raw, seed = torch.from_numpy(raw_np).cuda(), torch.from_numpy(seed_np).cuda()
out = torch.empty(q.out_bytes(w.n_blocks, w.m), dtype=torch.uint8, device="cuda")
for _ in range(5):
    q.toeplitz_extract(raw, w.n_blocks, w.n, w.m, seed, out=out)
torch.cuda.synchronize()
rows = []
proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap,"
                         "clocks_event_reasons.hw_slowdown,temperature.gpu", "--format=csv,noheader,nounits",
                         "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
threading.Thread(target=lambda: [rows.append((time.monotonic(), l.strip())) for l in proc.stdout], daemon=True).start()
time.sleep(1.0)
t0 = time.monotonic()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
calls = 0
while time.monotonic() - t0 < a.seconds:
    for _ in range(20):
        q.toeplitz_extract(raw, w.n_blocks, w.n, w.m, seed, out=out)
    calls += 20
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
t1 = time.monotonic()
proc.terminate()
inside = [r[1].split(", ") for r in rows if t0 + 0.2 <= r[0] <= t1]
sm = [float(r[0]) for r in inside]
pw = [float(r[1]) for r in inside]
print(json.dumps({"workload": w.name, "calls": calls, "us_per_call": e0.elapsed_time(e1) * 1e3 / calls,
                  "gbit_s": calls * w.raw_bits / (e0.elapsed_time(e1) * 1e-3) / 1e9,
                  "sm_mhz_median": statistics.median(sm) if sm else None, "sm_mhz_min": min(sm) if sm else None,
                  "power_w_median": statistics.median(pw) if pw else None,
                  "power_cap_active_frac": sum(r[2] == "Active" for r in inside) / max(1, len(inside)),
                  "samples": len(inside)}))
