#!/usr/bin/env python
"""Where the one-shot step's time goes beyond the steady-state extraction
(config 2 by default): device-event time per step of
  oneshot       qrng_toeplitz_extract_async (plan create + extract + release)
  oneshot+kt    the same with the bench's live kernel timing switched on
  steady        qrng_plan_extract with a reused plan
  plan          qrng_plan_create + qrng_plan_destroy alone
each with a 256 MiB L2 flush between steps outside the events."""
import argparse, json, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import qrng_synth as S
import paper_2011_04130_b200 as q

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--steps", type=int, default=30)
a = ap.parse_args()
q.load_library()
w = S.CONFIGS[a.config]
raw_np, seed_np = S.workload_inputs(w)
raw, seed = torch.from_numpy(raw_np).cuda(), torch.from_numpy(seed_np).cuda()
B = w.n_blocks
out = torch.empty(q.out_bytes(B, w.m), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    for s, e in ev:
        flush.zero_()
        s.record(st)
        fn()
        e.record(st)
    torch.cuda.synchronize()
    return sum(s.elapsed_time(e) for s, e in ev) / a.steps * 1e3


res = {}
res["oneshot_us"] = timed(lambda: q.toeplitz_extract(raw, B, w.n, w.m, seed, out=out, stream=st))
q.kernel_timing(True, aux=False)
res["oneshot_kt_us"] = timed(lambda: q.toeplitz_extract(raw, B, w.n, w.m, seed, out=out, stream=st))
q.kernel_timing(False)
with q.Plan(w.n, w.m, seed) as pl:
    res["steady_us"] = timed(lambda: pl.extract(raw, B, out=out, stream=st))
    q.kernel_timing(True, aux=False)
    res["steady_kt_us"] = timed(lambda: pl.extract(raw, B, out=out, stream=st))
    q.kernel_timing(False)


def plan_only():
    with q.Plan(w.n, w.m, seed) as p:
        pass


res["plan_us"] = timed(plan_only)
print(json.dumps({k: round(v, 2) for k, v in res.items()}))
