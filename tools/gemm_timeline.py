#!/usr/bin/env python
"""MMA-issue timeline of CTA 0 of the packed-mode tcgen05 kernel (needs a
-DQRNG_GEMM_TIMELINE build through QRNG_LIB_PATH): per stage, cycles spent
waiting (A / B / accumulator barriers) and issuing, and the gap pattern at
tile boundaries.

    python -m paper_2011_04130_b200.build --variant tl -DQRNG_GEMM_TIMELINE
    QRNG_LIB_PATH=$PWD/paper_2011_04130_b200/libqrng_tl.so python tools/gemm_timeline.py --config 2
"""
import argparse, json, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import qrng_synth as S
import paper_2011_04130_b200 as q

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
a = ap.parse_args()
q.load_library()
w = S.CONFIGS[a.config] if a.config in S.CONFIGS else S.sweep_workload(a.config)
raw_np, seed_np = S.workload_inputs(w)
raw, seed = torch.from_numpy(raw_np).cuda(), torch.from_numpy(seed_np).cuda()
with q.Plan(w.n, w.m, seed) as pl:
    for _ in range(3):
        pl.extract(raw, w.n_blocks)
    torch.cuda.synchronize()
    q.gemm_trace(reset=True)
    pl.extract(raw, w.n_blocks)
    torch.cuda.synchronize()
    tl = q.gemm_trace(reset=False).astype(np.int64)
tl = tl[tl[:, 1] != 0]
tag, ts, ti_, ta, tb, tA, tI = (tl[:, k] for k in range(7))
tile, stage = tag >> 8, tag & 255
span = tI[-1] - ts[0]
gap = np.r_[0, ts[1:] - tI[:-1]]
s0 = stage == 0
out = {"workload": w.name, "stages": int(len(tl)), "span_cycles": int(span), "cycles_per_stage": float(span / len(tl)),
       "stage0": {"tile_lookup": float((ti_ - ts)[s0].mean()), "acc_wait": float((ta - ti_)[s0].mean()),
                  "b_wait": float((tb - ta)[s0].mean()), "a_wait": float((tA - tb)[s0].mean()),
                  "issue": float((tI - tA)[s0].mean())},
       "other": {"b_wait": float((tb - ts)[~s0].mean()), "a_wait": float((tA - tb)[~s0].mean()),
                 "issue": float((tI - tA)[~s0].mean())},
       "gap_between_stages": float(gap[1:].mean())}
print(json.dumps(out))
