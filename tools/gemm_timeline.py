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
ap.add_argument("--per-cta", action="store_true", help="also print (cta, sm, tiles, loop us) for every CTA")
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
    tr = q.gemm_trace(reset=False).astype(np.int64)
tl, cta = tr[:512], tr[512:]
cta = cta[cta[:, 0] != 0]
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
if len(cta):
    # per-CTA phases (globaltimer ns, relative to the earliest CTA entry)
    t0 = cta[:, 0].min()
    out["cta_ns"] = {"ctas": int(len(cta)), "entry_spread": int(cta[:, 0].max() - t0),
                     "first_a_ready": [int(np.median(cta[:, 1] - cta[:, 0])), int((cta[:, 1] - cta[:, 0]).max())],
                     "mma_loop": [int(np.median(cta[:, 2] - cta[:, 1])), int((cta[:, 2] - cta[:, 1]).min()),
                                  int((cta[:, 2] - cta[:, 1]).max())],
                     "drain_to_exit": [int(np.median(cta[:, 3] - cta[:, 2])), int((cta[:, 3] - cta[:, 2]).max())],
                     "last_mma_end": int(cta[:, 2].max() - t0), "first_exit": int(cta[:, 3].min() - t0),
                     "last_exit": int(cta[:, 3].max() - t0),
                     "tiles_min_max": [int(cta[:, 4].min()), int(cta[:, 4].max())]}
    loop = cta[:, 2] - cta[:, 1]
    for k in np.unique(cta[:, 4]):  # loop time by tile count: static imbalance vs per-SM speed
        sel = cta[:, 4] == k
        out["cta_ns"][f"loop_us_at_{int(k)}_tiles"] = [int(sel.sum()), round(float(loop[sel].min()) / 1e3, 1),
                                                      round(float(np.median(loop[sel])) / 1e3, 1),
                                                      round(float(loop[sel].max()) / 1e3, 1)]
print(json.dumps(out))
if a.per_cta and len(cta):
    for c in range(len(cta)):
        print("cta", c, "sm", int(cta[c, 5]), "tiles", int(cta[c, 4]), "entry_us", round((cta[c, 0] - cta[:, 0].min()) / 1e3, 2),
              "loop_us", round((cta[c, 2] - cta[c, 1]) / 1e3, 1))
