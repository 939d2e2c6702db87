#!/usr/bin/env python
"""kind::mxf4 feasibility: layout/exactness probe (E2M1 0/1 operands, unit
scales, FP32 accumulation) against an integer reference, then MMA rates
(qrng_debug_mma_rate forms 4/5) next to the int8 stage shape (form 3)."""
import json, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2011_04130_b200 as q

q.load_library()
rng = np.random.default_rng(1)
for K in (64, 256, 1024):
    for N in (16, 192, 256):
        for kind in ("rand", "ones"):
            A = rng.integers(0, 2, (128, K), dtype=np.uint8) if kind == "rand" else np.ones((128, K), np.uint8)
            h = rng.integers(0, 2, N + K, dtype=np.uint8) if kind == "rand" else np.ones(N + K, np.uint8)
            B = np.stack([h[i:i + K] for i in range(N)])
            ref = A.astype(np.int64) @ B.T.astype(np.int64)
            for hf in (False, True):
                D = q.mxf4_probe(torch.from_numpy(A).cuda(), torch.from_numpy(h).cuda(), N, K, hf).cpu().numpy()
                ok = bool(np.array_equal(D.astype(np.int64), ref)) and bool(np.all(D == np.rint(D)))
                print(json.dumps({"K": K, "N": N, "data": kind, "hi_first": hf, "exact": ok,
                                  "max_abs_err": float(np.abs(D - ref).max())}), flush=True)
for n in (64, 128, 192, 256):
    print(json.dumps({"form": "mxf4 1-SM SS", "n": n, "tops": round(2 * q.mma_rate(4, n) / 1e12)}), flush=True)
for n0, n1 in ((192, 192), (128, 128), (256, 128), (192, 64)):
    print(json.dumps({"form": "mxf4 stage", "n0": n0, "n1": n1, "tops": round(2 * q.mma_rate(5, n0 | (n1 << 9)) / 1e12)}), flush=True)
    print(json.dumps({"form": "i8 stage", "n0": n0, "n1": n1, "tops": round(2 * q.mma_rate(3, n0 | (n1 << 9)) / 1e12)}), flush=True)
