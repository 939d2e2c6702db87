#!/usr/bin/env python
"""MMA issue cost in the GEMM kernel's stage shape (qrng_debug_mma_rate form 3):
4 K32 steps x two N tiles per elected issue block + one commit, runtime descriptors."""
import json, sys
sys.path.insert(0, '/root/repo')
import paper_2011_04130_b200 as q
q.load_library()
for n0, n1 in [(192,192),(192,64),(192,128),(192,160),(128,128),(256,128),(64,64)]:
    r = q.mma_rate(3, n0 | (n1 << 9))
    print(json.dumps({"n0": n0, "n1": n1, "tops": round(2*r/1e12)}))
