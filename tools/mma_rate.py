#!/usr/bin/env python
"""tcgen05 int8 MMA issue-rate microbenchmark (qrng_debug_mma_rate): TOPS per form and N.
Forms (int8): 0 = A in TMEM, 1 = A in SMEM; see include/qrng.h qrng_debug_mma_rate (form 2, the 2-SM pair,
was removed with the 2-SM kernel; tools/mma_shapes.py covers the E2M1 forms 4 and 5)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2011_04130_b200 as q

q.load_library()
forms = [int(f) for f in (sys.argv[1] if len(sys.argv) > 1 else "0,1").split(",")]
for form in forms:
    for n in (64, 128, 192, 256):
        try:
            r = q.mma_rate(form, n)
            print(json.dumps({"form": form, "n": n, "tops": 2 * r / 1e12}), flush=True)
        except Exception as e:
            print(json.dumps({"form": form, "n": n, "error": str(e)[:100]}), flush=True)
