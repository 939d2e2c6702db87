#!/usr/bin/env python
"""cuBLAS int8 GEMM reference rate on this B200 (torch._int_mm, 8192^3, best of 10,
CUDA events) -- context for the int8 tensor-core roofline of the GEMM path."""
import json
import torch

N = 8192
a = torch.randint(-8, 8, (N, N), dtype=torch.int8, device="cuda")
b = torch.randint(-8, 8, (N, N), dtype=torch.int8, device="cuda")
for _ in range(3):
    torch._int_mm(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    torch._int_mm(a, b)
    e.record()
    torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
print(json.dumps({"what": "torch._int_mm int8 8192^3 best of 10", "ms": best,
                  "tops": 2 * N ** 3 / best / 1e9}))
