#!/usr/bin/env python
"""Host-side cost per C-ABI call (enqueue time without synchronisation) vs the wall time per call, one-shot and plan-reused
(python tools/host_overhead.py [CONFIG], default config 2)."""
import time, torch, sys
sys.path.insert(0, '/root/repo')
import qrng_synth as S, paper_2011_04130_b200 as q
q.load_library()
w = S.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
raw_np, seed_np = S.workload_inputs(w)
raw, seed = torch.from_numpy(raw_np).cuda(), torch.from_numpy(seed_np).cuda()
out = torch.empty(q.out_bytes(w.n_blocks, w.m), dtype=torch.uint8, device="cuda")
for timing in (False, True):
    q.kernel_timing(timing)
    for _ in range(5): q.toeplitz_extract(raw, w.n_blocks, w.n, w.m, seed, out=out)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50): q.toeplitz_extract(raw, w.n_blocks, w.n, w.m, seed, out=out)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"timing={timing}: host enqueue {1e6*(t1-t0)/50:.1f} us/call, wall incl. sync {1e6*(t2-t0)/50:.1f} us/call")
    with q.Plan(w.n, w.m, seed) as pl:
        for _ in range(5): pl.extract(raw, w.n_blocks, out=out)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(50): pl.extract(raw, w.n_blocks, out=out)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
    print(f"timing={timing}: plan reused: host enqueue {1e6*(t1-t0)/50:.1f} us/call, wall {1e6*(t2-t0)/50:.1f} us/call")
q.kernel_timing(False)
