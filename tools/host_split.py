#!/usr/bin/env python
"""Host cost per call, split: the Python binding's checks vs the bare C-ABI call
(ctypes straight into libqrng.so), one-shot vs plan-reused (config 1 by default:
the small-batch case where the host, not the device, sets the call rate)."""
import ctypes, sys, time
import torch
sys.path.insert(0, '/root/repo')
import qrng_synth as S, paper_2011_04130_b200 as q
lib = q.load_library()
w = S.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
raw_np, seed_np = S.workload_inputs(w)
raw, seed = torch.from_numpy(raw_np).cuda(), torch.from_numpy(seed_np).cuda()
out = torch.empty(q.out_bytes(w.n_blocks, w.m), dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
sh = st.cuda_stream
pr, ps, po = raw.data_ptr(), seed.data_ptr(), out.data_ptr()


def per_call(fn, k=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return round((t1 - t0) / k * 1e6, 2)


res = {"workload": w.name}
res["python_oneshot_us"] = per_call(lambda: q.toeplitz_extract(raw, w.n_blocks, w.n, w.m, seed, out=out, stream=st))
res["c_oneshot_us"] = per_call(lambda: lib.qrng_toeplitz_extract_async(pr, w.n_blocks, w.n, w.m, ps, po, sh))
with q.Plan(w.n, w.m, seed) as pl:
    h = pl._h
    res["python_plan_us"] = per_call(lambda: pl.extract(raw, w.n_blocks, out=out, stream=st))
    res["c_plan_us"] = per_call(lambda: lib.qrng_plan_extract(h, pr, w.n_blocks, po, sh))
res["torch_empty_kernel_us"] = per_call(lambda: out[:16].zero_())
print(res)
