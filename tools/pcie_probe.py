#!/usr/bin/env python
"""Host<->device copy rates from pinned memory (the e2e bound): H2D alone, D2H
alone, and both directions at once on two streams.  Sizes = config 2's raw
input (16 MiB) and key (11.2 MiB)."""
import json
import torch

h_in = torch.empty(16 << 20, dtype=torch.uint8).pin_memory()
h_out = torch.empty(11744 * 1024, dtype=torch.uint8).pin_memory()
d_in = torch.empty_like(h_in, device="cuda")
d_out = torch.empty_like(h_out, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def h2d():
    d_in.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d_out, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(json.dumps({"h2d_gbs": h_in.numel() / t1 / 1e6, "d2h_gbs": h_out.numel() / t2 / 1e6,
                  "both_ms": t3, "both_h2d_equiv_gbs": h_in.numel() / t3 / 1e6,
                  "cfg2_e2e_bound_gbit_s": 134217728 / (max(t1, t2, t3) * 1e-3) / 1e9}))


# two concurrent H2D copies of half the batch each (two copy streams)
half = h_in.numel() // 2


def h2d2():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_in[:half].copy_(h_in[:half], non_blocking=True)
    with torch.cuda.stream(s2):
        d_in[half:].copy_(h_in[half:], non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t4 = timed(h2d2, reps=40)
t5 = timed(h2d, reps=40)
print(json.dumps({"h2d_two_streams_gbs": h_in.numel() / t4 / 1e6, "h2d_again_gbs": h_in.numel() / t5 / 1e6}))
