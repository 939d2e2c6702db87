#!/usr/bin/env python
"""Three-stream H2D / extract / D2H pipeline with per-stage CUDA events (config 2): where the streaming ingest spends its time."""
import sys, time, json, torch
sys.path.insert(0,'/root/repo')
import qrng_synth as S, paper_2011_04130_b200 as q
q.load_library()
w=S.CONFIGS[2]; raw_np, seed_np = S.workload_inputs(w); B=w.n_blocks
seed=torch.from_numpy(seed_np).cuda(); h_raw=torch.from_numpy(raw_np).pin_memory()
ob=q.out_bytes(B,w.m); depth=3
d_raw=[torch.empty_like(h_raw,device='cuda') for _ in range(depth)]
d_out=[torch.empty(ob,dtype=torch.uint8,device='cuda') for _ in range(depth)]
h_out=[torch.empty(ob,dtype=torch.uint8).pin_memory() for _ in range(depth)]
si,sc,so=torch.cuda.Stream(),torch.cuda.Stream(),torch.cuda.Stream()
E=lambda: torch.cuda.Event(enable_timing=True)
with q.Plan(w.n,w.m,seed) as pl:
    N=40; ev=[]
    start=E(); start.record(si)
    done=[None]*depth
    for k in range(N):
        sl=k%depth
        if done[sl] is not None: done[sl].synchronize()
        a,b,c,d,e,f=E(),E(),E(),E(),E(),E()
        with torch.cuda.stream(si):
            a.record(si); d_raw[sl].copy_(h_raw,non_blocking=True); b.record(si)
        sc.wait_event(b)
        c.record(sc); pl.extract(d_raw[sl],B,out=d_out[sl],stream=sc); d.record(sc)
        so.wait_event(d)
        with torch.cuda.stream(so):
            e.record(so); h_out[sl].copy_(d_out[sl],non_blocking=True); f.record(so)
        done[sl]=f; ev.append((a,b,c,d,e,f))
    torch.cuda.synchronize()
    h2d=[a.elapsed_time(b) for a,b,c,d,e,f in ev[5:]]
    cmp=[c.elapsed_time(d) for a,b,c,d,e,f in ev[5:]]
    d2h=[e.elapsed_time(f) for a,b,c,d,e,f in ev[5:]]
    per=[ev[i][0].elapsed_time(ev[i+1][0]) for i in range(5,N-1)]
    print(json.dumps({"h2d_ms":sum(h2d)/len(h2d),"compute_ms":sum(cmp)/len(cmp),"d2h_ms":sum(d2h)/len(d2h),"h2d_start_interval_ms":sum(per)/len(per)}))
