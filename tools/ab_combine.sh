#!/bin/bash
# A/B of the Karatsuba combine+pack forms on config 2 (fused form stages only
# the straddle heads, so 3 CTAs fit per SM): parity, bench, ncu durations.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_karatsuba.py tests/test_gpu_parity.py tests/test_gpu_modified.py -m gpu -q -x 2>&1 | tail -1
QRNG_CSR_FUSED=0 timeout 900 python -m pytest tests/test_gpu_karatsuba.py -m gpu -q -x 2>&1 | tail -1
for r in 1 2; do for f in 1 0; do QRNG_CSR_FUSED=$f python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('fused', $f, round(d['value'],1), round(d['steady_state']['value'],1), 'aux ms', round(r['aux']['ms_per_step'],4), 'step', round(d['ms_per_step'],4))"; done; done
for f in 1 0; do QRNG_CSR_FUSED=$f ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -k regex:"csr_stream" -c 2 python tools/one_extract.py --config 2 --reps 3 2>&1 | grep -E "duration|grid_size" | tr '\n' ' '; echo " fused=$f"; done
python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('cfg3', round(d['value'],1))"
