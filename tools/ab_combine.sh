#!/bin/bash
# A/B: lazy Q-buffer wait in the grouped GEMM (QRNG_GEMM_LAZY_QWAIT) on configs 2 and 3.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_karatsuba.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -1
for r in 1 2; do for f in 1 0; do QRNG_GEMM_LAZY_QWAIT=$f python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('lazy', $f, round(d['value'],1), round(d['steady_state']['value'],1), 'kern', round(r['kernel_ms_per_step'],4), 'step', round(d['ms_per_step'],4))"; done; done
for f in 1 0; do QRNG_GEMM_LAZY_QWAIT=$f python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('cfg3 lazy', $f, round(d['value'],1))"; done
python tools/oneshot_breakdown.py
