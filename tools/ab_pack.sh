#!/bin/bash
for r in 1 2; do for ps in 0 1; do
  QRNG_KARA_PACK_SPLIT=$ps QRNG_GEMM_PACKED=$ps python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > /tmp/b.json
  python -c "import json; d=json.load(open('/tmp/b.json')); print('split/packed', $ps, round(d['value'],1), round(d['steady_state']['value'],1), round(d['roofline']['kernel_ms_per_step'],4))"
done; done
