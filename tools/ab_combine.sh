#!/bin/bash
# A/B of the combine kernel's group buffers in flight (QRNG_CSR_NBUF builds) on config 2.
mkdir -p gpurun_out
for v in nbuf3 nbuf4; do QRNG_LIB_PATH=paper_2011_04130_b200/libqrng_$v.so timeout 600 python -m pytest tests/test_gpu_karatsuba.py -m gpu -q -x 2>&1 | tail -1; done
for r in 1 2; do for v in "" nbuf3 nbuf4; do
  L=paper_2011_04130_b200/libqrng${v:+_$v}.so
  QRNG_LIB_PATH=$L python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('$v', round(d['value'],1), round(d['steady_state']['value'],1), 'aux ms', round(r['aux']['ms_per_step'],4), 'step', round(d['ms_per_step'],4))"
done; done
for v in "" nbuf3 nbuf4; do L=paper_2011_04130_b200/libqrng${v:+_$v}.so; QRNG_LIB_PATH=$L ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"csr_stream" -c 2 python tools/one_extract.py --config 2 --reps 3 2>&1 | grep -E "duration" | tr '\n' ' '; echo " $v"; done
