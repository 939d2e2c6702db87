mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_karatsuba.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print(round(d['value'],1), round(d['steady_state']['value'],1), 'aux ms', round(r['aux']['ms_per_step'],4), 'kern', round(r['kernel_ms_per_step'],4))"; done
ncu --metrics gpu__time_duration.sum,sm__inst_executed.sum --clock-control none -k regex:"csr_stream|qbuf" -c 4 python tools/one_extract.py --config 2 --reps 3 2>&1 | grep -E "csr_stream|qbuf|duration|inst_exec"
