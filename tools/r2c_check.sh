python -m paper_2011_04130_b200.build > /dev/null || exit 1
python tools/oneshot_jitter.py --config 4 --steps 60 --smi 1 | tee gpurun_out/jitter_r2c.txt
python tools/oneshot_jitter.py --config 4 --steps 60 --smi 1 | tee -a gpurun_out/jitter_r2c.txt
python tools/oneshot_jitter.py --config 4 --steps 60 --smi 0 | tee -a gpurun_out/jitter_r2c.txt
for i in 1 2 3; do python bench.py --config 4 --configs none --no-e2e --no-cpu-baseline --steps 20 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg4 bench', round(d['value'],2), round(d['ms_per_step_max_rank0'],3), d['clocks'])" | tee -a gpurun_out/jitter_r2c.txt; done
