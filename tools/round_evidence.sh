#!/bin/bash
# One GPU pass that refreshes the round's evidence: tests, smoke, the bench
# lines of every config, the bench launch list under ncu and one full ncu
# capture of the headline kernel.  Usage: bash tools/round_evidence.sh TAG
T=${1:-rX}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$T.txt 2>&1; tail -1 gpurun_out/pytest_gpu_$T.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 20 --warmup 3 2>/dev/null | tail -1 > gpurun_out/bench_default_$T.json
for c in 1 3 4 41; do python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_cfg${c}_$T.json; done
python bench.py --config 2 --variant modified --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_mod2_$T.json
python bench.py --config 4 --variant modified --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_mod4_$T.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_launches_bench_cfg2.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:toeplitz_gemm_kernel -s 1 -c 1 \
    -o gpurun_out/${T}_gemm_cfg2 python tools/one_extract.py --config 2 --reps 2 > /dev/null 2>&1
for f in gpurun_out/bench_*_$T.json; do
  python - "$f" <<'PY'
import json, sys
d = json.load(open(sys.argv[1])); r = d.get("roofline") or {}
print(sys.argv[1].split("/")[-1], round(d["value"], 1), "steady", round((d.get("steady_state") or {}).get("value", 0), 1),
      "e2e", round((d.get("e2e") or {}).get("value") or 0, 1), "frac", round(r.get("frac", 0), 3), r.get("bound"),
      round(r.get("achieved", 0)), d["config"].get("path"), d.get("clocks", {}).get("reasons"))
PY
done
