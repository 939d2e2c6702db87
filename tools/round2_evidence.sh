#!/bin/bash
# One GPU pass that refreshes the round's evidence (round 2 layout):
# tests, smoke, the default bench line (headline + configs object), the bench
# launch list under ncu, and one `ncu --set full` capture of the dominant
# kernel of every workload (traffic = dram bytes per launch).
#   bash tools/round2_evidence.sh TAG
T=${1:-r2x}
mkdir -p gpurun_out
python -m paper_2011_04130_b200.build > /dev/null || exit 1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$T.txt 2>&1; tail -1 gpurun_out/pytest_gpu_$T.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
S0=$SECONDS; timeout 1200 python bench.py > gpurun_out/bench_default_$T.json 2> gpurun_out/bench_default_$T.err
echo "default bench wall $((SECONDS - S0)) s" | tee gpurun_out/bench_default_${T}_wall.txt
timeout 900 python bench.py --gpus 2 --configs cfg4a,cfg5_n2^16,next4_n2^24 --no-e2e > gpurun_out/bench_g2gloo_$T.json 2> gpurun_out/bench_g2gloo_$T.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_launches_bench_cfg2.csv python bench.py --steps 3 --warmup 3 --configs none \
    --no-e2e --no-cpu-baseline --no-parity > /dev/null 2>&1
cap() {  # name config kernel-regex (on the demangled name, so template arguments can select) [source]
  ncu --set full --clock-control none ${4:+--import-source on} --kernel-name-base demangled -k "regex:$3" -s 1 -c 1 -o gpurun_out/${T}_$1 \
      python tools/one_extract.py --config $2 --reps 2 > gpurun_out/${T}_$1.log 2>&1
  echo "$1 rc=$?"
}
cap gemm_cfg2 2 'toeplitz_gemm_kernel' src
cap bits_cfg1 1 bits_kernel
cap gemm_cfg3 3 toeplitz_gemm_kernel
cap ntt_segment_cfg4 4 'ntt_segment_kernel<.int.15, .int.1,'
cap ntt_pass_cfg4 4 'ntt_pass_kernel<.int.6, .int.8,'
cap gemm_cfg5_n2^10 10 toeplitz_gemm_kernel
cap ntt_segment_cfg5_n2^19 19 'ntt_segment_kernel<.int.15, .int.1,'
cap ntt_segment_cfg5_n2^22 22 'ntt_segment_kernel<.int.15, .int.1,'
cap gemm_cfg5_n2^13 13 toeplitz_gemm_kernel
cap gemm_cfg5_n2^16 16 toeplitz_gemm_kernel
cap gemm_cfg5_n2^18 18 toeplitz_gemm_kernel
cap ntt_segment_cfg41 41 'ntt_segment_kernel<.int.15, .int.1,'
cap ntt_segment_next4 124 'ntt_segment_kernel<.int.15, .int.1,'
for f in gpurun_out/${T}_*.ncu-rep; do echo "== $f"; python tools/ncu_summary.py $f; done > gpurun_out/${T}_ncu_summaries.txt 2>&1
python tools/ncu_traffic.py $T gpurun_out/${T}_*.ncu-rep > gpurun_out/${T}_ncu_traffic.json
# keep the headline capture (with source) and the NTT segment capture; the rest
# live on as summaries + traffic (gpurun copies back at most 64 MiB)
for f in gpurun_out/${T}_*.ncu-rep; do case $f in *gemm_cfg2*|*ntt_segment_cfg4.*) ;; *) rm -f "$f";; esac; done
ls -la gpurun_out/
python - gpurun_out/bench_default_$T.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
print("headline", round(d["value"], 1), "steady", round(d["steady_state"]["value"], 1), "e2e", round(d["e2e"]["value"], 1),
      "frac", round(r["frac"], 3), d.get("parity_all"), d["clocks"])
for k, v in d.get("configs", {}).items():
    r = v.get("roofline") or {}
    print(k, round(v["value"], 2), r.get("bound"), round(r.get("frac", 0), 3), (v.get("parity") or {}).get("status"))
PY
