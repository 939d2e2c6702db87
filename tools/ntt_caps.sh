#!/bin/bash
# ncu --set full captures of the NTT extraction kernels only (segment kernels
# in SEG mode, the CRT pass), for the traffic entries of the NTT workloads:
#   bash tools/ntt_caps.sh TAG
T=${1:-r2x}
mkdir -p gpurun_out
python -m paper_2011_04130_b200.build > /dev/null || exit 1
cap() {
  ncu --set full --clock-control none --kernel-name-base demangled -k "regex:$3" -s 1 -c 1 -o gpurun_out/${T}_$1 \
      python tools/one_extract.py --config $2 --reps 2 > gpurun_out/${T}_$1.log 2>&1
  echo "$1 rc=$?"
}
cap ntt_segment_cfg4 4 'ntt_segment_kernel<.int.15, .int.1,'
cap ntt_pass_cfg4 4 'ntt_pass_kernel<.int.6, .int.8,'
cap ntt_segment_cfg41 41 'ntt_segment_kernel<.int.15, .int.1,'
cap ntt_segment_cfg5_n2^19 19 'ntt_segment_kernel<.int.15, .int.1,'
cap ntt_segment_cfg5_n2^22 22 'ntt_segment_kernel<.int.15, .int.1,'
for f in gpurun_out/${T}_ntt*.ncu-rep; do echo "== $f"; python tools/ncu_summary.py $f; done > gpurun_out/${T}_ntt_ncu_summaries.txt 2>&1
python tools/ncu_traffic.py $T gpurun_out/${T}_ntt*.ncu-rep > gpurun_out/${T}_ntt_ncu_traffic.json
for f in gpurun_out/${T}_ntt*.ncu-rep; do case $f in *ntt_segment_cfg4.*) ;; *) rm -f "$f";; esac; done
