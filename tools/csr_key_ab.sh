# long-row combine: staged key kernel vs gather key kernel vs the one-phase gather (QRNG_CSR_ZPACK=0)
python -m paper_2011_04130_b200.build > /dev/null
for v in "QRNG_CSR_STAGE=1" "QRNG_CSR_STAGE=0" "QRNG_CSR_ZPACK=0"; do for c in 3 16 17 18; do
  env $v python bench.py --config $c --configs none --no-e2e --no-cpu-baseline > gpurun_out/k.json 2>/dev/null; python tools/line.py "$v cfg$c" < gpurun_out/k.json
done; done
