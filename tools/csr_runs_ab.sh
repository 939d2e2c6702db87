# key-row combine for long rows (>= 512 words): runs in conflict-free batches (default) vs the CSR key kernels (QRNG_CSR_RUNS=0)
python -m paper_2011_04130_b200.build > /dev/null || exit 1
for i in 1 2; do for v in 1 0; do for c in 3 15 16 17 18; do
  QRNG_CSR_RUNS=$v python bench.py --config $c --configs none --no-e2e --no-cpu-baseline > gpurun_out/cr.json 2>/dev/null; python tools/line.py "runs=$v cfg$c" < gpurun_out/cr.json
done; done; done
