# tile-run work distribution A/B (gemm_tc.cu tile_runs): QRNG_GEMM_RUNLEN tiles per run;
# bit-exact parity checked by bench.py on every line
python -m paper_2011_04130_b200.build > /dev/null || exit 1
for i in 1 2; do for r in 16 24 32 48 64; do for c in 2 3 10 13 16 17 18; do
  QRNG_GEMM_RUNLEN=$r python bench.py --config $c --configs none --no-e2e --no-cpu-baseline > gpurun_out/ru.json 2>/dev/null; python tools/line.py "runlen=$r cfg$c" < gpurun_out/ru.json
done; done; done
