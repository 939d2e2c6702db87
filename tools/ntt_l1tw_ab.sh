# segment kernel level-1 twiddles: Shoup table in shared memory (default) vs Montgomery chains (QRNG_NTT_L1TW=0)
python -m paper_2011_04130_b200.build > /dev/null || exit 1
for i in 1 2; do for v in 1 0; do for c in 4 19 22; do
  QRNG_NTT_L1TW=$v python bench.py --config $c --configs none --no-e2e --no-cpu-baseline > gpurun_out/l1.json 2>/dev/null; python tools/line.py "l1tw=$v cfg$c" < gpurun_out/l1.json
done; done; done
