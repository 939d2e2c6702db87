# tile-geometry lookahead A/B (libqrng_nolook.so = without), 3 runs each
for i in 1 2 3; do for lib in libqrng.so libqrng_nolook.so; do for c in 2 3; do
  QRNG_LIB_PATH=$PWD/paper_2011_04130_b200/$lib python bench.py --config $c --configs none --no-e2e --no-cpu-baseline > gpurun_out/la.json 2>/dev/null; python tools/line.py "$lib cfg$c" < gpurun_out/la.json
done; done; done
