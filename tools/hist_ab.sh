# the GEMM / NTT kernels of an earlier commit (libqrng_<commit>.so built from git archive) vs HEAD
for i in 1 2; do for lib in libqrng_cbd8577.so libqrng.so; do for c in 18 10 1 2 3 4; do
  QRNG_LIB_PATH=$PWD/paper_2011_04130_b200/$lib python bench.py --config $c --configs none --no-e2e --no-cpu-baseline > gpurun_out/h.json 2>/dev/null; python tools/line.py "$lib cfg$c" < gpurun_out/h.json
done; done; done
