# HEAD-before-runs build (libqrng_old.so) vs tile runs (default) vs strided order (QRNG_GEMM_RUNS=0)
python -m paper_2011_04130_b200.build > /dev/null || exit 1
for i in 1 2; do for v in old new new0; do for c in 18 10 1 2 3 17; do
  lib=libqrng.so; [ $v = old ] && lib=libqrng_old.so; rr=""; [ $v = new0 ] && rr=0
  QRNG_GEMM_RUNS=$rr QRNG_LIB_PATH=$PWD/paper_2011_04130_b200/$lib python bench.py --config $c --configs none --no-e2e --no-cpu-baseline > gpurun_out/ru.json 2>/dev/null; python tools/line.py "$v cfg$c" < gpurun_out/ru.json
done; done; done
