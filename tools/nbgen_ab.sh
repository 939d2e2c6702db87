python -m paper_2011_04130_b200.build > /dev/null
for b in 4 5; do python -m paper_2011_04130_b200.build --variant bg$b -DQRNG_GEMM_NBGEN=$b > /dev/null; done
for i in 1 2; do for lib in libqrng.so libqrng_bg4.so libqrng_bg5.so; do for c in 2 3; do
  QRNG_LIB_PATH=$PWD/paper_2011_04130_b200/$lib python bench.py --config $c --configs none --no-e2e --no-cpu-baseline > gpurun_out/bg.json 2>/dev/null; python tools/line.py "$lib cfg$c" < gpurun_out/bg.json
done; done; done
