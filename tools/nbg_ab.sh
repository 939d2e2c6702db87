# B-generator warp count with tile runs (B reuse): forced 1 / 2 / 4 (-DQRNG_GEMM_NBG_FORCE builds)
# vs the default (3; 4 for packed launches with > 64 leaves)
python -m paper_2011_04130_b200.build > /dev/null || exit 1
for k in 1 2 4; do python -m paper_2011_04130_b200.build --variant nbg$k -DQRNG_GEMM_NBG_FORCE=$k > /dev/null || exit 1; done
for i in 1 2; do for lib in libqrng.so libqrng_nbg1.so libqrng_nbg2.so libqrng_nbg4.so; do for c in 2 3 17 10; do
  QRNG_LIB_PATH=$PWD/paper_2011_04130_b200/$lib python bench.py --config $c --configs none --no-e2e --no-cpu-baseline > gpurun_out/nb.json 2>/dev/null; python tools/line.py "$lib cfg$c" < gpurun_out/nb.json
done; done; done
