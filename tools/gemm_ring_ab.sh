# tcgen05 kernel ring depths: A stages, B slots, transform prefetch (config 2 and 3)
python -m paper_2011_04130_b200.build > /dev/null
python -m paper_2011_04130_b200.build --variant a3 -DQRNG_GEMM_ASTAGES=3 > /dev/null
python -m paper_2011_04130_b200.build --variant b4 -DQRNG_GEMM_BSLOTS=4 > /dev/null
python -m paper_2011_04130_b200.build --variant pf3 -DQRNG_GEMM_PF=3 > /dev/null
python -m paper_2011_04130_b200.build --variant a3b4 -DQRNG_GEMM_ASTAGES=3 -DQRNG_GEMM_BSLOTS=4 > /dev/null
for lib in libqrng.so libqrng_a3.so libqrng_b4.so libqrng_pf3.so libqrng_a3b4.so; do
  for c in 2 3; do
    QRNG_LIB_PATH=$PWD/paper_2011_04130_b200/$lib python bench.py --config $c --configs none --no-e2e --no-cpu-baseline 2>/dev/null | python tools/line.py "$lib cfg$c"
  done
done
