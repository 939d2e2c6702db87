#!/bin/bash
# Radix-32 packed forward pass (P = 2^20: n = 2^19) under a 3-CTA launch bound
# (145 -> 80 registers, no spill; default) vs no bound (-DQRNG_NTT_PASS_BOUND=0
# also drops the radix-64 bounds), same box.
python -m paper_2011_04130_b200.build > /dev/null || exit 1
python -m paper_2011_04130_b200.build --variant nobound -DQRNG_NTT_PASS_BOUND=0 > /dev/null || exit 1
for i in 1 2; do for lib in libqrng.so libqrng_nobound.so; do for c in 19 4; do
  QRNG_LIB_PATH=$PWD/paper_2011_04130_b200/$lib python bench.py --config $c --configs none --no-e2e --no-cpu-baseline 2>/dev/null | python tools/line.py "$lib cfg$c"
done; done; done
