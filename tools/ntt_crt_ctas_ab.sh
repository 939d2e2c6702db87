#!/bin/bash
# CRT pass (packed NTT form) at 3 CTAs per SM (default) vs 2 (128 registers, no spill).
python -m paper_2011_04130_b200.build > /dev/null || exit 1
python -m paper_2011_04130_b200.build --variant crt2 -DQRNG_NTT_CRT_CTAS=2 > /dev/null || exit 1
for i in 1 2; do for lib in libqrng.so libqrng_crt2.so; do for c in 4 19; do
  QRNG_LIB_PATH=$PWD/paper_2011_04130_b200/$lib python bench.py --config $c --configs none --no-e2e --no-cpu-baseline 2>/dev/null | python tools/line.py "$lib cfg$c"
done; done; done
