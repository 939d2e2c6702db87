#!/bin/bash
# NTT emit pass: warp-uniform skip of the q outside the key window (default)
# vs every q through the window test (-DQRNG_NTT_EMIT_SKIP=0).
python -m paper_2011_04130_b200.build > /dev/null || exit 1
python -m paper_2011_04130_b200.build --variant noskip -DQRNG_NTT_EMIT_SKIP=0 > /dev/null || exit 1
for i in 1 2; do for lib in libqrng.so libqrng_noskip.so; do for c in 4 19 22; do
  QRNG_LIB_PATH=$PWD/paper_2011_04130_b200/$lib python bench.py --config $c --configs none --no-e2e --no-cpu-baseline 2>/dev/null | python tools/line.py "$lib cfg$c"
done; done; done
