#!/bin/bash
# Seed-spectrum layout: interleaved by 16-byte groups across sub-DFTs (default)
# vs one contiguous row per sub-DFT (-DQRNG_NTT_SHAT_ILV=0), same box.
python -m paper_2011_04130_b200.build > /dev/null || exit 1
python -m paper_2011_04130_b200.build --variant rowshat -DQRNG_NTT_SHAT_ILV=0 > /dev/null || exit 1
for i in 1 2; do for lib in libqrng.so libqrng_rowshat.so; do for c in 4 19 22; do
  QRNG_LIB_PATH=$PWD/paper_2011_04130_b200/$lib python bench.py --config $c --configs none --no-e2e --no-cpu-baseline 2>/dev/null | python tools/line.py "$lib cfg$c"
done; done; done
