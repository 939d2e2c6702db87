#!/bin/bash
# Combine + pack (csr_stream_pack_kernel) threads per CTA: 512 (default) vs 384 / 256
# (register budget at 3 CTAs per SM: 42 / 56 / 85 registers; 384 keeps both
# 192-thread block sets busy).  Configs 2, 2^13, 2^14 (the rows it serves).
python -m paper_2011_04130_b200.build > /dev/null || exit 1
python -m paper_2011_04130_b200.build --variant t384 -DQRNG_CSR_THREADS=384 > /dev/null || exit 1
python -m paper_2011_04130_b200.build --variant t256 -DQRNG_CSR_THREADS=256 > /dev/null || exit 1
for i in 1 2; do for lib in libqrng.so libqrng_t384.so libqrng_t256.so; do for c in 2 13 14; do
  QRNG_LIB_PATH=$PWD/paper_2011_04130_b200/$lib python bench.py --config $c --configs none --no-e2e --no-cpu-baseline 2>/dev/null | python tools/line.py "$lib cfg$c"
done; done; done
