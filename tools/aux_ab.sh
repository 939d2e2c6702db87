#!/bin/bash
# Karatsuba Q buffers, round 2: the one-pass slice kernel (QRNG_QSLICE=1,
# default) against the generation kernel (0) on the shallow-tree workloads it
# covers (config 2 = 2^13 with 16384 blocks; sweep 2^13 / 2^14 / 2^15 over 2^30
# bits) plus config 3 (depth 5: 32 slices, not covered -- a control).
# (The same script measured a warp-per-block combine + pack, QRNG_CSR_WARP,
# slower than the staged stream form and removed.)
python -m paper_2011_04130_b200.build > /dev/null || exit 1
for i in 1 2; do for v in 1 0; do for c in 2 13 14 15 3; do
  QRNG_QSLICE=$v python bench.py --config $c --configs none --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python tools/line.py "qslice=$v cfg$c" < gpurun_out/ab.json
done; done; done
