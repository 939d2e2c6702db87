#!/bin/bash
# NTT multi-pass sizes: the packed three-prime form (4 blocks per group, 3
# primes, CRT; default) against one block per transform (QRNG_NTT_CRT=0).
python -m paper_2011_04130_b200.build > /dev/null || exit 1
for i in 1 2; do for v in 1 0; do for c in 4 41 19 20; do
  QRNG_NTT_CRT=$v python bench.py --config $c --configs none --no-e2e --no-cpu-baseline --path ntt 2>/dev/null | python tools/line.py "crt=$v cfg$c"
done; done; done
