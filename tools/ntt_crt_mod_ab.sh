#!/bin/bash
# Modified Toeplitz [T | I_m] on the NTT path: the packed three-prime form (its
# CRT pass XORs the identity block) vs one block per transform (QRNG_NTT_CRT=0).
python -m paper_2011_04130_b200.build > /dev/null || exit 1
for i in 1 2; do for v in 1 0; do for c in 4 3; do
  QRNG_NTT_CRT=$v python bench.py --config $c --variant modified --path ntt --configs none --no-e2e --no-cpu-baseline 2>/dev/null | python tools/line.py "crt=$v mod cfg$c"
done; done; done
