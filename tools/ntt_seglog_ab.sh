set -e
python -m paper_2011_04130_b200.build > /dev/null
for v in 14 13; do python -m paper_2011_04130_b200.build --variant seg$v -DQRNG_NTT_SEGLOG=$v > /dev/null; done
for lib in libqrng.so libqrng_seg14.so libqrng_seg13.so; do
  for c in 4 19 22; do
    QRNG_LIB_PATH=$PWD/paper_2011_04130_b200/$lib python bench.py --config $c --configs none --no-e2e --no-cpu-baseline --no-parity --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', $c, round(d['value'],2), round(d['roofline']['frac'],3))"
  done
done
