# NTT transform CTAs: 1024 / 512 / 256 threads (sub-DFTs per thread unrolled together)
python -m paper_2011_04130_b200.build > /dev/null
for t in 512 256; do python -m paper_2011_04130_b200.build --variant t$t -DQRNG_NTT_MAXT=$t > /dev/null; done
for lib in libqrng.so libqrng_t512.so libqrng_t256.so; do
  for c in 4 19 22 15; do
    QRNG_LIB_PATH=$PWD/paper_2011_04130_b200/$lib python bench.py --config $c --path ntt --configs none --no-e2e --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', $c, round(d['value'],2), round(d['roofline']['frac'],3), d['parity']['status'])"
  done
done
