# Karatsuba depth 7 (2187 leaves: leaf table 70 KB in the GEMM kernel's shared memory)
# at the NTT-side sweep points, and what AUTO picks with the cap raised.
python -m paper_2011_04130_b200.build > /dev/null
python -m paper_2011_04130_b200.build --variant ml4096 -DQRNG_KARA_MAXLEAVES=4096 > /dev/null
for c in 18 19 20; do
  for d in 6 7; do
    QRNG_LIB_PATH=$PWD/paper_2011_04130_b200/libqrng_ml4096.so timeout 300 python bench.py --config $c --path gemm --karatsuba $d --configs none --no-e2e --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('kara', $c, $d, round(d['value'],2), d['config']['karatsuba_leaves'], round(r['frac'],3), round(r['kernel_ms_per_step'],3), round(r.get('aux',{}).get('ms_per_step',0),3), d['parity']['status'])" || echo "$c $d failed"
  done
done
# the planner's own choice with the raised cap (AUTO path, auto depth)
for c in 18 19 20; do
  QRNG_LIB_PATH=$PWD/paper_2011_04130_b200/libqrng_ml4096.so timeout 300 python bench.py --config $c --configs none --no-e2e --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | python tools/line.py "auto ml4096 cfg$c"
done
