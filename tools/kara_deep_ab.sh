# Karatsuba depth past the auto limit (6) at the NTT-side sweep points (NEXT-2(i) option one)
python -m paper_2011_04130_b200.build > /dev/null
for c in 19 20; do
  for d in 6 7 8 9; do
    timeout 300 python bench.py --config $c --path gemm --karatsuba $d --configs none --no-e2e --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print($c, $d, round(d['value'],2), d['config']['karatsuba_leaves'], round(r['frac'],3), round(r['kernel_share_of_step'],3), round(r.get('aux',{}).get('ms_per_step',0),3), d['parity']['status'])" || echo "$c $d failed"
  done
done
