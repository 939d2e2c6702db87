# Karatsuba depth scan after the two-phase combine (config 5 points, 2^30 bits)
python -m paper_2011_04130_b200.build > /dev/null
for c in 15 16 17 18; do for d in 3 4 5 6; do
  python bench.py --config $c --path gemm --karatsuba $d --configs none --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/d.json 2>/dev/null; python tools/line.py "cfg$c d$d" < gpurun_out/d.json
done; done
