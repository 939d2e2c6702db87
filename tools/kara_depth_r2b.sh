# Karatsuba depth scan with the tile-run kernel (B reuse): does the planner's depth still win?
python -m paper_2011_04130_b200.build > /dev/null
for spec in "2:1 2 3" "13:1 2 3" "14:2 3 4" "3:4 5 6" "16:4 5 6" "17:5 6 7" "18:5 6"; do
  c=${spec%%:*}; ds=${spec#*:}
  for d in $ds; do
    python bench.py --config $c --path gemm --karatsuba $d --configs none --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/d.json 2>/dev/null; python tools/line.py "cfg$c d$d" < gpurun_out/d.json
  done
done
