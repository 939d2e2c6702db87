import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_04130_b200 as q
q.load_library()
for n0,n1 in [(192,192),(224,224),(224,0),(128,128),(256,0)]:
    form = 5 if n0 <= 224 else 4
    n = n0 | (n1 << 9) if form == 5 else n0
    r = max(q.mma_rate(form, n) for _ in range(3))
    print(form, n0, n1, round(r*2/1e12, 1), "TOPS")
