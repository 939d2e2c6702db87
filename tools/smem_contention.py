"""MMA-rate probe under shared-memory store contention: the E2M1 stage shape
(form 5, two 224-row N tiles) while another warp stores k B/clk into shared
memory (qrng_debug_mma_rate form 5 + 16k).  The product kernel's transform
warps write ~15 B/clk of A operand per SM."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_04130_b200 as q
q.load_library()
n = 224 | (224 << 9)
for k in [0, 4, 8, 16, 24, 32, 48, 64]:
    r = max(q.mma_rate(5 + 16 * k, n) for _ in range(3))
    print("writer_B_per_clk", k, round(r * 2 / 1e12, 1), "TOPS")
