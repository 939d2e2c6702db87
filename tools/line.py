#!/usr/bin/env python
"""Print the key fields of a bench.py JSON line read from stdin (quick A/B runs).
    python bench.py ... | python tools/line.py LABEL"""
import json, sys
lab = sys.argv[1] if len(sys.argv) > 1 else ""
lines = [l for l in sys.stdin.read().splitlines() if l.startswith("{")]
if not lines:
    print(lab, "NO LINE"); sys.exit(0)
d = json.loads(lines[-1])
r = d.get("roofline") or {}
c = d.get("config", {})
out = [lab, round(d["value"], 2), "steady", round((d.get("steady_state") or {}).get("value", 0), 2),
       c.get("path"), "d", c.get("karatsuba_depth"), "leaves", c.get("karatsuba_leaves"),
       "frac", round(r.get("frac", 0), 3), "mb", round(r.get("frac_of_mma_microbench", 0), 3),
       "kern_us", round(r.get("kernel_ms_per_step", 0) * 1e3, 1),
       "aux_us", round((r.get("aux") or {}).get("ms_per_step", 0) * 1e3, 1),
       (d.get("parity") or {}).get("status")]
print(*out)
