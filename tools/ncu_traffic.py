#!/usr/bin/env python
"""dram__bytes_read.sum + dram__bytes_write.sum per launch of each captured
dominant kernel (one `ncu --set full` capture per workload) as the JSON that
bench.py reads for roofline.traffic (profiles/ncu_traffic.json).

    python tools/ncu_traffic.py TAG gpurun_out/TAG_*.ncu-rep > traffic.json
"""
import csv, json, os, re, subprocess, sys

WORKLOAD = {"cfg1": "cfg1_n1024", "cfg2": "cfg2_n8192", "cfg3": "cfg3_n65536", "cfg4": "cfg4a_n1048576",
            "cfg41": "cfg4b_n1048576", "next4": "next4_n2^24"}
tag, reps = sys.argv[1], sys.argv[2:]
out = {}
for rep in reps:
    name = os.path.basename(rep)[len(tag) + 1:-len(".ncu-rep")]  # e.g. gemm_cfg2, ntt_segment_cfg5_n2^19
    m = re.match(r"(gemm|bits|ntt_segment|ntt_pass)_(cfg\d+|next4)(?:_(n2\^\d+))?$", name)
    if not m:
        continue
    kind, cfg, pt = m.groups()
    wl = f"cfg5_{pt}" if pt else WORKLOAD[cfg]
    path = kind if kind in ("gemm", "bits") else "ntt"
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    h, u, v = r[0], r[1], r[2]  # names, units, values
    SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9}

    def val(k):
        if k not in h:
            return None
        i = h.index(k)
        return float(v[i].replace(",", "")) * SCALE.get(u[i], 1)
    rd, wr, t = val("dram__bytes_read.sum"), val("dram__bytes_write.sum"), val("gpu__time_duration.sum")
    key = f"{wl}/{path}" if kind != "ntt_pass" else f"{wl}/ntt_pass"
    out[key] = {"bytes_per_launch": (rd or 0) + (wr or 0), "dram_read": rd, "dram_write": wr,
                "duration_ns_under_ncu": t, "kernel": kind,
                "source": f"profiles/{tag}_{name} (ncu --set full, one launch, clocks not locked)"}
json.dump(out, sys.stdout, indent=1)
print()
