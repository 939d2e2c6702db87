#!/usr/bin/env python
"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) by kernel.

    python tools/launch_summary.py launches.csv [--per N]   (N = extractions in the capture)
"""
import collections, csv, sys


def main():
    path = sys.argv[1]
    per = int(sys.argv[sys.argv.index("--per") + 1]) if "--per" in sys.argv else 1
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    iN, iM, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    for r in rows[1:]:
        k = r[iN].split("(")[0][-40:]
        agg[k][r[iM]] += float(r[iV].replace(",", ""))
        if r[iM] == "gpu__time_duration.sum":
            cnt[k] += 1
    tot = sum(v["gpu__time_duration.sum"] for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
        t = v["gpu__time_duration.sum"]
        print(f"{k:42s} x{cnt[k] // per:3d} {t / per / 1000:9.1f} us {100 * t / tot:5.1f}%  "
              f"rd {v.get('dram__bytes_read.sum', 0) / per / 1e6:8.1f} MB  wr {v.get('dram__bytes_write.sum', 0) / per / 1e6:8.1f} MB")


if __name__ == "__main__":
    main()
