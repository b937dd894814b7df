"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by
kernel: launches, total device time and share. Per-launch times under ncu are
cold-cache and serialised — compare shares, not absolutes.

  python tools/launch_summary.py gpurun_out/launches.csv [top]
"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.DictReader(lines)
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        short = name.split("(")[0].replace("void ", "")[:90]
        unit = r.get("Metric Unit", "ns")
        v = float(r["Metric Value"].replace(",", ""))
        v = v * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
        agg[short][0] += 1
        agg[short][1] += v
        total += v
    print(f"{'kernel':92s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
    for k, (c, ms) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{k:92s} {c:8d} {ms:10.2f} {100 * ms / total:6.1f}%")
    print(f"{'TOTAL':92s} {sum(c for c, _ in agg.values()):8d} {total:10.2f}")


if __name__ == "__main__":
    main()
