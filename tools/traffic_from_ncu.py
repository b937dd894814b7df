"""Summarise an ncu launch list captured with
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv
into (a) a per-kernel table (launches, device-time share, DRAM bytes per
launch) and (b) profiles/dominant_kernel_traffic.json, which bench.py reads
for roofline.traffic.

  python tools/traffic_from_ncu.py gpurun_out/r2_c3_launches.csv profiles/r02_launches_bench_c3.txt [--config=c3]

Per-launch times under ncu are serialised and cold-cache: compare shares,
not absolute times. DRAM bytes are per launch and do not depend on that.
"""
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
BSCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
OURS = ("tall_gemm", "tall_gram", "gram_reduce", "decode", "table_apply", "split_", "tc_decode", "residual",
        "pair_stats", "synth3d", "colmajor")


def short(name):
    return name.split("(")[0].replace("void ", "").split("<")[0].replace("fdmd::", "")


def main():
    src, dst = sys.argv[1], sys.argv[2]
    with open(src) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    launches = defaultdict(dict)
    meta = {}
    for r in csv.DictReader(lines):
        key = int(r["ID"])
        m, u, v = r["Metric Name"], r["Metric Unit"], float(r["Metric Value"].replace(",", ""))
        if m == "gpu__time_duration.sum":
            v *= SCALE.get(u, 1e-6)
        else:
            v *= BSCALE.get(u, 1.0)
        launches[key][m] = v
        meta[key] = (r["Kernel Name"], r["Grid Size"], r["Block Size"])
    # steps of bench.py: a step starts at the first tall_gram / tall_gemm after a tc_decode
    # (fit -> reconstruct); keep the last COMPLETE step (a later step start exists)
    ids = sorted(launches)
    starts, seen_rec = [], True
    for k in ids:
        s = short(meta[k][0])
        if "tc_decode" in s:
            seen_rec = True
        elif ("tall_gemm" in s or "tall_gram" in s) and seen_rec:   # the fit's first tall kernel
            starts.append(k)
            seen_rec = False
    if "--all" not in sys.argv and len(starts) >= 2:
        lo, hi = starts[-2], starts[-1]
        launches = {k: v for k, v in launches.items() if lo <= k < hi}
    agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    total = 0.0
    for k, d in launches.items():
        s = short(meta[k][0])
        t = d.get("gpu__time_duration.sum", 0.0)
        agg[s][0] += 1
        agg[s][1] += t
        agg[s][2] += d.get("dram__bytes_read.sum", 0.0)
        agg[s][3] += d.get("dram__bytes_write.sum", 0.0)
        total += t
    out = [f"# {os.path.basename(src)}: {len(launches)} launches of one complete bench step "
           f"(fit + reconstruct), "
           f"{total:.1f} ms device time under ncu",
           "# kernel | launches | ms total | share | DRAM read GB/launch | DRAM write GB/launch | libfdmd?"]
    for s, (n, t, rd, wr) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        ours = "yes" if any(o in s for o in OURS) else ""
        out.append(f"{s[:60]:60s} {n:5d} {t:10.2f} {t / total:6.1%} {rd / n / 1e9:9.3f} {wr / n / 1e9:9.3f} {ours}")
    # dominant libfdmd kernel by device time
    ours = [(t, s) for s, (n, t, rd, wr) in agg.items() if any(o in s for o in OURS)]
    dom = max(ours)[1]
    n, t, rd, wr = agg[dom]
    per = [{"grid": meta[k][1], "ms": round(d.get("gpu__time_duration.sum", 0.0), 3),
            "dram_read_GB": round(d.get("dram__bytes_read.sum", 0.0) / 1e9, 3),
            "dram_write_GB": round(d.get("dram__bytes_write.sum", 0.0) / 1e9, 3)}
           for k, d in sorted(launches.items()) if short(meta[k][0]) == dom]
    out.append("")
    out.append(f"# dominant libfdmd kernel: {dom} ({n} launches, {t / total:.1%} of device time)")
    for p in per:
        out.append(f"   grid {p['grid']:>14s}  {p['ms']:9.3f} ms  read {p['dram_read_GB']:8.3f} GB  "
                   f"write {p['dram_write_GB']:8.3f} GB")
    with open(dst, "w") as f:
        f.write("\n".join(out) + "\n")
    js = {"kernel": dom, "source": os.path.relpath(dst, ROOT), "launches": n,
          "traffic_bytes_per_launch": (rd + wr) / n, "dram_read_bytes_per_launch": rd / n,
          "dram_write_bytes_per_launch": wr / n, "share_of_device_time_under_ncu": round(t / total, 4),
          "per_launch": per,
          "kernels": {s: {"launches": a[0], "traffic_bytes_per_launch": (a[2] + a[3]) / a[0],
                          "share_of_device_time_under_ncu": round(a[1] / total, 4)}
                      for s, a in agg.items() if any(o in s for o in OURS)}}
    # keyed by bench config (bench.py's traffic_from_profiles reads configs[<config>])
    config = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--config=")), "c3")
    path = os.path.join(ROOT, "profiles", "dominant_kernel_traffic.json")
    try:
        allj = json.load(open(path))
    except Exception:
        allj = {}
    if "configs" not in allj:
        allj = {"configs": {}}
    allj["configs"][config] = js
    with open(path, "w") as f:
        json.dump(allj, f, indent=1)
    print("\n".join(out[:30]))


if __name__ == "__main__":
    main()
