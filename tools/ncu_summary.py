"""Summarise an ncu report: per kernel time, DRAM bytes, tensor-pipe activity,
top stall reasons, and the hottest SASS instructions (needs -lineinfo).

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--source]
"""
import csv
import io
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    rep = sys.argv[1]
    hdr, units, rows = raw(rep)
    ix = {h: i for i, h in enumerate(hdr)}
    stall = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("_per_issue_active.ratio")]
    for r in rows:
        def g(k, d=""):
            return r[ix[k]] if k in ix else d
        name = g("Kernel Name")[:90]
        print(f"== {name}")
        print(f"   time {g('gpu__time_duration.sum')} {units[ix['gpu__time_duration.sum']]}"
              f"  dram rd {g('dram__bytes_read.sum')} {units[ix['dram__bytes_read.sum']]}"
              f"  wr {g('dram__bytes_write.sum')} {units[ix['dram__bytes_write.sum']]}"
              f"  tensor% {g('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active')}"
              f"  regs {g('launch__registers_per_thread')}  warps% {g('sm__warps_active.avg.pct_of_peak_sustained_active')}"
              f"  smem-excess {g('derived__memory_l1_wavefronts_shared_excessive')}")
        st = sorted(((float(r[ix[k]] or 0), k) for k in stall), reverse=True)[:7]
        print("   stalls: " + ", ".join(f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}" for v, k in st))
    if "--source" in sys.argv:
        out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                             capture_output=True, text=True).stdout
        lines = list(csv.reader(io.StringIO(out)))
        hdr2 = None
        data = []
        for ln in lines:
            if "Source" in ln and "Warp Stall Sampling (All Samples)" in ln:
                hdr2 = ln
                continue
            if hdr2 and len(ln) == len(hdr2):
                try:
                    data.append((int(ln[hdr2.index("Warp Stall Sampling (All Samples)")]), ln[hdr2.index("Source")].strip()))
                except ValueError:
                    pass
        tot = sum(d[0] for d in data) or 1
        agg = {}
        for s, src in data:
            toks = src.split()
            op = (toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")).split(".")[0]
            agg[op] = agg.get(op, 0) + s
        print("   samples by opcode: " + ", ".join(f"{k}={100 * v / tot:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]))
        for s, src in sorted(data, reverse=True)[:12]:
            print(f"     {100 * s / tot:5.1f}%  {src[:80]}")


if __name__ == "__main__":
    main()
