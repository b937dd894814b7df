"""Time the tcgen05 reconstruction at config-4 size (n = 50,331,648, r = 200).

    python tools/prof_tc.py [--n N]
GB/s = algorithmic bytes (U once per launch as fp32-equivalent 4*n*r, frames
4*n*B) / launch time, CUDA events.
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_05339_b200 import device as dv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=50331648)
    ap.add_argument("--r", type=int, default=200)
    ap.add_argument("--batches", type=int, nargs="*", default=[32, 128, 256, 384, 512, 640])
    a = ap.parse_args()
    n, r = a.n, a.r
    ops = dv.get_ops()
    U = dv.alloc_tall(n, r, torch.float32, "col")
    U.buf.normal_()
    tcb = ops.tc_basis(U)
    del U
    torch.cuda.empty_cache()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    free, total = torch.cuda.mem_get_info()
    print(f"mem free {free/1e9:.1f} GB of {total/1e9:.1f} GB after the split basis")
    for B in a.batches:
        coef = torch.randn(r, B, dtype=torch.float32, device="cuda")
        out = torch.empty((B, n), dtype=torch.float32, device="cuda")
        ops.tc_decode(tcb, coef, out=out)
        ts = []
        for _ in range(3):
            ev[0].record(); ops.tc_decode(tcb, coef, out=out); ev[1].record(); torch.cuda.synchronize()
            ts.append(ev[0].elapsed_time(ev[1]))
        ms = min(ts)
        gbs = (4.0 * n * r + 4.0 * n * B) / ms / 1e6
        print(f"tc_decode B={B:5d}  {ms:8.3f} ms  {B / ms * 1e3:9.1f} frames/s  {gbs:8.1f} GB/s")
        del out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
