"""Launch each libfdmd hot kernel once at a fixed size (for ncu captures).

  python tools/prof_kernels.py [--n 6291456] [--which all|gemm|gram|syrk|decode]
"""

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_05339_b200 import device as dv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=6291456)
    ap.add_argument("--m", type=int, default=201)
    ap.add_argument("--l", type=int, default=200)
    ap.add_argument("--which", default="all")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    ops = dv.get_ops()
    n, m, l = a.n, a.m, a.l
    S = dv.alloc_tall(n, m, torch.float32, "row")
    S.buf.normal_()
    Q = dv.alloc_tall(n, l, torch.float64, "row")
    Om = torch.randn(m, l, dtype=torch.float64, device="cuda")
    U = dv.alloc_tall(n, l, torch.float32, "col")
    U.buf.normal_()
    coef = torch.randn(l, 32, dtype=torch.float32, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for _ in range(a.reps):
        res = {}
        if a.which in ("all", "gemm"):
            ev[0].record(); ops.tall_gemm(S, Om, Q); ev[1].record(); torch.cuda.synchronize()
            res["gemm S*Om"] = (ev[0].elapsed_time(ev[1]), 2.0 * n * m * l)
        if a.which in ("all", "syrk"):
            ev[0].record(); ops.tall_gram(Q, Q, symmetric=True); ev[1].record(); torch.cuda.synchronize()
            res["syrk QtQ"] = (ev[0].elapsed_time(ev[1]), 1.0 * n * l * l)
        if a.which in ("all", "gram"):
            ev[0].record(); ops.tall_gram(S, Q); ev[1].record(); torch.cuda.synchronize()
            res["gram StQ"] = (ev[0].elapsed_time(ev[1]), 2.0 * n * m * l)
            ev[0].record(); ops.tall_gram(Q, S); ev[1].record(); torch.cuda.synchronize()
            res["gram QtS"] = (ev[0].elapsed_time(ev[1]), 2.0 * n * m * l)
        if a.which in ("all", "trsm"):
            R = torch.triu(torch.randn(l, l, dtype=torch.float64, device="cuda"))
            ev[0].record(); ops.tall_gemm(Q, R, Q); ev[1].record(); torch.cuda.synchronize()
            res["gemm QR inplace"] = (ev[0].elapsed_time(ev[1]), 2.0 * n * l * l)
            ev[0].record(); ops.tall_gemm(Q, R, Q, upper=True); ev[1].record(); torch.cuda.synchronize()
            res["trsm QR upper"] = (ev[0].elapsed_time(ev[1]), 1.0 * n * l * l)
        if a.which in ("all", "decode"):
            out = torch.empty((32, n), dtype=torch.float32, device="cuda")
            ev[0].record(); ops.decode(U, coef, out=out); ev[1].record(); torch.cuda.synchronize()
            res["decode B=32"] = (ev[0].elapsed_time(ev[1]), 2.0 * n * l * 32)
            ev[0].record(); ops.decode(U, coef[:, :1], out=out[:1]); ev[1].record(); torch.cuda.synchronize()
            res["decode B=1"] = (ev[0].elapsed_time(ev[1]), 4.0 * n * l)
        for k, (ms, fl) in res.items():
            unit = "GB/s" if k == "decode B=1" else "TF/s"
            val = fl / ms / 1e6 if unit == "GB/s" else fl / ms / 1e9
            print(f"{k:18s} {ms:8.3f} ms  {val:8.2f} {unit}")


if __name__ == "__main__":
    main()
