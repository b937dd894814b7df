"""Panel-Gram launch geometry sweep at config-3 size (n = 50,331,648): the
three Grams of the fit — X^T X (S fp32, symmetric 200), Q1^T Q1 (Q fp64,
symmetric 200) and Q^T S (200 x 201) — timed with CUDA events for several
row-split counts (FDMD_GRAM_SPLITS, read per call by panel_plan).

  python tools/gram_sweep.py [--n 50331648] [--splits 0,99,148,296,444]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_05339_b200 import device as dv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=50331648)
    ap.add_argument("--splits", default="0,99,148,296,444,592")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--after-hbm", action="store_true",
                    help="also time each Gram right after ~130 ms of HBM streaming (the bench's reconstruct phase)")
    a = ap.parse_args()
    ops = dv.get_ops()
    n, m, l = a.n, 201, 200
    S = dv.alloc_tall(n, m, torch.float32, "row")
    S.buf.normal_()
    Q = dv.alloc_tall(n, l, torch.float64, "row")
    Q.buf.normal_()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    Um = torch.randn((200, 200), dtype=torch.float64, device="cuda") / 200.0
    cases = {
        "XtX f32 sym 200": (lambda: ops.tall_gram(S, S, K1=200, K2=200, symmetric=True), 1.0 * n * 200 * 200),
        "XtX+border f32 sym 200|1": (lambda: ops.tall_gram_bordered(S, 200), 1.0 * n * 200 * 200 + 2.0 * n * 200),
        "Xts_m border alone": (lambda: ops.tall_tdot(S, 200, 200), 2.0 * n * 200),
        "lift S Umap planes K=200": (lambda: ops.tall_gemm_planes(S, Um, bound=1e3), 2.0 * n * 200 * 200),
        "QtQ f64 sym 200": (lambda: ops.tall_gram(Q, Q, symmetric=True), 1.0 * n * 200 * 200),
        "QtS f64xf32 200x201": (lambda: ops.tall_gram(Q, S), 2.0 * n * 200 * 201),
    }
    out = {}
    for sp in [int(x) for x in a.splits.split(",")]:
        if sp > 0:
            os.environ["FDMD_GRAM_SPLITS"] = str(sp)
        else:
            os.environ.pop("FDMD_GRAM_SPLITS", None)
        for name, (fn, fl) in cases.items():
            fn()
            torch.cuda.synchronize()
            best = 1e9
            for _ in range(a.reps):
                ev[0].record()
                fn()
                ev[1].record()
                torch.cuda.synchronize()
                best = min(best, ev[0].elapsed_time(ev[1]))
            key = f"{name} splits={sp or 'default'}"
            out[key] = {"ms": round(best, 2), "TFLOPs_alg": round(fl / best / 1e9, 2)}
            print(f"{key:40s} {best:8.2f} ms  {fl / best / 1e9:6.2f} TF/s", flush=True)
    if a.after_hbm:
        os.environ.pop("FDMD_GRAM_SPLITS", None)
        big = torch.empty((8 << 30) // 4, dtype=torch.float32, device="cuda")
        big2 = torch.empty_like(big)
        for name, (fn, fl) in cases.items():
            for rep in range(a.reps):
                for _ in range(8):          # 8 x 16 GB moved ~ 130 ms at ~6.5 TB/s
                    big2.copy_(big)
                ev[0].record()
                fn()
                ev[1].record()
                torch.cuda.synchronize()
                ms = ev[0].elapsed_time(ev[1])
                key = f"{name} after HBM streaming #{rep}"
                out[key] = {"ms": round(ms, 2), "TFLOPs_alg": round(fl / ms / 1e9, 2)}
                print(f"{key:40s} {ms:8.2f} ms  {fl / ms / 1e9:6.2f} TF/s", flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
