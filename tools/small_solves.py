"""Latency of the fit's r x r solves on the device (r = 200): the SVD of
B = Q^T X (gesvdj / gesvd / gesvda through torch, cuSOLVER) and the
eigenvalues of K (cuSOLVER Xgeev via libfdmd, torch.linalg.eigvals).

  python tools/small_solves.py
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_05339_b200 import device as dv  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return min(ts), float(np.median(ts))


def main():
    r = 200
    rng = np.random.default_rng(0)
    # a B with a DMD-like spectrum: singular values over 4 decades
    U = np.linalg.qr(rng.standard_normal((r, r)))[0]
    V = np.linalg.qr(rng.standard_normal((r, r)))[0]
    s = np.logspace(3, -1, r)
    B = torch.as_tensor((U * s) @ V.T, device="cuda")
    K = torch.as_tensor(rng.standard_normal((r, r)) / np.sqrt(r), device="cuda")
    ops = dv.get_ops()
    rows = {}
    for drv in ("gesvdj", "gesvd", "gesvda"):
        try:
            rows[f"svd {drv}"] = timeit(lambda: torch.linalg.svd(B, full_matrices=False, driver=drv))
        except Exception as exc:   # pragma: no cover
            rows[f"svd {drv}"] = repr(exc)
    rows["eigh(B^T B) (syevd)"] = timeit(lambda: torch.linalg.eigh(B.t() @ B))
    rows["Xgeev values only"] = timeit(lambda: ops.geev(K, vectors=False))
    rows["Xgeev with vectors"] = timeit(lambda: ops.geev(K, vectors=True))
    rows["torch eigvals (cuda)"] = timeit(lambda: torch.linalg.eigvals(K))
    rows["qr 200x200 (geqrf)"] = timeit(lambda: torch.linalg.qr(K))
    for k, v in rows.items():
        print(f"{k:28s} {v if isinstance(v, str) else f'min {v[0]:7.2f} ms  median {v[1]:7.2f} ms'}")


if __name__ == "__main__":
    main()

