"""Time the small dense r x r operations of the fit on the device (CUDA events).

    python tools/probe_small.py [r]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2502_05339_b200 import device as dv  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


def main():
    r = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    rng = np.random.default_rng(0)
    # a DMD-like operator: rotation-ish spectrum inside the unit disk
    Q, _ = np.linalg.qr(rng.standard_normal((r, r)))
    lam = 0.99 * np.exp(1j * rng.uniform(0, np.pi, r // 2))
    Dm = np.zeros((r, r))
    for k, z in enumerate(lam):
        Dm[2 * k:2 * k + 2, 2 * k:2 * k + 2] = [[z.real, -z.imag], [z.imag, z.real]]
    K = torch.as_tensor(Q @ Dm @ Q.T, device="cuda")
    G = torch.as_tensor(rng.standard_normal((4 * r, r)), device="cuda")
    G = G.T @ G
    B = torch.as_tensor(rng.standard_normal((r + 10, r + 1)), device="cuda")
    ops = dv.get_ops()
    out = {
        "geev_vectors_ms": timed(lambda: ops.geev(K, True)),
        "geev_values_ms": timed(lambda: ops.geev(K, False)),
        "torch_eig_ms": timed(lambda: torch.linalg.eig(K)),
        "svd_B_ms": timed(lambda: torch.linalg.svd(B, full_matrices=False)),
        "svdvals_B_ms": timed(lambda: torch.linalg.svdvals(B)),
        "svd_gesvdj_ms": timed(lambda: torch.linalg.svd(B[:r, :r], full_matrices=False, driver="gesvdj")),
        "svd_gesvda_ms": timed(lambda: torch.linalg.svd(B[:r, :r], full_matrices=False, driver="gesvda")),
        "svd_gesvd_sq_ms": timed(lambda: torch.linalg.svd(B[:r, :r], full_matrices=False, driver="gesvd")),
        "eigh_G_ms": timed(lambda: torch.linalg.eigh(G)),
        "cholesky_G_ms": timed(lambda: torch.linalg.cholesky(G)),
        "cholesky_ex_G_ms": timed(lambda: torch.linalg.cholesky_ex(G)),
        "solve_tri_ms": timed(lambda: torch.linalg.solve_triangular(torch.linalg.cholesky(G).mT,
                                                                    torch.eye(r, device="cuda", dtype=torch.float64),
                                                                    upper=True)),
        "cond_R_ms": timed(lambda: torch.linalg.cond(torch.linalg.cholesky(G).mT)),
        "eigvalsh_G_ms": timed(lambda: torch.linalg.eigvalsh(G)),
        "inv_ms": timed(lambda: torch.linalg.inv(G)),
        "qr_ms": timed(lambda: torch.linalg.qr(B)),
        "lstsq_ms": timed(lambda: torch.linalg.lstsq(B, B[:, :3])),
    }
    for k, v in out.items():
        print(f"{k:24s} {v:9.2f}")
    Bs = B[:r, :r]
    U1, s1, V1 = torch.linalg.svd(Bs, full_matrices=False, driver="gesvd")
    U2, s2, V2 = torch.linalg.svd(Bs, full_matrices=False, driver="gesvdj")
    print("gesvdj vs gesvd: sigma rel", float(((s2 - s1) / s1).abs().max()),
          " |U^T U2| diag min", float((U1.T @ U2).diagonal().abs().min()))


if __name__ == "__main__":
    main()


def overlap_probe(r=200):
    """Is cusolver Xgeev host-bound? Run it on a side stream while a large
    DMMA GEMM occupies the device; compare wall times."""
    from paper_2502_05339_b200.device import alloc_tall
    rng = np.random.default_rng(1)
    K = torch.as_tensor(rng.standard_normal((r, r)) / np.sqrt(r), device="cuda")
    ops = dv.get_ops()
    n = 1 << 24
    A = alloc_tall(n, r, torch.float64, "row", zero=True)
    C = alloc_tall(n, r, torch.float64, "row", zero=True)
    Bm = torch.eye(r, dtype=torch.float64, device="cuda")

    def gemm():
        for _ in range(3):
            ops.tall_gemm(A, Bm, C)

    t_gemm = timed(gemm, 2)
    t_geev = timed(lambda: ops.geev(K, False), 3)
    side = torch.cuda.Stream()

    def both():
        gemm()
        with torch.cuda.stream(side):
            ops.geev(K, False)
    t_both = timed(both, 2)
    print(f"gemm {t_gemm:.1f} ms  geev {t_geev:.1f} ms  gemm+geev(side stream) {t_both:.1f} ms")


if __name__ == "__main__" and len(sys.argv) > 2:
    overlap_probe(int(sys.argv[1]))
