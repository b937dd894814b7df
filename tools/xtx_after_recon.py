"""Is the fit's first Gram slowed by the reconstruct phase that precedes it
in a bench step? Times the config-3 snapshot Gram X^T X (n = 50.3 M, fp32,
symmetric 200) alone, right after 1024 frames of tcgen05 reconstruction
(config-4 basis, 256-frame launches), and after the same reconstruction
followed by an idle gap; prints the SM clock nvidia-smi reports around each.

  python tools/xtx_after_recon.py
"""
import os
import subprocess
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_05339_b200 import device as dv  # noqa: E402
from paper_2502_05339_b200.runtime import ModalBasis  # noqa: E402


def smi_clock():
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                              "--format=csv,noheader"], capture_output=True, text=True, timeout=10).stdout.strip()
        return out
    except Exception as exc:   # pragma: no cover
        return repr(exc)


def main():
    n, m, r = 50331648, 201, 200
    ops = dv.get_ops()
    S = dv.alloc_tall(n, m, torch.float32, "row")
    S.buf.normal_()
    U = dv.alloc_tall(n, r, torch.float32, "col")
    U.buf.normal_()
    rng = np.random.default_rng(4)
    lam = 0.99 * np.exp(1j * rng.uniform(0.05, 1.0, r))
    W = (rng.standard_normal((r, r)) + 1j * rng.standard_normal((r, r))) / np.sqrt(2 * r)
    b = rng.standard_normal(r) + 1j * rng.standard_normal(r)
    mb = ModalBasis(U, W, lam, b)
    mb.tc_state()
    mb.release_fp32()
    del U
    torch.cuda.empty_cache()
    times = rng.uniform(0.0, 300.0, 1024)
    out = torch.empty((256, n), dtype=torch.float32, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]

    def xtx():
        ev[0].record()
        ops.tall_gram(S, S, K1=200, K2=200, symmetric=True)
        ev[1].record()
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1])

    def recon():
        ev[2].record()
        for c0 in range(0, 1024, 256):
            mb.reconstruct(times[c0:c0 + 256], out=out)
        ev[3].record()

    for _ in range(2):
        xtx()
    for rep in range(3):
        t = xtx()
        print(f"alone                   XtX {t:7.2f} ms   smi after: {smi_clock()}", flush=True)
    for rep in range(3):
        recon()
        t = xtx()
        print(f"after recon (no gap)    XtX {t:7.2f} ms   recon {ev[2].elapsed_time(ev[3]):6.2f} ms  "
              f"smi after: {smi_clock()}", flush=True)
    for gap in (0.01, 0.05, 0.2, 1.0):
        recon()
        torch.cuda.synchronize()
        time.sleep(gap)
        t = xtx()
        print(f"after recon + {gap:4.2f} s   XtX {t:7.2f} ms", flush=True)


if __name__ == "__main__":
    main()
