"""Streamed snapshot upload (linalg.PendingUpload) bandwidth at config-3 size
for several chunk sizes, upload only (no per-chunk compute)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2502_05339_b200 import device as dv
from paper_2502_05339_b200 import linalg as la

n, m = 50331648, 201
host = torch.empty((n, m), dtype=torch.float32, pin_memory=True)
host[: n // 64].normal_()
S = dv.alloc_tall(n, m, torch.float32, "row", zero=True)
for mb in (256, 512, 1024, 2048):
    for rep in range(2):
        p = la.PendingUpload(host, S, chunk_bytes=mb << 20)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        p.run()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"chunk {mb:5d} MB: {host.numel() * 4 / dt / 1e9:.1f} GB/s ({dt * 1e3:.0f} ms)")
