"""Where the B = 1024 reconstruct time goes: 4 x 256-frame ModalBasis.reconstruct
calls vs the bare tc_decode2 launches on precomputed coefficients."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2502_05339_b200 import device as dv
from paper_2502_05339_b200.runtime import ModalBasis

n, r = 50331648, 200
U = dv.alloc_tall(n, r, torch.float32, "col")
U.buf[:r].normal_()
rng = np.random.default_rng(0)
lam = 0.99 * np.exp(1j * rng.uniform(0.05, 1.0, r))
W = (rng.standard_normal((r, r)) + 1j * rng.standard_normal((r, r))) / np.sqrt(2 * r)
b = rng.standard_normal(r) + 1j * rng.standard_normal(r)
mb = ModalBasis(U, W, lam, b)
mb.release_fp32()
del U
times = rng.uniform(0, 300, 1024)
out = torch.empty((256, n), dtype=torch.float32, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for rep in range(2):
    torch.cuda.synchronize(); ev[0].record()
    for c0 in range(0, 1024, 256):
        mb.reconstruct(times[c0:c0 + 256], out=out)
    ev[1].record(); torch.cuda.synchronize()
    full = ev[0].elapsed_time(ev[1])
    Cs = [mb.coefficients(times[c0:c0 + 256]) for c0 in range(0, 1024, 256)]
    torch.cuda.synchronize(); ev[0].record()
    for C in Cs:
        dv.get_ops().tc_decode(mb.tc_state(), C, out=out)
    ev[1].record(); torch.cuda.synchronize()
    bare = ev[0].elapsed_time(ev[1])
    torch.cuda.synchronize(); ev[0].record()
    for c0 in range(0, 1024, 256):
        mb.coefficients(times[c0:c0 + 256])
    ev[1].record(); torch.cuda.synchronize()
    coef = ev[0].elapsed_time(ev[1])
    print(f"full {full:.2f} ms  bare tc_decode {bare:.2f} ms  coefficients {coef:.2f} ms")
