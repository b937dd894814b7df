"""Time the fp32 -> fp16 hi/lo basis split (tc_basis) at config-4 size."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2502_05339_b200 import device as dv

n, r = 50331648, 200
U = dv.alloc_tall(n, r, torch.float32, "col")
U.buf.normal_()
ops = dv.get_ops()
t = ops.tc_basis(U)
del t
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
e[0].record()
t = ops.tc_basis(U)
e[1].record()
torch.cuda.synchronize()
ms = e[0].elapsed_time(e[1])
print(f"split_basis {ms:.2f} ms  {(8.0 * n * r) / ms / 1e6:.0f} GB/s (read 4nr + write 4nr)")
