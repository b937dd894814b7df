import sys, torch
sys.path.insert(0, '.')
from paper_2502_05339_b200 import device as dv
n, r = 12582912, 200
B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
ops = dv.get_ops()
U = dv.alloc_tall(n, r, torch.float32, "col"); U.buf.normal_()
tcb = ops.tc_basis(U)
coef = torch.randn(r, B, dtype=torch.float32, device="cuda")
out = torch.empty((B, n), dtype=torch.float32, device="cuda")
for _ in range(2):
    ops.tc_decode(tcb, coef, out=out)
torch.cuda.synchronize()
print("ok")
