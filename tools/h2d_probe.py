"""Host<->device copy bandwidth probe (pinned, pageable, pitched/staged)."""
import time

import torch

n = 1 << 30  # 1 GiB
for pin in (True, False):
    h = torch.empty(n, dtype=torch.uint8, pin_memory=pin)
    h.fill_(1)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        d.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"H2D pinned={pin}: {n / dt / 1e9:.1f} GB/s")
    torch.cuda.synchronize()
    t = time.perf_counter()
    h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    print(f"D2H pinned={pin}: {n / (time.perf_counter() - t) / 1e9:.1f} GB/s")
big = torch.empty((10 << 30) // 4, dtype=torch.float32, pin_memory=True)
d = torch.empty_like(big, device="cuda")
torch.cuda.synchronize()
t = time.perf_counter()
d.copy_(big, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D pinned 10 GiB: {big.numel() * 4 / (time.perf_counter() - t) / 1e9:.1f} GB/s")
