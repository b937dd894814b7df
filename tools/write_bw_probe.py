import torch, time
n = 6 * 1024**3  # 24 GB f32
x = torch.empty(n, dtype=torch.float32, device="cuda")
y = torch.empty(n // 2, dtype=torch.float32, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for name, fn, byt in [("fill", lambda: x.fill_(1.0), 4 * n), ("copy", lambda: y.copy_(x[: n // 2]), 4 * n),
                      ("strided-frames", lambda: x.view(256, -1)[:, : 50331648 // 2].fill_(2.0), 4 * 256 * 50331648 // 2)]:
    fn(); torch.cuda.synchronize()
    ev[0].record()
    for _ in range(3): fn()
    ev[1].record(); torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / 3
    print(f"{name}: {ms:.2f} ms  {byt / ms / 1e6:.0f} GB/s")
