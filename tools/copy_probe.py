"""torch copy_ bandwidth vs size on this GPU (read + write bytes), for
context on the route copy's roofline fraction at its own size."""
import torch
for mb in (56, 112, 224, 448, 1024, 2048):
    n = mb << 20
    a = torch.empty(n, dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    for _ in range(3):
        b.copy_(a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(10):
        e0.record()
        b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{mb:5d} MB copy: {best * 1000:8.1f} us  {2 * n / (best * 1e-3) / 1e9:7.1f} GB/s")
