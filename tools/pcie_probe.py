"""Raw pinned-memory copy bandwidth on this box (H2D, D2H, both at once), and
H2D while the SMs stream HBM copies (the e2e situation: the upload of step
k+1 runs under step k's exchanges)."""
import torch

n = 224 << 20
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
big_a = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
big_b = torch.empty_like(big_a)
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def timed(stream, fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


print("h2d", f"{n / timed(s1, h2d) / 1e6:.1f} GB/s")
print("d2h", f"{n / timed(s2, d2h) / 1e6:.1f} GB/s")


def both():
    h2d()
    d2h()
    s1.wait_stream(s2)


print("both", f"{2 * n / timed(s1, both) / 1e6:.1f} GB/s (sum)")


def h2d_loaded():
    with torch.cuda.stream(s3):  # ~6 TB/s of device copies beside the upload
        for _ in range(12):
            big_b.copy_(big_a)
    h2d()


print("h2d under HBM copy load", f"{n / timed(s1, h2d_loaded, reps=5) / 1e6:.1f} GB/s")
