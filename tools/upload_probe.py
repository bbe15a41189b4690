"""Why the e2e upload sometimes runs below the PCIe probe: H2D bandwidth of a
224 MB image from pinned buffers allocated three ways (diagnostics):
torch pin_memory=True (cudaHostAlloc), and anonymous mmap + MADV_HUGEPAGE +
cudaHostRegister (2 MB pages: fewer IOMMU translations)."""
import mmap
import os

import torch

N = 36372 * 6144
print("THP:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip()
      if os.path.exists("/sys/kernel/mm/transparent_hugepage/enabled") else "n/a")
s = torch.cuda.Stream()
dev = torch.empty(N, dtype=torch.uint8, device="cuda")


def rate(h, reps=8):
    with torch.cuda.stream(s):
        dev.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    with torch.cuda.stream(s):
        for _ in range(reps):
            dev.copy_(h, non_blocking=True)
    e1.record(s)
    torch.cuda.synchronize()
    return N * reps / e0.elapsed_time(e1) / 1e6


def thp_pinned(n):
    m = mmap.mmap(-1, n + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    m.madvise(mmap.MADV_HUGEPAGE)
    t = torch.frombuffer(m, dtype=torch.uint8)
    t.fill_(0)  # fault the pages in (as huge pages where possible)
    off = (-t.data_ptr()) % (2 << 20)
    t = t[off:off + n]
    rc = torch.cuda.cudart().cudaHostRegister(t.data_ptr(), n, 0)
    assert int(rc) == 0, rc
    return t, m


for trial in range(3):
    a = torch.empty(N, dtype=torch.uint8, pin_memory=True)
    b, keep = thp_pinned(N)
    c = torch.empty(N, dtype=torch.uint8).pin_memory()
    print(f"trial {trial}: pin_memory=True {rate(a):.1f} GB/s  thp+register {rate(b):.1f} GB/s  "
          f".pin_memory() {rate(c):.1f} GB/s")
    del a, c
