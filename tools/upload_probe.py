"""Why the e2e upload runs below the PCIe probe: time the same 224 MB
host->device image through sb_world_upload and through torch copies,
from the same pinned buffer (diagnostics)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_06001_b200 as sb  # noqa: E402

rows = 36372
sizes = [rows * 16, rows * 6144, rows * 16]
host = [torch.empty(n, dtype=torch.uint8).pin_memory() for n in sizes]
w = sb.World(8, 24, [6144], capacity_rows=rows, n_aux=1, aux_row_bytes=16) if False else None
s = torch.cuda.Stream()


def t(fn, reps=8):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


dev = [torch.empty(n, dtype=torch.uint8, device="cuda") for n in sizes]


def torch_copy():
    with torch.cuda.stream(s):
        for d, h in zip(dev, host):
            d.copy_(h, non_blocking=True)


big_h = torch.empty(sizes[1], dtype=torch.uint8, pin_memory=True)


def torch_copy_fresh():
    with torch.cuda.stream(s):
        dev[1].copy_(big_h, non_blocking=True)


for name, fn, nbytes in (("torch copy, .pin_memory() buffers", torch_copy, sum(sizes)),
                         ("torch copy, pin_memory=True buffer", torch_copy_fresh, sizes[1])):
    ms = t(fn)
    print(f"{name}: {ms:.3f} ms  {nbytes / ms / 1e6:.1f} GB/s")
print("host ptr alignment", [h.data_ptr() % 4096 for h in host], big_h.data_ptr() % 4096)
