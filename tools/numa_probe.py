"""H2D bandwidth from host buffers first-touched on each NUMA node (diagnostics):
explains the 46 vs 55 GB/s run-to-run spread of the e2e upload."""
import glob
import mmap
import os

import torch

p = torch.cuda.get_device_properties(0)
bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
node_file = f"/sys/bus/pci/devices/{bus}/numa_node"
print("gpu", bus, "numa_node", open(node_file).read().strip() if os.path.exists(node_file) else "n/a")
nodes = sorted(glob.glob("/sys/devices/system/node/node[0-9]*"))
print("nodes", [os.path.basename(n) for n in nodes], "affinity", len(os.sched_getaffinity(0)))


def cpus(node):
    out = set()
    for part in open(f"{node}/cpulist").read().strip().split(","):
        a, _, b = part.partition("-")
        out.update(range(int(a), int(b or a) + 1))
    return out


N = 224 << 20
dev = torch.empty(N, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
orig = os.sched_getaffinity(0)
for node in nodes:
    c = cpus(node) & orig
    if not c:
        continue
    os.sched_setaffinity(0, c)
    m = mmap.mmap(-1, N, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    t = torch.frombuffer(m, dtype=torch.uint8)
    t.fill_(1)
    os.sched_setaffinity(0, orig)
    assert int(torch.cuda.cudart().cudaHostRegister(t.data_ptr(), N, 0)) == 0
    with torch.cuda.stream(s):
        dev.copy_(t, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    with torch.cuda.stream(s):
        for _ in range(8):
            dev.copy_(t, non_blocking=True)
    e1.record(s)
    torch.cuda.synchronize()
    print(os.path.basename(node), f"{8 * N / e0.elapsed_time(e1) / 1e6:.1f} GB/s")
    torch.cuda.cudart().cudaHostUnregister(t.data_ptr())
    del t
