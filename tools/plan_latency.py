"""C2 plan latency: eager events and CUDA graph replay, plus the kernel's own
cycle trace (diagnostics).   python tools/plan_latency.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_06001_b200 as sb  # noqa: E402
from paper_2508_06001_b200 import datagen  # noqa: E402

C2 = ["g2b8i256f1s0", "g2b4i512f1s0", "g2b2i768f1s0", "g2b1i1024f1s0"]
ids, lens = datagen.metadata("scenario", 8, codes=C2, step=0, seed=7)
dm = sb.DeviceMeta.from_lists(ids, lens)
p = sb.Planner("g1n4+g2n2", 8, max_seqs=sum(len(x) for x in ids))
for _ in range(5):
    p.plan(dm)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    p.plan(dm)
e1.record()
torch.cuda.synchronize()
eager = 1000 * e0.elapsed_time(e1) / 50
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    p.plan(dm)
g.replay()
torch.cuda.synchronize()
e0.record()
for _ in range(50):
    g.replay()
e1.record()
torch.cuda.synchronize()
graph = 1000 * e0.elapsed_time(e1) / 50
p.trace(True)
p.plan(dm)
torch.cuda.synchronize()
t = p.trace(True)
print(f"eager {eager:.2f} us  graph {graph:.2f} us  kernel {int(t[13] - t[0])} cycles")
