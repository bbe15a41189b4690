"""Per-phase cycle trace of the fused planner (diagnostics, needs a GPU).

    python tools/trace_planner.py [c2|c1]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_06001_b200 as sb  # noqa: E402
from paper_2508_06001_b200 import datagen  # noqa: E402

C2 = ["g2b8i256f1s0", "g2b4i512f1s0", "g2b2i768f1s0", "g2b1i1024f1s0"]
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
if cfg == "c1":
    ids, lens = datagen.metadata("c1", 8, seed=1, step=0, per_rank=32)
    topo = "g1n8"
else:
    ids, lens = datagen.metadata("scenario", 8, codes=C2, step=0, seed=7)
    topo = "g1n4+g2n2"
dm = sb.DeviceMeta.from_lists(ids, lens)
p = sb.Planner(topo, 8, max_seqs=sum(len(x) for x in ids))
p.trace(True)
for _ in range(5):
    p.plan(dm)
torch.cuda.synchronize()
t = p.trace(True)
names = ["load", "workload", "offsets", "dup", "totals", "sort", "greedy", "bases", "emit", "offsets2",
         "rank_lists", "send", "wir"]
d = np.diff(t[:14])
for n, c in zip(names, d):
    print(f"{n:12s} {int(c):8d} cycles")
print("total", int(t[13] - t[0]), "cycles")
