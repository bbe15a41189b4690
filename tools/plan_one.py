"""One fused-planner launch at n sequences (C1 law) for ncu source captures.

    ncu -k regex:k_plan_small -c 1 --set full --import-source on python tools/plan_one.py 256 g1n8
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_06001_b200 as sb  # noqa: E402
from paper_2508_06001_b200 import datagen  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
topo = sys.argv[2] if len(sys.argv) > 2 else "g1n8"
path = sys.argv[3] if len(sys.argv) > 3 else "small"
ids, lens = datagen.metadata("c1", 8, seed=1, step=0, per_rank=n // 8)
dm = sb.DeviceMeta.from_lists(ids, lens)
p = sb.Planner(topo, 8, max_seqs=n)
p.set_path(path)
for _ in range(3):
    p.plan(dm)
torch.cuda.synchronize()
