"""Multi-kernel planner stage times by CUDA events (diagnostics):
prep | sort | greedy | emit | lists at a few sizes (C1 law, 8 ranks, g1n8).

    python tools/plan_timing.py [n ...]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_06001_b200 as sb  # noqa: E402
from paper_2508_06001_b200 import datagen  # noqa: E402

for n in [int(x) for x in sys.argv[1:]] or [2048, 4096, 16384]:
    ids, lens = datagen.metadata("c1", 8, seed=1, step=0, per_rank=n // 8)
    dm = sb.DeviceMeta.from_lists(ids, lens)
    p = sb.Planner("g1n8", 8, max_seqs=n)
    p.set_path("large")
    p.enable_timing(True)
    for _ in range(5):
        p.plan(dm)
    torch.cuda.synchronize()
    t = p.timing()
    print(n, {k: round(v, 1) for k, v in t.items()}, "sum", round(sum(t.values()), 1), flush=True)
