"""Fused single-CTA planner vs hybrid vs the multi-kernel path: plan latency
by CUDA graph replay (C1 law, 8 ranks) -- picks the auto-path thresholds
(diagnostics).

    python tools/path_compare.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_06001_b200 as sb  # noqa: E402
from paper_2508_06001_b200 import datagen  # noqa: E402


def plan_us(p, dm, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            p.plan(dm, s)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                p.plan(dm, s)
        g.replay()
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
        s.synchronize()
    return 1000 * e0.elapsed_time(e1) / reps


sizes = [int(x) for x in sys.argv[1:]] or [64, 128, 256, 512, 768, 1024, 1536, 2048]
for n in sizes:
    ids, lens = datagen.metadata("c1", 8, seed=1, step=0, per_rank=max(1, n // 8))
    dm = sb.DeviceMeta.from_lists(ids, lens)
    row = []
    for topo in ("g1n8", "g2n4", "g4n2"):
        for path in ("small", "hybrid", "large"):
            p = sb.Planner(topo, 8, max_seqs=n)
            p.set_path(path)
            row.append(f"{topo}/{path} {plan_us(p, dm):7.1f}")
    print(n, " | ".join(row), flush=True)
