"""Per-phase planner latency across the C4 sweep (diagnostics, needs a GPU).

Large path: CUDA events between the planner kernels (sb_planner_timing).
Small path: clock64 stamps per phase of the fused single-CTA planner.

    python tools/plan_profile.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_06001_b200 as sb  # noqa: E402
from paper_2508_06001_b200 import datagen  # noqa: E402

SMALL = ["load", "workload", "offsets", "dup", "totals", "sort", "greedy", "bases", "emit", "offsets2",
         "rank_lists", "send", "wir"]
C2 = ["g2b8i256f1s0", "g2b4i512f1s0", "g2b2i768f1s0", "g2b1i1024f1s0"]
for n in (sys.argv[1:] or ["c2", 256, 512, 1024, 2048, 4096, 16384]):
    n = n if n == "c2" else int(n)
    if n == "c2":
        ids, lens = datagen.metadata("scenario", 8, codes=C2, step=0, seed=7)
        n = sum(len(x) for x in ids)
        topos = ["g1n4+g2n2"]
    else:
        ids, lens = datagen.metadata("c1", 8, seed=1, step=0, per_rank=n // 8)
        topos = ["g1n8", "g2n4", "g8n1"]
    dm = sb.DeviceMeta.from_lists(ids, lens)
    for topo in topos:
        for path in (["small", "large"] if n <= 2048 else ["large"]):
            p = sb.Planner(topo, 8, max_seqs=n)
            p.set_path(path)
            if path == "small":
                p.trace(True)
                for _ in range(5):
                    p.plan(dm)
                torch.cuda.synchronize()
                t = p.trace(True)
                d = np.diff(t[:14])
                print(f"n={n} {topo} small: total {int(t[13]-t[0])} cyc;",
                      " ".join(f"{a}={int(c)}" for a, c in zip(SMALL, d)),
                      f"| greedy setup={int(t[14]-t[6])} chain={int(t[15]-t[14])} epilogue={int(t[7]-t[15])}"
                      if t[15] > t[14] > t[6] > 0 else "")
            else:
                p.enable_timing(True)
                for _ in range(5):
                    p.plan(dm)
                torch.cuda.synchronize()
                tm = p.timing()
                print(f"n={n} {topo} large:", " ".join(f"{k}={v:.1f}" for k, v in tm.items()))
