"""Per-phase cycle trace of the fused planner (diagnostics, needs a GPU).

    python tools/trace_planner.py [c2|c1|c1:<n>] [topology] [small|hybrid|large]
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
if cfg.startswith("c1"):  # c1 (256 sequences) or c1:<n>
    n = int(cfg.split(":")[1]) if ":" in cfg else 256
    ids, lens = datagen.metadata("c1", 8, seed=1, step=0, per_rank=n // 8)
    topo = "g1n8"
else:
    ids, lens = datagen.metadata("scenario", 8, codes=C2, step=0, seed=7)
    topo = "g1n4+g2n2"
if len(sys.argv) > 2:
    topo = sys.argv[2]
dm = sb.DeviceMeta.from_lists(ids, lens)
p = sb.Planner(topo, 8, max_seqs=sum(len(x) for x in ids))
if len(sys.argv) > 3:
    p.set_path(sys.argv[3])
p.trace(True)
for _ in range(5):
    p.plan(dm)
torch.cuda.synchronize()
t = p.trace(True)
if p.last_path() == "hybrid":  # three kernels: per-kernel spans (clocks of different SMs)
    print("hybrid: prefix", int(t[12] - t[0]), "greedy chain", int(t[15] - t[14]), "suffix", int(t[13] - t[11]),
          "cycles")
    sys.exit(0)
names = ["load", "seq+totals+offsets", "sort", "greedy+dup", "emit+wir", "lists", "ties"]
marks = [int(x) for x in t[:7]] + [int(t[13])]
for i, n in enumerate(names):
    print(f"{n:20s} {marks[i + 1] - marks[i]:8d} cycles")
print("total", int(t[13] - t[0]), "cycles")
sub = {"P1 totals chain done": 11, "P1 origin offsets done": 12, "P4 per-seq pass done (max)": 10,
       "P5 offsets done (warp 0)": 7, "P5 rank lists done (max)": 8, "P5 send lists done (max)": 9}
for k, i in sub.items():
    if t[i] > 0:
        print(f"  {k:32s} +{int(t[i] - t[0]):8d} cycles from start")
if t[15] > t[14] > 0:
    print("greedy chain (replica 0):", int(t[15] - t[14]), "cycles;", "phase 3 start -> chain",
          int(t[14] - t[3]), "chain end -> phase 4", int(t[4] - t[15]))
if os.environ.get("SB_TRACE_P3"):
    print("P3 setup: phase 3 start -> greedy entry", int(t[11] - t[3]), "-> target divided", int(t[12] - t[11]),
          "-> chain start", int(t[14] - t[12]))
    print("P3 epilogue: chain end -> greedy return", int(t[7] - t[15]), "-> q pass", int(t[8] - t[7]),
          "-> bag bases", int(t[9] - t[8]), "-> phase 4", int(t[4] - t[9]))
