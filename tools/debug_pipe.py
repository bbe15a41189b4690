"""Diagnostics: capture multigpu.PlanAhead.pair() in a CUDA graph with one
process (device barriers) and print where capture fails."""
import os
import sys
import traceback

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2508_06001_b200 as sb  # noqa: E402
from paper_2508_06001_b200 import multigpu  # noqa: E402

os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29611")
dist.init_process_group("gloo", rank=0, world_size=1)
torch.cuda.set_device(0)
W, topo = 8, sys.argv[1] if len(sys.argv) > 1 else "g2n4"
meta = oracle.meta_c1(W, 5, 2, 0)
group = multigpu.PeerGroup(barrier_mode="device")
planner = sb.Planner(topo, W, max_seqs=64)
rows = int(sum(int(x.sum()) for x in meta.lens))
mk = lambda: multigpu.make_world(group, W, 4, [64], capacity_rows=rows, max_bag=planner.max_bag)
A, B, Cw, D, E = mk(), mk(), mk(), mk(), mk()
gathers = [multigpu.MetaGather(group, W, 8), multigpu.MetaGather(group, W, 8)]
for g in gathers:
    g.set_local(meta.ids, meta.lens)
dm = gathers[0].gather()
A.layout_origin(dm)
A.fill_witness(dm)
phases = multigpu.x_phases(A, B, Cw, D, E, planner.max_bag > 1)
pipe = multigpu.PlanAhead(group, gathers, [planner, sb.Planner(topo, W, max_seqs=64)], phases)
pipe.prime()
for _ in range(2):
    pipe.pair()
torch.cuda.synchronize()
print("eager ok")
mode = sys.argv[2] if len(sys.argv) > 2 else "global"
try:
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, capture_error_mode=mode):
        pipe.pair()
    g.replay()
    torch.cuda.synchronize()
    print("graph ok", mode)
    for r in range(W):
        assert np.array_equal(E.read_rank(1, r), A.read_rank(1, r))
    print("round trip ok")
except Exception:
    traceback.print_exc()
