"""Uniform (T5) balancer on the device: plan + item exchange + reverse.

The paper's appendix balancer for identical-cost items: T5-encoded prompts
(512 tokens x 4096 bf16 = 4 MB each) held unevenly by the ranks of the C2
stream (8/8/4/4/2/2/1/1 images per rank) are evened out, then sent home.
Prints one JSON line (device-timed, CUDA events; HBM GB/s of the copies).

    python tools/bench_uniform.py
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_06001_b200 as sb  # noqa: E402

W, RPI, ROW = 8, 512, 8192  # ranks, rows per item (tokens), bytes per row (4096 bf16)
counts = [8, 8, 4, 4, 2, 2, 1, 1]
items = sum(counts)
mk = lambda: sb.World(W, 8, [ROW], capacity_rows=items * RPI)
A, B, C = mk(), mk(), mk()
lens = [[c * RPI] if c else [] for c in counts]
ids = [[r + 1] if c else [] for r, c in enumerate(counts)]
dm = sb.DeviceMeta.from_lists(ids, lens)
A.layout_origin(dm)
A.fill_witness(dm)
ub = sb.UniformBalancer(W)
d_counts = torch.tensor(counts, dtype=torch.int64, device="cuda")
for _ in range(5):
    ub.plan(d_counts)
    ub.route(A, B, rows_per_item=RPI)
    ub.route(B, C, rows_per_item=RPI, reverse=True)
torch.cuda.synchronize()
C.status()
assert C.compare(A) == 0, "uniform round trip not bit-exact"
plan = ub.plan(d_counts).download()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
K = 50
ms = np.zeros(3)
for _ in range(K):
    ev[0].record()
    ub.plan(d_counts)
    ev[1].record()
    ub.route(A, B, rows_per_item=RPI)
    ev[2].record()
    ub.route(B, C, rows_per_item=RPI, reverse=True)
    ev[3].record()
    torch.cuda.synchronize()
    ms += [ev[i].elapsed_time(ev[i + 1]) for i in range(3)]
ms /= K
moved = 2 * items * RPI * (ROW + 16)  # every row read + written once per exchange (kept rows copied too)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json"))).get("hbm_gbs", 6550.4)
print(json.dumps({
    "bench": "uniform (T5) balancer: balance_uniform_items + item exchange + reverse (balancer.cpp:411-462)",
    "counts": counts, "final_counts": plan["final_counts"], "moves": plan["moves"],
    "total_moved": plan["total_moved"], "item_bytes": RPI * (ROW + 16),
    "plan_us": 1000 * ms[0], "route_us": 1000 * ms[1], "reverse_us": 1000 * ms[2],
    "route_gbs": moved / (ms[1] * 1e-3) / 1e9, "reverse_gbs": moved / (ms[2] * 1e-3) / 1e9,
    "hbm_peak_gbs": peak, "round_trip_bit_exact": True}))
