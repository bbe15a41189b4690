"""Regenerate the upstream-generator and C5 stream fixtures from the
UNMODIFIED reference (oracle/_ref/ref_harness, built by oracle/Makefile).

  tests/golden/batches.json -- next_batch (data_sim.cpp:225-248) per rank for
      several scenarios / seeds / steps, and parse_data_code verdicts
      (data_sim.cpp:39-76) incl. ParseError offsets;
  tests/golden/uniform.json -- balance_uniform_items / reverse_uniform_plan
      (balancer.cpp:411-462) on hand and random count vectors;
  tests/golden/stream.json  -- all 1000 steps of the C5 schedule planned
      by plan_routing: per-step tokens, sequences, chunks, WIR and total
      workload bits, capacity violations.

    python tests/golden/make_stream_golden.py
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_2508_06001_b200.scenarios import C5_SCENARIOS, C5_SEED, C5_TOPOLOGY, C5_WORLD  # noqa: E402

C2 = ["g2b8i256f1s0", "g2b4i512f1s0", "g2b2i768f1s0", "g2b1i1024f1s0"]
C3 = ["g1b1i1024f51s1", "g1b1i512f85s1", "g2b2i512f1s0", "g2b4i256f1s0", "g2b1i1024f1s0"]

BATCH_CASES = [
    {"codes": C2, "world": 8, "seed": 7, "steps": [0, 1, 5, 999]},
    {"codes": C3, "world": 8, "seed": 7, "steps": [0, 3]},
    {"preset": "lowres_image", "world": 32, "seed": 1, "steps": [0, 2]},
    {"preset": "mixed_image", "world": 32, "seed": 3735928559, "steps": [0, 7]},
    {"preset": "joint_image_video", "world": 64, "seed": 42, "steps": [0, 1000000]},
    {"text": "# C5 joint-8\ngroup_size 8\ng2b4i256f1s0\ng1b5i512f1s0  # tail comment\n\ng1b1i2048f1s0\n"
             "g1b10i256f4s0\ng1b1i512f4s0\ng1b2i256f85s1\ng1b1i512f85s1\n", "world": 16, "seed": 11,
     "steps": [0, 1]},
] + [{"codes": c, "world": C5_WORLD, "seed": C5_SEED, "steps": [0, 1, 2, 3, 4, 5, 17]} for c in C5_SCENARIOS]

PARSE = ["g1b1i16f1s0", "g8b32i256f1s0", "g1048576b1i16f1s1", "", "x1b1i16f1s0", "g0b1i16f1s0", "gb1i16f1s0",
         "g1b0i16f1s0", "g1b1i250f1s0", "g1b1i0f1s0", "g1b1i16f0s0", "g1b1i16f1s2", "g1b1i16f1s0x",
         "g1048577b1i16f1s0", "g1b1i16f1", "g1b1i16f1s", "g2b2i256f1s01"]


def harness(cmd, payload):
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_harness")
    p = subprocess.run([exe, cmd], input=json.dumps(payload).encode(), capture_output=True, check=True)
    return json.loads(p.stdout)


def main():
    batches = harness("batches", {"cases": BATCH_CASES, "parse": PARSE})
    batches["inputs"] = {"cases": BATCH_CASES, "parse": PARSE}
    with open(os.path.join(HERE, "batches.json"), "w") as f:
        json.dump(batches, f, separators=(",", ":"))
    stream = harness("stream", {"world": C5_WORLD, "topology": C5_TOPOLOGY,
                                "scenarios": [{"codes": c} for c in C5_SCENARIOS], "seed": C5_SEED,
                                "steps": 1000, "full_every": 0})
    stream["inputs"] = {"world": C5_WORLD, "topology": C5_TOPOLOGY, "scenarios": C5_SCENARIOS, "seed": C5_SEED}
    with open(os.path.join(HERE, "stream.json"), "w") as f:
        json.dump(stream, f, separators=(",", ":"))
    import random
    rng = random.Random(2508)
    counts = [[4, 0], [3, 3, 3], [5, 0, 0], [0], [0, 0, 0, 0], [7], [1, 0, 0, 0, 0, 0, 0, 9], [2, -1]]
    for _ in range(60):
        w = rng.choice([2, 3, 4, 8, 16, 64])
        counts.append([rng.choice([0, rng.randint(0, 5), rng.randint(0, 200)]) for _ in range(w)])
    uni = harness("uniform", {"counts": counts})
    with open(os.path.join(HERE, "uniform.json"), "w") as f:
        json.dump(uni, f, separators=(",", ":"))
    print("wrote batches.json, stream.json and uniform.json")


if __name__ == "__main__":
    main()
