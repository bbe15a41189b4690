"""Regenerate the golden fixtures from the UNMODIFIED reference.

Runs oracle/_ref/ref_harness (the reference seqbal library compiled from
/root/reference/proj/src by oracle/Makefile, driven through its public C++
API) on every case below and writes tests/golden/cases.json.  The committed
fixture pins both the C oracle (tests/test_oracle_golden.py) and the CUDA
path (tests/test_gpu_parity.py) without needing /root/reference at test time.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

FLUX = {"d_model": 3072, "n_heads": 24, "d_head": 128, "n_blocks": 57, "gamma": 0.49}
SMALL4 = {"d_model": 64, "n_heads": 4, "d_head": 16, "n_blocks": 2, "gamma": 0.49}  # exchange_test.cpp:17-22
SMALL8 = {"d_model": 64, "n_heads": 8, "d_head": 8, "n_blocks": 2, "gamma": 0.49}

# Data scenarios; codes are reference data_sim grammar.
C2_CODES = ["g2b8i256f1s0", "g2b4i512f1s0", "g2b2i768f1s0", "g2b1i1024f1s0"]
C3_CODES = ["g1b1i1024f51s1", "g1b1i512f85s1", "g2b2i512f1s0", "g2b4i256f1s0", "g2b1i1024f1s0"]


def explicit(lens, ids=None):
    m = {"kind": "explicit", "lens": lens}
    if ids is not None:
        m["ids"] = ids
    return m


def cases():
    out = []

    def add(name, **kw):
        c = {"world": kw.pop("world"), "topology": kw.pop("topology"), "model": kw.pop("model", FLUX),
             "meta": kw.pop("meta")}
        c.update(kw)
        out.append((name, c))

    # Hand cases mirroring the reference tests' shapes.
    add("split10_g2n1", world=2, topology="g2n1", model=SMALL4, meta=explicit([[10], []]),
        payload_width=8, route=True, ulysses=True)
    add("serial_parallel_g2n2", world=4, topology="g2n2", model=SMALL4,
        meta=explicit([[100, 3], [57], [13, 13, 13], []]), payload_width=8, route=True, ulysses=True)
    add("mutated_g2n1", world=2, topology="g2n1", model=SMALL4, meta=explicit([[40, 7], [11]]),
        payload_width=8, route=True, ulysses=True)
    add("bag4_g4n1", world=4, topology="g4n1", model=SMALL4, meta=explicit([[23, 5], [], [], []]),
        payload_width=8, route=True, ulysses=True)
    add("ulysses_g4n1_3seq", world=4, topology="g4n1", model=SMALL4, meta=explicit([[100, 37, 5], [], [], []]),
        payload_width=8, route=True, ulysses=True)
    add("zero_len_g8n1", world=8, topology="g8n1", model=SMALL8,
        meta=explicit([[0, 3, 0], [], [], [], [], [], [], []]), payload_width=8, route=True, ulysses=True)
    add("all_zero_g1n2", world=2, topology="g1n2", model=SMALL4, meta=explicit([[0, 0], [0]]),
        payload_width=8, route=True, ulysses=False)
    add("empty_world_g1n4", world=4, topology="g1n4", model=SMALL4, meta=explicit([[], [], [], []]),
        payload_width=8, route=True, ulysses=False)
    add("balanced_g1n4", world=4, topology="g1n4", meta=explicit([[500], [500], [500], [500]]))
    add("single_loaded_g8n1", world=8, topology="g8n1",
        meta=explicit([[800, 640, 320], [], [], [], [], [], [], []]), payload_width=24, route=True, ulysses=True)
    add("replicas_g1n2_w4", world=4, topology="g1n2", meta=explicit([[1000], [10], [2000], [20]]),
        payload_width=24, route=True, ulysses=False)
    add("reverse_mix_g1n2+g2n1", world=4, topology="g1n2+g2n1",
        meta=explicit([[900, 30], [64], [4096], [128, 128]]), payload_width=24, route=True, ulysses=True)
    add("head_reject_g8n1_12heads", world=8, topology="g8n1",
        model={"d_model": 3072, "n_heads": 12, "d_head": 256, "n_blocks": 57, "gamma": 0.49},
        meta=explicit([[10], [], [], [], [], [], [], []]))
    add("explicit_ids_tiebreak", world=2, topology="g1n2",
        meta=explicit([[300, 300, 300], [300]], ids=[[7, 3, 9], [1]]), payload_width=24, route=True)

    # Randomised small cases (heterogeneous bags, ragged/empty ranks, zeros).
    rng = random.Random(20250806)
    topos = [("g1n4", 4), ("g2n2", 4), ("g4n1", 4), ("g1n2+g2n1", 4), ("g1n1+g2n1+g1n1", 4),
             ("g1n2", 4), ("g2n1", 4), ("g1n2+g2n1+g4n1", 16), ("g8n1", 8), ("g2n1+g1n2+g4n1", 8)]
    for t in range(40):
        topo, world = topos[t % len(topos)]
        lens = [[rng.choice([0, 1, 2, 3, rng.randint(1, 200), rng.randint(1, 4096)])
                 for _ in range(rng.randint(0, 4))] for _ in range(world)]
        model = SMALL8 if "g8" in topo else SMALL4
        add(f"rand{t:02d}_{topo}", world=world, topology=topo, model=model, meta=explicit(lens),
            payload_width=8, route=True, ulysses=True)

    # Bench-shaped configs (plans in full, worlds as digests at width 24).
    for topo in ["g1n8", "g2n4", "g4n2", "g8n1", "g1n4+g2n2"]:
        add(f"c1_{topo}", world=8, topology=topo,
            meta={"kind": "c1", "seed": 1, "step": 0, "per_rank": 32}, payload_width=24,
            route=True, ulysses=True)
    for topo in ["g1n8", "g2n4", "g1n4+g2n2"]:
        add(f"c2_{topo}", world=8, topology=topo,
            meta={"kind": "scenario", "codes": C2_CODES, "group_size": 8, "step": 0, "seed": 7},
            payload_width=24, route=True, ulysses=True)
    for topo in ["g4n2", "g8n1"]:
        add(f"c3_{topo}", world=8, topology=topo,
            meta={"kind": "scenario", "codes": C3_CODES, "group_size": 8, "step": 0, "seed": 7},
            payload_width=24, route=True, ulysses=True)
    add("c1_two_replicas_g1n2+g2n1+g4n1", world=16, topology="g1n2+g2n1+g4n1",
        meta={"kind": "c1", "seed": 3, "step": 5, "per_rank": 6}, payload_width=24, route=True, ulysses=True)
    # C5-like: a few steps of the dynamic stream (plan only, digests).
    for step in range(3):
        add(f"c5_step{step}_g2n4", world=8, topology="g2n4", full=False,
            meta={"kind": "scenario", "codes": C2_CODES, "group_size": 8, "step": step, "seed": 11})

    # C4 plan-scaling sweep: digests only.
    for n in [256, 1024, 4096, 16384]:
        for topo in ["g1n8", "g2n4", "g4n2", "g8n1"]:
            add(f"c4_n{n}_{topo}", world=8, topology=topo, full=False,
                meta={"kind": "c1", "seed": 4, "step": 0, "per_rank": n // 8})
    return out


def main():
    if not oracle.ref_available():
        oracle.build(quiet=False)
    res = []
    for name, case in cases():
        print(name, flush=True)
        res.append({"name": name, "case": case, "result": oracle.ref_run("dump", case, timeout=1800)})
    with open(os.path.join(HERE, "cases.json"), "w") as f:
        json.dump(res, f, separators=(",", ":"))
    print("wrote", len(res), "cases")


if __name__ == "__main__":
    main()
