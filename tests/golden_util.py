"""Helpers for the committed reference fixtures (tests/golden/cases.json)."""
from __future__ import annotations

import functools
import json
import os
import struct

import numpy as np

import oracle

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cases.json")


@functools.lru_cache(maxsize=1)
def load_cases():
    with open(GOLDEN) as f:
        return json.load(f)


def case_by_name(name):
    for c in load_cases():
        if c["name"] == name:
            return c
    raise KeyError(name)


def hexd(x: int) -> str:
    return f"{x:016x}"


def dbits(d: float) -> str:
    return hexd(struct.unpack("<Q", struct.pack("<d", d))[0])


def meta_for(case) -> oracle.Meta:
    m = case["meta"]
    W = case["world"]
    if m["kind"] == "explicit":
        return oracle.meta_explicit(m["lens"], m.get("ids"))
    if m["kind"] == "c1":
        return oracle.meta_c1(W, m["per_rank"], m["seed"], m["step"])
    if m["kind"] == "scenario":
        return oracle.meta_scenario(W, m["codes"], m["step"], m["seed"])
    raise ValueError(m["kind"])


def model_for(case):
    md = case["model"]
    return md["d_model"], md["n_heads"], md["gamma"]


def chunks_digest(c_id, c_idx, c_start, c_end, c_src, c_dst) -> str:
    n = len(c_id)
    words = np.zeros((n, 6), np.uint64)
    words[:, 0] = np.asarray(c_id, np.uint64)
    words[:, 1] = np.asarray(c_idx, np.int64).astype(np.uint64)
    words[:, 2] = np.asarray(c_start, np.int64).astype(np.uint64)
    words[:, 3] = np.asarray(c_end, np.int64).astype(np.uint64)
    words[:, 4] = np.asarray(c_src, np.int64).astype(np.uint64)
    words[:, 5] = np.asarray(c_dst, np.int64).astype(np.uint64)
    return hexd(oracle.digest(words))


def lists_digest(lists) -> str:
    w = []
    for l in lists:
        w.append(len(l))
        w.extend(int(x) for x in l)
    return hexd(oracle.digest(np.asarray(w, np.uint64)))


def segs_digest(segs) -> str:
    w = []
    for l in segs:
        w.append(len(l))
        for s in l:
            w.extend([int(s[0]), int(s[1]) % 2**64, int(s[2]) % 2**64])
    return hexd(oracle.digest(np.asarray(w, np.uint64)))


def plan_digests(plan: oracle.Plan) -> dict:
    return {
        "n_chunks": plan.n_chunks,
        "chunks_digest": chunks_digest(plan.c_id, plan.c_idx, plan.c_start, plan.c_end, plan.c_src, plan.c_dst),
        "send_digest": lists_digest(plan.send),
        "recv_digest": lists_digest(plan.recv),
        "origin_digest": segs_digest(plan.origin),
        "target_digest": segs_digest(plan.target),
    }


def check_plan(plan: oracle.Plan, ref: dict, recv_ties_ok: bool = False):
    """Compare a plan (oracle or device) with a reference plan_json entry."""
    d = plan_digests(plan)
    assert d["n_chunks"] == ref["n_chunks"]
    assert d["chunks_digest"] == ref["chunks_digest"]
    assert d["send_digest"] == ref["send_digest"]
    assert d["origin_digest"] == ref["origin_digest"]
    assert d["target_digest"] == ref["target_digest"]
    if d["recv_digest"] != ref["recv_digest"]:
        assert recv_ties_ok, "recv lists differ"
        # Only permutations among equal (segment, start) keys are allowed.
        assert "recv" in ref
        for r, (mine, theirs) in enumerate(zip(plan.recv, ref["recv"])):
            key = lambda c: (int(plan.c_start[c]), int(plan.c_id[c]))
            assert [key(c) for c in mine] == [key(c) for c in theirs], f"rank {r}"
            assert sorted(mine) == sorted(theirs)
    if "chunks" in ref:
        assert plan.chunk_rows() == [tuple(c) for c in ref["chunks"]]
        assert plan.send == ref["send"]
        assert [[tuple(s) for s in r] for r in plan.origin] == [[tuple(s) for s in r] for r in ref["origin"]]
        assert [[tuple(s) for s in r] for r in plan.target] == [[tuple(s) for s in r] for r in ref["target"]]


def check_report(rep: oracle.Report, ref: dict):
    assert [dbits(x) for x in rep.per_gpu_workload] == ref["per_gpu_workload"]
    assert [dbits(x) for x in rep.per_bag_occupancy] == ref["per_bag_occupancy"]
    assert rep.capacity_violations == ref["capacity_violations"]
    assert dbits(rep.total_workload) == ref["total_workload"]
    assert dbits(rep.wir) == ref["wir"]


def world_summary(world: oracle.World) -> dict:
    ranks = []
    for b in world.ranks:
        i, p, pl = oracle.rank_digests(b)
        ranks.append({"rows": b.rows, "width": (b.payload.shape[1] if b.payload.ndim == 2 else world.row_bytes) // 8,
                      "head_lo": b.head_lo, "head_hi": b.head_hi, "mode": b.mode,
                      "ids_digest": hexd(i), "pos_digest": hexd(p), "payload_digest": hexd(pl),
                      "segments": [list(s) for s in b.segments]})
    return {"ranks": ranks, "checksum": hexd(oracle.checksum(world))}


def check_world(world: oracle.World, ref: dict, checksum: bool = True):
    got = world_summary(world) if checksum else {"ranks": world_summary(world)["ranks"]}
    assert len(got["ranks"]) == len(ref["ranks"])
    for r, (a, b) in enumerate(zip(got["ranks"], ref["ranks"])):
        for k in ("rows", "width", "head_lo", "head_hi", "mode", "ids_digest", "pos_digest", "payload_digest"):
            assert a[k] == b[k], f"rank {r} {k}: {a[k]} != {b[k]}"
        assert [list(s) for s in a["segments"]] == [list(s) for s in b["segments"]], f"rank {r} segments"
    if checksum:
        assert got["checksum"] == ref["checksum"]
