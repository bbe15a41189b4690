"""Pin the CPU oracle (oracle/) against the reference.

Two sources of truth:
  * known-answer values copied from the reference's own GTest suites
    (cited file:line below);
  * tests/golden/cases.json, produced by the UNMODIFIED reference library via
    oracle/_ref/ref_harness (tests/golden/make_golden.py).
"""
import math

import numpy as np
import pytest

import oracle
from golden_util import (case_by_name, check_plan, check_report, check_world, load_cases,
                         meta_for, model_for)


# ----------------------------------------------------------- known answers
def test_payload_witness_frozen_bits():
    # exchange_test.cpp:41-47
    assert oracle.payload_value(1, 0, 0) == 0.46704238970739009
    assert oracle.payload_value(1, 0, 1) == 0.53572046009155783
    assert oracle.payload_value(2, 7, 3) == 0.7723988757309479
    assert oracle.payload_value(1, 2, 3) != oracle.payload_value(3, 2, 1)


def test_workload_goldens():
    # workload_model_test.cpp:52-62: gamma=1 reduces to raw FLOPs; gamma 0.385
    assert oracle.gamma_weighted_workload(1024, 3072, 1.0) == 244813135872.0
    assert abs(oracle.gamma_weighted_workload(1024, 3072, 0.385) - 236888921210.88) <= 1e-3
    assert oracle.gamma_weighted_workload(0, 3072, 0.49) == 0.0


def test_workload_strictly_increasing_in_length():
    # workload_model_test.cpp:64-72 -- also what lets the device sort key on
    # (workload bits) behave like (length); we check the bits path anyway.
    prev = oracle.gamma_weighted_workload(0)
    for l in list(range(1, 5000)) + [65536, 131072, 1 << 20]:
        w = oracle.gamma_weighted_workload(l)
        assert w > prev
        prev = w


def test_assign_hand_trace_with_fallback():
    # balancer_test.cpp:33-49
    ids, w, bags = oracle.assign_to_bags([0, 1, 2, 3], [10, 8, 5, 1], [1, 1])
    assert list(ids) == [0, 1, 2, 3]
    assert list(bags) == [0, 1, 1, 0]
    loads = [sum(x for x, b in zip(w, bags) if b == j) for j in range(2)]
    assert loads == [11, 13]


def test_assign_spread_single_tiebreak_zero():
    # balancer_test.cpp:51-83
    _, _, bags = oracle.assign_to_bags([0, 1, 2, 3], [4, 4, 4, 4], [1, 1, 1, 1])
    assert sorted(bags) == [0, 1, 2, 3]
    _, _, bags = oracle.assign_to_bags([0, 1, 2], [4, 1, 9], [1])
    assert list(bags) == [0, 0, 0]
    ids, _, _ = oracle.assign_to_bags([7, 3, 9], [5, 5, 8], [1])
    assert list(ids) == [9, 3, 7]
    with pytest.raises(ValueError):
        oracle.assign_to_bags([0], [1], [])
    with pytest.raises(ValueError):
        oracle.assign_to_bags([0], [-1], [1])
    assert len(oracle.assign_to_bags([0, 1], [0, 0], [1, 1])[0]) == 2


def test_chunk_lengths():
    # balancer_test.cpp:85-95
    assert oracle.chunk_lengths(10, 2) == [5, 5]
    assert oracle.chunk_lengths(10, 4) == [3, 3, 2, 2]
    assert oracle.chunk_lengths(3, 8) == [1, 1, 1, 0, 0, 0, 0, 0]


def test_wir_rules():
    # metrics.cpp:20-31
    assert oracle.wir([0.0, 0.0]) == 1.0
    assert math.isinf(oracle.wir([0.0, 1.0]))
    assert oracle.wir([2.0, 4.0]) == 2.0


def test_topology_grammar():
    assert oracle.parse_topology("g1n2+g2n1+g4n1").bag_sizes == [1, 1, 2, 4]
    for bad in ["", "g", "g0n1", "x1n1", "g1n1+", "g1n1x"]:
        with pytest.raises(ValueError):
            oracle.parse_topology(bad)


# ---------------------------------------------------------- golden fixtures
CASES = [c["name"] for c in load_cases()]


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference(name):
    c = case_by_name(name)
    case, ref = c["case"], c["result"]
    meta = meta_for(case)
    assert [[[int(i), int(l)] for i, l in zip(meta.ids[r], meta.lens[r])] for r in range(meta.world)] == ref["meta"]
    d, h, g = model_for(case)
    topo = oracle.parse_topology(case["topology"])
    if "error" in ref:
        with pytest.raises(ValueError):
            oracle.plan_routing(meta, topo, d, h, g)
        return
    plan, rep = oracle.plan_routing(meta, topo, d, h, g)
    check_plan(plan, ref["plan"])
    check_report(rep, ref["report"])
    rev = oracle.reverse_plan(plan)
    check_plan(rev, ref["reverse"])  # std::sort tie order included
    check_plan(oracle.identity_plan(meta), ref["identity"])
    assert oracle.reverse_plan(rev).recv == plan.recv  # involution on ours too

    if not case.get("route"):
        return
    w0 = oracle.make_world(meta, case["payload_width"], h)
    check_world(w0, ref["world0"])
    routed = oracle.route(w0, plan)
    check_world(routed, ref["routed"])
    for u in ref.get("ulysses", []):
        bag = topo.bag_ranks(u["bag"])
        bag = [case_by_rank + u["replica"] * topo.unit_size for case_by_rank in bag]
        staged = oracle.World(routed.row_bytes, routed.n_heads, list(routed.ranks))
        full = oracle.pre_attn(staged, bag)
        assert full == u["full_lens"]
        check_world(staged, u["pre"])
        oracle.post_attn(staged, bag)
        assert oracle.worlds_equal(staged, routed) == u["post_identity"] is True
    mutated = oracle.perturb(routed)
    check_world(mutated, ref["mutated"], checksum=False)
    back = oracle.reverse_route(mutated, plan)
    check_world(back, ref["returned"], checksum=False)
    assert ref["roundtrip_identity"] is True
    assert oracle.worlds_equal(oracle.reverse_route(routed, plan), w0)
