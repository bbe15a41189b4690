"""Host-side logic of the product package (no GPU): the bench's metadata
generators and the topology grammar, checked against the oracle."""
import numpy as np
import pytest

import oracle
from paper_2508_06001_b200 import api, datagen

C2 = ["g2b8i256f1s0", "g2b4i512f1s0", "g2b2i768f1s0", "g2b1i1024f1s0"]
C3 = ["g1b1i1024f51s1", "g1b1i512f85s1", "g2b2i512f1s0", "g2b4i256f1s0", "g2b1i1024f1s0"]


@pytest.mark.parametrize("seed,step,per", [(1, 0, 32), (4, 0, 2048), (3, 5, 6)])
def test_c1_generator_matches_oracle(seed, step, per):
    m = oracle.meta_c1(8, per, seed, step)
    for r in range(8):
        ids, lens = datagen.c1_batch(seed, step, r, per)
        assert np.array_equal(ids, m.ids[r]) and np.array_equal(lens, m.lens[r])


@pytest.mark.parametrize("codes,step,seed", [(C2, 0, 7), (C3, 0, 7), (C2, 2, 11),
                                             (["g32b32i256f1s0"], 3, 1),
                                             (["g8b2i256f85s1", "g4b1i512f85s1", "g4b1i2048f1s0"], 1, 5)])
def test_scenario_generator_matches_oracle(codes, step, seed):
    world = sum(datagen.parse_data_code(c)[0] for c in codes)
    m = oracle.meta_scenario(world, codes, step, seed)
    for r in range(world):
        ids, lens = datagen.next_batch(codes, r, step, seed)
        assert np.array_equal(ids, m.ids[r]) and np.array_equal(lens, m.lens[r])


def test_visual_tokens_known_values():
    # acceptance criterion 8: i512f85s1 == round(1024*mult)*25
    assert datagen.visual_tokens(512, 85, 1, 1.0) == 1024 * 25
    assert datagen.visual_tokens(256, 1, 0, 0.96) == round(256 * 0.96)
    assert datagen.visual_tokens(16, 1, 0, 0.5) == 1  # at least one token


@pytest.mark.parametrize("spec", ["g1n8", "g2n4", "g1n2+g2n1+g4n1", "g8n4", "g1n4+g2n2", "g3n1+g1n1"])
def test_topology_parse_matches_oracle(spec):
    assert api.parse_topology(spec).bag_sizes == oracle.parse_topology(spec).bag_sizes
    t = api.parse_topology(spec)
    assert api.parse_topology(t.format()).bag_sizes == t.bag_sizes  # format_topology round trip


@pytest.mark.parametrize("bad,offset", [("", 0), ("x", 0), ("g", 1), ("g0n1", 1), ("g1x", 2), ("g1n1+", 5),
                                        ("g1n1g", 4), ("g99999999n1", 1)])
def test_topology_parse_errors_carry_offset(bad, offset):
    # topology_test.cpp:56-71: malformed grammar rejected with byte offsets
    with pytest.raises(api.ParseError, match=rf"offset {offset}\)"):
        api.parse_topology(bad)


@pytest.mark.parametrize("bad,msg", [("g1048576n2", "unit size too large (at offset 0)"),
                                     ("g1024n1025", "unit size too large (at offset 0)"),
                                     ("g٣n1", "expected digits for bag size (at offset 1)"),
                                     ("g1048576n2+g1x", "expected 'n' (at offset 13)")])
def test_topology_unit_size_and_ascii_digits(bad, msg):
    # topology.cpp:16-27 (parse_int accepts '0'-'9' only) and :58 (unit size
    # checked after the whole spec parsed, offset 0)
    with pytest.raises(api.ParseError) as e:
        api.parse_topology(bad)
    assert str(e.value) == msg


def test_topology_largest_unit_accepted():
    assert api.parse_topology("g1048576n1").unit_size == 1 << 20
