"""Uniform (T5) balancer: the oracle against the unmodified reference
(tests/golden/uniform.json), and -- on the GPU -- the device plan and the
item exchange against the oracle, round trip bit-exact."""
import json
import os

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "uniform.json")) as f:
    GOLD = json.load(f)


@pytest.mark.parametrize("i", range(len(GOLD)))
def test_oracle_matches_reference(i):
    g = GOLD[i]
    if "error" in g:
        with pytest.raises(ValueError):
            oracle.balance_uniform_items(g["counts"])
        return
    final, moves, total = oracle.balance_uniform_items(g["counts"])
    assert final == g["final_counts"]
    assert [list(m) for m in moves] == g["moves"]
    assert total == g["total_moved"]
    assert [list(m) for m in oracle.reverse_uniform_plan(moves)] == g["reverse_moves"]
    assert max(final) - min(final) <= 1 if final else True


def test_reference_examples():
    """SPEC.md balance_uniform_items examples (balancer_test.cpp:298-332)."""
    assert oracle.balance_uniform_items([4, 0])[::2] == ([2, 2], 2)
    assert oracle.balance_uniform_items([3, 3, 3])[::2] == ([3, 3, 3], 0)
    f, _, t = oracle.balance_uniform_items([5, 0, 0])
    assert sorted(f) == [1, 2, 2] and t == 3


@pytest.mark.gpu
@pytest.mark.parametrize("i", [j for j, g in enumerate(GOLD) if "error" not in g and g["counts"]])
def test_device_plan_matches_reference(i):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2508_06001_b200 as sb
    g = GOLD[i]
    ub = sb.UniformBalancer(len(g["counts"]))
    got = ub.plan(g["counts"]).download()
    assert got["final_counts"] == g["final_counts"]
    assert [list(m) for m in got["moves"]] == g["moves"]
    assert got["total_moved"] == g["total_moved"]


@pytest.mark.gpu
def test_device_negative_count_is_config_error():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2508_06001_b200 as sb
    ub = sb.UniformBalancer(2)
    with pytest.raises(sb.ConfigError, match="negative count"):
        ub.plan([2, -1]).download()


@pytest.mark.gpu
@pytest.mark.parametrize("i", [j for j, g in enumerate(GOLD) if "error" not in g and g["counts"]][:30])
def test_item_exchange_round_trip(i):
    """Items (3 rows each: 16 B metadata + 256 B payload) land where the
    oracle layout says, and the reverse exchange restores every byte."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2508_06001_b200 as sb
    g = GOLD[i]
    counts, W, rpi, pay = g["counts"], len(g["counts"]), 3, 256
    total_rows = sum(counts) * rpi
    mk = lambda: sb.World(W, 8, [pay], capacity_rows=max(1, total_rows))
    A, B, C = mk(), mk(), mk()
    lens = [[c * rpi] if c else [] for c in counts]
    ids = [[r + 1] if counts[r] else [] for r in range(W)]
    dm = sb.DeviceMeta.from_lists(ids, lens)
    A.layout_origin(dm)
    rng = np.random.default_rng(i)
    content = []
    for r in range(W):
        meta = np.zeros((counts[r] * rpi, 2), np.uint64)
        meta[:, 0] = r
        meta[:, 1] = np.arange(counts[r] * rpi)
        p = rng.integers(0, 256, size=(counts[r] * rpi, pay), dtype=np.uint8)
        A.write_rank(0, r, meta)
        A.write_rank(1, r, p)
        content.append((meta, p))
    ub = sb.UniformBalancer(W).plan(counts)
    ub.route(A, B, rows_per_item=rpi)
    B.status()
    final, moves, _ = oracle.balance_uniform_items(counts)
    lay = oracle.uniform_item_layout(counts, final, moves)
    for d in range(W):
        got = B.read_rank(1, d).reshape(-1, pay)
        assert got.shape[0] == final[d] * rpi
        exp = [content[s][1][k * rpi:(k + 1) * rpi] for s, k in lay[d]]
        exp = np.concatenate(exp) if exp else np.zeros((0, pay), np.uint8)
        assert np.array_equal(got, exp), d
    ub.route(B, C, rows_per_item=rpi, reverse=True)
    C.status()
    for r in range(W):
        assert np.array_equal(C.read_rank(1, r).reshape(-1, pay), content[r][1])
        assert np.array_equal(C.read_rank(0, r).view(np.uint64).reshape(-1, 2), content[r][0])
