"""Device upstream generator and step driver against the unmodified
reference: next_batch per rank (tests/golden/batches.json) bit-exactly, and
the C5 schedule's per-step plans (tests/golden/stream.json: WIR and total
workload bits, chunks, violations) with every simulate_step inline check
holding on the device (simulator.cpp:106-159)."""
import json
import os

import numpy as np
import pytest

from paper_2508_06001_b200.scenarios import C5_SCENARIOS, C5_SEED, C5_TOPOLOGY, C5_WORLD, PRESETS

pytestmark = pytest.mark.gpu
sb = pytest.importorskip("paper_2508_06001_b200")

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "batches.json")) as f:
    BATCHES = json.load(f)
with open(os.path.join(HERE, "golden", "stream.json")) as f:
    STREAM = json.load(f)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def _scenario(case):
    if "codes" in case:
        return sb.Scenario(case["codes"])
    if "preset" in case:
        return sb.Scenario(preset=case["preset"])
    return sb.Scenario(text=case["text"])


def dbits(x):
    return np.float64(x).view(np.uint64).item()


@pytest.mark.parametrize("ci", range(len(BATCHES["cases"])))
def test_device_generator_matches_reference(ci):
    case, gold = BATCHES["inputs"]["cases"][ci], BATCHES["cases"][ci]
    sch = sb.Schedule([_scenario(case)], case["world"], case["seed"])
    for st in gold["steps"]:
        meta = sch.generate(st["step"])
        ids, lens = meta.to_lists()
        for r in range(case["world"]):
            ref = np.asarray(st["ranks"][r], dtype=np.uint64).reshape(-1, 3)
            assert np.array_equal(ids[r], ref[:, 0]), (st["step"], r)
            assert np.array_equal(lens[r], (ref[:, 1] + ref[:, 2]).astype(np.int64)), (st["step"], r)


def test_schedule_cycles_scenarios_and_bounds():
    """Step s uses scenario s mod K; the capacity bounds hold for every step."""
    sch = sb.Schedule([sb.Scenario(c) for c in C5_SCENARIOS], C5_WORLD, C5_SEED)
    for step in range(9):
        ids, lens = sch.generate(step).to_lists()
        codes = C5_SCENARIOS[step % len(C5_SCENARIOS)]
        from paper_2508_06001_b200 import datagen
        for r in range(C5_WORLD):
            i2, l2 = datagen.next_batch(codes, r, step, C5_SEED)
            assert np.array_equal(ids[r], i2) and np.array_equal(lens[r], l2)
        assert sum(len(x) for x in ids) <= sch.max_seqs
        assert sum(int(x.sum()) for x in lens) <= sch.max_rows


def _c5_driver(verify=True, cap=128, width=768):
    sch = sb.Schedule([sb.Scenario(c) for c in C5_SCENARIOS], C5_WORLD, C5_SEED)
    planner = sb.Planner(C5_TOPOLOGY, C5_WORLD, max_seqs=sch.max_seqs)
    return sch, planner, sb.Driver(planner, sch, n_heads=24, payload_row_bytes=width, verify=verify, record_cap=cap)


def test_driver_c5_matches_reference_and_checks_hold():
    """All 1000 steps of the C5 schedule: every step's plan (tokens,
    sequences, chunks, WIR and total-workload bits, violations, max/mean)
    equals the unmodified reference's, and simulate_step's checks hold."""
    n = STREAM["steps"]
    assert n == 1000
    sch, planner, drv = _c5_driver(width=768, cap=n)  # 96 doubles per row keeps the test small
    drv.set_step(0)
    drv.run(n)
    prog = drv.progress()
    assert prog["next_step"] == n and prog["steps_run"] == n and prog["failed"] == 0
    recs = drv.records()
    for g in STREAM["per_step"]:
        r = recs[g["step"]]
        assert r["step"] == g["step"]
        assert r["scenario"] == g["step"] % len(C5_SCENARIOS)
        assert r["tokens"] == g["tokens"] and r["sequences"] == g["sequences"] and r["chunks"] == g["chunks"]
        assert f"{dbits(r['wir']):016x}" == g["wir"], g["step"]
        assert f"{dbits(r['total_workload']):016x}" == g["total_workload"], g["step"]
        assert r["capacity_violations"] == g["violations"]
        assert r["max_over_mean"] == g["max_over_mean"]
        assert r["verified"] == 1 and r["checks"] == 15, (g["step"], r["checks"])


def test_driver_step_graph_replay_advances():
    """One captured step replays with the device step counter advancing."""
    import torch
    sch, planner, drv = _c5_driver(width=192, cap=16)
    drv.set_step(5)
    drv.step()  # eager warm-up allocates every lazily sized buffer outside the capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        drv.step()
    for _ in range(6):
        g.replay()
    torch.cuda.synchronize()
    prog = drv.progress()
    # set_step(5): one eager step (5), the capture records without running, 6 replays (6..11)
    assert prog["failed"] == 0
    recs = {r["step"]: r for r in drv.records() if r["verified"]}
    last = prog["next_step"] - 1
    for s in range(last - 5, last + 1):
        gold = next(x for x in STREAM["per_step"] if x["step"] == s)
        assert f"{dbits(recs[s]['wir']):016x}" == gold["wir"]
        assert recs[s]["checks"] == 15


def test_driver_plan_ahead_matches_serial():
    """The plan-ahead schedule (step s+1 prepared under step s's copies, two
    alternating slots) gives the serial schedule's records, checks and
    worlds; an even-length graph of it replays with the counter advancing."""
    import torch
    n = 12
    sch, planner, ser = _c5_driver(width=192, cap=32)
    ser.set_step(0)
    ser.run(n)
    ser_recs = ser.records()
    ser_sum = ser.world(4).checksum()
    _, planner2, pip = _c5_driver(width=192, cap=32)
    pip.set_pipeline(True)
    pip.set_step(0)
    pip.run(n)
    prog = pip.progress()
    assert prog == {"next_step": n, "steps_run": n, "failed": 0}
    pip_recs = pip.records()
    for s in range(n):
        a, b = ser_recs[s], pip_recs[s]
        assert a == b, s
        assert a["verified"] == 1 and a["checks"] == 15
    assert pip.world(4).checksum() == ser_sum
    # graph of two steps, replayed: steps n .. n+5
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        pip.step()
        pip.step()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    prog = pip.progress()
    assert prog["next_step"] == n + 6 and prog["failed"] == 0
    recs = {r["step"]: r for r in pip.records() if r["verified"]}
    for s in range(n, n + 6):
        gold = next((x for x in STREAM["per_step"] if x["step"] == s), None)
        assert recs[s]["checks"] == 15
        if gold:
            assert f"{dbits(recs[s]['wir']):016x}" == gold["wir"]
    # back to the serial schedule at the device counter
    pip.set_pipeline(False)
    pip.step()
    assert pip.progress()["next_step"] == n + 7
    r = {x["step"]: x for x in pip.records()}[n + 6]
    assert r["checks"] == 15


def test_world_compare_detects_differences():
    """The check primitive the driver relies on: equal worlds compare 0,
    a perturbed copy does not, and perturbing both restores equality."""
    sch = sb.Schedule([sb.Scenario(C5_SCENARIOS[0])], C5_WORLD, C5_SEED)
    meta = sch.generate(3)
    mk = lambda: sb.World(C5_WORLD, 24, [192], capacity_rows=sch.max_rows)
    a, b = mk(), mk()
    for w in (a, b):
        w.layout_origin(meta)
        w.fill_witness(meta)
    assert a.compare(b) == 0
    b.perturb()
    assert a.compare(b) > 0
    a.perturb()
    assert a.compare(b) == 0


def test_fill_meta_equals_witness_metadata():
    """sb_world_fill_meta writes exactly the witness' row metadata."""
    for codes in C5_SCENARIOS:
        sch = sb.Schedule([sb.Scenario(codes)], C5_WORLD, C5_SEED)
        meta = sch.generate(4)
        mk = lambda: sb.World(C5_WORLD, 24, [192], capacity_rows=sch.max_rows)
        a, b = mk(), mk()
        for w in (a, b):
            w.layout_origin(meta)
        a.fill_witness(meta)
        b.fill_meta(meta)
        for r in range(C5_WORLD):
            assert np.array_equal(a.read_rank(0, r), b.read_rank(0, r)), r
