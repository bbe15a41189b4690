"""The plan-ahead schedule of bench.py (batch k+1 planned and its exchanges
prepared on a side stream while batch k's copies run; two planners
alternate) with a DIFFERENT batch every step.

Preparing batch k+1 rewrites the destination worlds' layout tables (base,
pitch, rows per rank) while batch k's copy kernels are still moving rows.
That is only correct because copy jobs carry resolved pointers; these tests
pin it with changing sequence lengths, so batch k+1's layout differs from
batch k's.  Every step's routed image is compared with the oracle's route
(exchange.cpp:127-194) and every round trip (route, pre_attn, post_attn,
reverse_route) must restore the batch's origin world bit-exactly.
"""
import numpy as np
import pytest

import oracle
from paper_2508_06001_b200 import multigpu

pytestmark = pytest.mark.gpu
sb = pytest.importorskip("paper_2508_06001_b200")

W, HEADS, WIDTH = 8, 4, 16  # 16 doubles = 128-B payload rows


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def _batch(k):
    return oracle.meta_c1(W, 3 + (k % 4), seed=11, step=k)


@pytest.mark.parametrize("topo", ["g1n8", "g1n2+g2n1+g4n1", "g2n4"])
def test_plan_ahead_with_changing_batches(topo):
    import torch
    P = sb.Planner
    n_steps = 8
    metas = [_batch(k) for k in range(n_steps)]
    rows = max(int(sum(int(x.sum()) for x in m.lens)) for m in metas)
    dms = [sb.DeviceMeta.from_lists(m.ids, m.lens) for m in metas]
    planners = [P(topo, W, max_seqs=64), P(topo, W, max_seqs=64)]
    G = planners[0].max_bag
    mk = lambda: sb.World(W, HEADS, [WIDTH * 8], capacity_rows=rows, aux_row_bytes=[16], max_bag=G)
    A = [mk(), mk()]   # origin images: batch k lives in A[k % 2]
    E = [mk(), mk()]   # restored images
    B, Cw, D = mk(), mk(), mk()  # shared by every batch

    def ops(k):
        a, e = A[k % 2], E[k % 2]
        if G > 1:
            return [(P.ROUTE, a, B, 0), (P.PRE_ATTN, B, Cw, 2), (P.POST_ATTN, Cw, D, 3), (P.REVERSE, D, e, 1)]
        return [(P.ROUTE, a, B, 0), (P.REVERSE, B, e, 1)]

    main = torch.cuda.current_stream()
    side = torch.cuda.Stream()

    def plan_and_prepare(k, evl):
        """On the side stream: the batch's origin world, its plan, and every
        exchange's destination layout + copy jobs."""
        pl = planners[k % 2]
        a = A[k % 2]
        a.layout_origin(dms[k], side)
        a.fill_witness(dms[k], side)
        pl.plan(dms[k], side)
        for i, (op, src, dst, slot) in enumerate(ops(k)):
            pl.prepare(op, src, dst, slot, side)
            evl[i].record(side)

    def snap(w, t):  # async copy of a tensor's packed arena on the main stream
        base, nbytes = w.arena(t)
        return multigpu.device_bytes(base, nbytes).clone()

    evs = [[torch.cuda.Event() for _ in range(4)] for _ in range(2)]
    free = [torch.cuda.Event(), torch.cuda.Event()]
    routed, restored = [], []
    side.wait_stream(main)
    with torch.cuda.stream(side):
        plan_and_prepare(0, evs[0])
    for k in range(n_steps):  # no host synchronisation inside the schedule
        if k + 1 < n_steps:
            # batch k+1 uses the other planner / origin world: wait until the
            # step that last used them (k-1) has finished its copies
            if k >= 1:
                side.wait_event(free[(k + 1) % 2])
            with torch.cuda.stream(side):
                plan_and_prepare(k + 1, evs[(k + 1) % 2])
        for i, (op, src, dst, slot) in enumerate(ops(k)):
            main.wait_event(evs[k % 2][i])
            planners[k % 2].run(slot)
            if op == P.ROUTE:
                routed.append(snap(B, 1))
        restored.append((snap(E[k % 2], 0), snap(E[k % 2], 1)))
        free[k % 2].record(main)
    torch.cuda.synchronize()
    for w in A + E + [B, Cw, D]:
        w.status()
    for k in range(n_steps):
        plan, _ = oracle.plan_routing(metas[k], oracle.parse_topology(topo))
        w0 = oracle.make_world(metas[k], WIDTH, HEADS)
        want = np.concatenate([r.payload.reshape(-1) for r in oracle.route(w0, plan).ranks])
        got = routed[k].cpu().numpy()[:want.size]
        assert np.array_equal(got, want), f"step {k}: routed payload differs from the oracle"
        home = np.concatenate([r.payload.reshape(-1) for r in w0.ranks])
        assert np.array_equal(restored[k][1].cpu().numpy()[:home.size], home), f"step {k}: round trip payload"
        ids = np.concatenate([r.ids for r in w0.ranks])
        meta = restored[k][0].cpu().numpy()[:16 * ids.size].view(np.uint64).reshape(-1, 2)
        assert np.array_equal(meta[:, 0], ids), f"step {k}: round trip ids"


def test_plan_ahead_layouts_really_change():
    """The batches above are not all the same shape (else the test would not
    exercise a layout rewrite under running copies)."""
    shapes = {tuple(int(x.sum()) for x in _batch(k).lens) for k in range(8)}
    assert len(shapes) >= 4
