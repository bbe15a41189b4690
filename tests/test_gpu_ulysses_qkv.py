"""Ulysses on q, k, v (out) and o (back): the DiT attention pattern the
reference's comm model assumes -- "outbound phase carries q, k and v (3x token
bytes) and the return phase ... (1x)" (metrics.cpp:85-121) -- on the device
exchange engine, checked byte for byte against the oracle's pre_attn /
post_attn (exchange.cpp:255-436) applied to each tensor separately.

q, k, v and o carry distinct payloads (per-byte transforms of the witness, so
every tensor is a different byte image) and a whole-row aux tensor (RoPE ids
derived from (sample_id, position)) that must travel with its rows: routed
with the chunk, replicated to every bag member by pre_attn and taken from
member 0 by post_attn."""
import copy

import numpy as np
import pytest

import oracle
from paper_2508_06001_b200 import multigpu

pytestmark = pytest.mark.gpu

sb = pytest.importorskip("paper_2508_06001_b200")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


HEADS = 24


def tensor_image(payload: np.ndarray, k: int) -> np.ndarray:
    """Byte image of tensor k (0 = o, 1..3 = q, k, v): a per-byte transform of
    the witness payload, so it commutes with any row / column movement."""
    return ((payload.astype(np.uint16) + 37 * (k + 1)) % 256).astype(np.uint8)


def aux_rows(ids: np.ndarray, pos: np.ndarray) -> np.ndarray:
    """RoPE-like aux row of (id, pos): 16 bytes, a pure function of the row's
    metadata, so its expected value in any layout follows from the metadata."""
    a = np.empty((len(ids), 2), np.uint64)
    a[:, 0] = np.asarray(ids, np.uint64) ^ np.uint64(0x9E3779B97F4A7C15)
    a[:, 1] = np.asarray(pos, np.uint64) * np.uint64(3) + np.uint64(1)
    return a


def meta_rows(ids, pos):
    m = np.empty((len(ids), 2), np.uint64)
    m[:, 0] = ids
    m[:, 1] = np.asarray(pos, np.int64).view(np.uint64)
    return m


def read_meta(world, r):
    m = world.read_rank(0, r).view(np.uint64).reshape(-1, 2)
    return m[:, 0], m[:, 1].view(np.int64)


def ulysses_expected(routed: oracle.World, topo: oracle.Topology, W: int) -> oracle.World:
    want = copy.deepcopy(routed)
    U = topo.unit_size
    for rep in range(W // U):
        for b, g in enumerate(topo.bag_sizes):
            if g > 1:
                oracle.pre_attn(want, [rep * U + x for x in topo.bag_ranks(b)])
    return want


@pytest.mark.parametrize("world,topo,per_rank", [(8, "g4n2", 3), (8, "g8n1", 2), (8, "g1n2+g2n1+g4n1", 4),
                                                 (16, "g2n4", 2), (8, "g1n8", 3)])
def test_qkv_out_o_back_vs_oracle(world, topo, per_rank):
    W = world
    width = HEADS * 4  # doubles per row: 768 B, head slices of 32 B .. 96 B (16-B aligned)
    rb = width * 8
    meta = oracle.meta_c1(W, per_rank, seed=11, step=0)
    tp = oracle.parse_topology(topo)
    plan, _ = oracle.plan_routing(meta, tp)
    w0 = oracle.make_world(meta, width, HEADS)
    routed = oracle.route(w0, plan)
    want = ulysses_expected(routed, tp, W)

    dm = sb.DeviceMeta.from_lists(meta.ids, meta.lens)
    planner = sb.Planner(topo, W, max_seqs=sum(len(x) for x in meta.ids))
    planner.plan(dm)
    G = planner.max_bag
    rows = int(sum(int(x.sum()) for x in meta.lens))

    # x (hidden states) with RoPE aux: route -- aux rows travel with their row
    X = sb.World(W, HEADS, [rb], capacity_rows=rows, aux_row_bytes=[16], max_bag=G)
    XB = sb.World(W, HEADS, [rb], capacity_rows=rows, aux_row_bytes=[16], max_bag=G)
    X.layout_origin(dm)
    X.fill_witness(dm)
    for r in range(W):
        X.write_rank(2, r, aux_rows(w0.ranks[r].ids, w0.ranks[r].pos))
    sb.route(planner, X, XB)
    XB.status()
    for r in range(W):
        ids, pos = read_meta(XB, r)
        assert np.array_equal(ids, routed.ranks[r].ids) and np.array_equal(pos, routed.ranks[r].pos)
        assert np.array_equal(XB.read_rank(1, r), routed.ranks[r].payload.reshape(-1)), f"x rank {r}"
        assert np.array_equal(XB.read_rank(2, r).view(np.uint64).reshape(-1, 2), aux_rows(ids, pos)), f"aux {r}"

    # q, k, v written in the chunk layout (as a projection of XB would), then
    # one pre_attn moves all three plus metadata and aux
    QKV = sb.World(W, HEADS, [rb] * 3, capacity_rows=rows, aux_row_bytes=[16], max_bag=G)
    QKVu = sb.World(W, HEADS, [rb] * 3, capacity_rows=rows, aux_row_bytes=[16], max_bag=G)
    QKV.layout_plan(planner, sb.World.TARGET)
    for r in range(W):
        rr = routed.ranks[r]
        QKV.write_rank(0, r, meta_rows(rr.ids, rr.pos))
        for t in range(3):
            QKV.write_rank(1 + t, r, tensor_image(rr.payload, 1 + t))
        QKV.write_rank(4, r, aux_rows(rr.ids, rr.pos))
    sb.pre_attn(planner, QKV, QKVu)
    QKVu.status()
    for r in range(W):
        wr = want.ranks[r]
        ids, pos = read_meta(QKVu, r)
        assert np.array_equal(ids, wr.ids) and np.array_equal(pos, wr.pos), f"pre_attn metadata rank {r}"
        for t in range(3):
            got = QKVu.read_rank(1 + t, r)
            assert np.array_equal(got, tensor_image(wr.payload, 1 + t).reshape(-1)), f"pre_attn tensor {t} rank {r}"
        assert np.array_equal(QKVu.read_rank(4, r).view(np.uint64).reshape(-1, 2), aux_rows(ids, pos)), \
            f"pre_attn aux rank {r}"

    # o produced by attention in the Ulysses layout; post_attn brings it back
    # to the chunk layout, reverse_route home
    O = sb.World(W, HEADS, [rb], capacity_rows=rows, max_bag=G)
    Oc = sb.World(W, HEADS, [rb], capacity_rows=rows, max_bag=G)
    E = sb.World(W, HEADS, [rb], capacity_rows=rows, max_bag=G)
    O.layout_plan(planner, sb.World.ULYSSES)
    for r in range(W):
        wr = want.ranks[r]
        O.write_rank(0, r, meta_rows(wr.ids, wr.pos))
        O.write_rank(1, r, tensor_image(wr.payload, 0))
    sb.post_attn(planner, O, Oc)
    Oc.status()
    for r in range(W):
        rr = routed.ranks[r]
        ids, pos = read_meta(Oc, r)
        assert np.array_equal(ids, rr.ids) and np.array_equal(pos, rr.pos), f"post_attn metadata rank {r}"
        assert np.array_equal(Oc.read_rank(1, r), tensor_image(rr.payload, 0).reshape(-1)), f"post_attn rank {r}"
    sb.reverse_route(planner, Oc, E)
    E.status()
    for r in range(W):
        o = w0.ranks[r]
        ids, pos = read_meta(E, r)
        assert np.array_equal(ids, o.ids) and np.array_equal(pos, o.pos)
        assert np.array_equal(E.read_rank(1, r), tensor_image(o.payload, 0).reshape(-1)), f"o home rank {r}"


def test_layout_plan_matches_exchange_layouts():
    """sb_world_layout_plan(TARGET / ULYSSES / ORIGIN) gives the per-rank rows
    and pitches the exchanges themselves produce."""
    W, topo = 8, "g1n2+g2n1+g4n1"
    meta = oracle.meta_c1(W, 3, seed=2, step=0)
    dm = sb.DeviceMeta.from_lists(meta.ids, meta.lens)
    planner = sb.Planner(topo, W, max_seqs=24)
    planner.plan(dm)
    rows = int(sum(int(x.sum()) for x in meta.lens))
    mk = lambda: sb.World(W, HEADS, [192, 384], capacity_rows=rows, aux_row_bytes=[16], max_bag=4)
    A, B, C, L = mk(), mk(), mk(), mk()
    A.layout_origin(dm)
    for t in range(A.T):  # defined bytes (compute-sanitizer initcheck), though only layouts are checked
        multigpu.device_bytes(*A.arena(t)).zero_()
    sb.route(planner, A, B)
    sb.pre_attn(planner, B, C)
    for which, ref in ((sb.World.TARGET, B), (sb.World.ULYSSES, C), (sb.World.ORIGIN, A)):
        L.layout_plan(planner, which)
        for t in range(4):
            r1, p1 = L.shape(t)
            r2, p2 = ref.shape(t)
            assert np.array_equal(r1, r2) and np.array_equal(p1, p2), (which, t)
