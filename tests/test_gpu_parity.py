"""Parity of the CUDA path (libseqbal_cuda.so through the C-ABI) against the
reference fixtures (tests/golden/cases.json, produced by the unmodified
reference) and the CPU oracle.  Integer/byte work: bit-exact everywhere;
the FP64 BalanceReport is compared bit for bit as well."""
import numpy as np
import pytest

import oracle
from golden_util import case_by_name, check_plan, check_report, dbits, hexd, load_cases, meta_for, model_for

pytestmark = pytest.mark.gpu

sb = pytest.importorskip("paper_2508_06001_b200")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def device_meta(meta: oracle.Meta):
    return sb.DeviceMeta.from_lists(meta.ids, meta.lens)


def host_plan_as_oracle(hp, meta: oracle.Meta) -> oracle.Plan:
    """Reassemble a device plan into the oracle's Plan record for comparison."""
    W = hp.world
    recv = hp.recv
    target = [[(int(hp.c_id[c]), int(hp.c_start[c]), int(hp.c_end[c] - hp.c_start[c])) for c in recv[r]]
              for r in range(W)]
    origin = [[(int(i), 0, int(l)) for i, l in zip(meta.ids[r], meta.lens[r])] for r in range(W)]
    return oracle.Plan(W, hp.c_id, hp.c_idx, hp.c_start, hp.c_end, hp.c_src, hp.c_dst, hp.send, recv,
                       origin, target)


def reverse_as_oracle(hp, fwd: oracle.Plan) -> oracle.Plan:
    return oracle.Plan(hp.world, hp.c_id, hp.c_idx, hp.c_start, hp.c_end, hp.c_dst, hp.c_src, hp.rev_send,
                       hp.rev_recv, origin=fwd.target, target=fwd.origin)


def report_as_oracle(hp) -> oracle.Report:
    return oracle.Report(hp.per_gpu_workload, hp.per_bag_occupancy, hp.capacity_violations, hp.total_workload,
                         hp.wir)


def rank_digests(world, r):
    meta = world.read_rank(0, r).view(np.uint64).reshape(-1, 2)
    ids = np.ascontiguousarray(meta[:, 0])
    pos = np.ascontiguousarray(meta[:, 1])
    pay = world.read_rank(1, r)
    return len(ids), hexd(oracle.digest(ids)), hexd(oracle.digest(pos)), hexd(oracle.digest(pay)), pay.nbytes


def check_dev_world(world, ref, ranks=None):
    for r, rr in enumerate(ref["ranks"]):
        if ranks is not None and r not in ranks:
            continue
        rows, di, dp, dpl, nbytes = rank_digests(world, r)
        assert rows == rr["rows"], f"rank {r} rows"
        assert di == rr["ids_digest"], f"rank {r} ids"
        assert dp == rr["pos_digest"], f"rank {r} positions"
        assert dpl == rr["payload_digest"], f"rank {r} payload"
        if rows:
            assert nbytes // rows == rr["width"] * 8, f"rank {r} width"


def planner_paths_equal(a, b):
    for k in ("c_id", "c_idx", "c_start", "c_end", "c_src", "c_dst", "send_off", "send_idx", "recv_off", "recv_idx",
              "rev_recv_idx", "target_rows"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    for k in ("per_gpu_workload", "per_bag_occupancy"):
        assert np.array_equal(getattr(a, k).view(np.uint64), getattr(b, k).view(np.uint64)), k
    assert a.capacity_violations == b.capacity_violations
    assert dbits(a.total_workload) == dbits(b.total_workload) and dbits(a.wir) == dbits(b.wir)


def make_planner(case, meta):
    d, h, g = model_for(case)
    md = case["model"]
    model = sb.Model(d_model=d, n_heads=h, d_head=md["d_head"], n_blocks=md["n_blocks"], gamma=g)
    return sb.Planner(case["topology"], case["world"], model, max_seqs=max(1, sum(len(x) for x in meta.ids)))


CASES = [c["name"] for c in load_cases()]


@pytest.mark.parametrize("name", CASES)
def test_device_plan_and_exchange_match_reference(name):
    c = case_by_name(name)
    case, ref = c["case"], c["result"]
    meta = oracle_meta = meta_for(case)
    if "error" in ref:
        with pytest.raises(sb.ConfigError):
            make_planner(case, meta)
        return
    planner = make_planner(case, meta)
    dm = device_meta(meta)
    planner.plan(dm)
    hp = planner.download()
    fwd = host_plan_as_oracle(hp, meta)
    check_plan(fwd, ref["plan"])
    check_report(report_as_oracle(hp), ref["report"])
    check_plan(reverse_as_oracle(hp, fwd), ref["reverse"])  # libstdc++ tie order replayed

    # the other planner pipelines (fused single-CTA, hybrid, multi-kernel) must agree bit for bit
    n_seqs = sum(len(x) for x in meta.ids)
    for path in (["large", "small", "hybrid"] if n_seqs <= 2048 else []):
        other = make_planner(case, meta)
        other.set_path(path)
        planner_paths_equal(hp, other.plan(dm).download())
        if len(other.topology.bag_sizes) <= 64:
            assert other.last_path() == path

    # identity_plan on the same planner slots
    planner.plan_identity(dm)
    ident = planner.download()
    check_plan(host_plan_as_oracle(ident, meta), ref["identity"])
    planner.plan(dm)

    if not case.get("route"):
        return
    W, width = case["world"], case["payload_width"]
    _, h, _ = model_for(case)
    rows = max(1, int(sum(int(x.sum()) for x in meta.lens)))
    mk = lambda: sb.World(W, h, [width * 8], capacity_rows=rows, max_bag=planner.max_bag)
    A, B, Cw, D, E = mk(), mk(), mk(), mk(), mk()
    A.layout_origin(dm)
    A.fill_witness(dm)
    check_dev_world(A, ref["world0"])
    assert hexd(A.checksum()) == ref["world0"]["checksum"]
    sb.route(planner, A, B)
    B.status()
    check_dev_world(B, ref["routed"])
    assert hexd(B.checksum()) == ref["routed"]["checksum"]
    if ref.get("ulysses"):
        sb.pre_attn(planner, B, Cw)
        Cw.status()
        topo = oracle.parse_topology(case["topology"])
        for u in ref["ulysses"]:
            bag = [x + u["replica"] * topo.unit_size for x in topo.bag_ranks(u["bag"])]
            check_dev_world(Cw, u["pre"], ranks=set(bag))
        assert hexd(Cw.checksum()) == ref["routed"]["checksum"]
        sb.post_attn(planner, Cw, D)
        D.status()
        for r in range(W):
            assert rank_digests(D, r) == rank_digests(B, r), f"post(pre(x)) != x on rank {r}"
    B.perturb()
    check_dev_world(B, ref["mutated"])
    sb.reverse_route(planner, B, E)
    E.status()
    check_dev_world(E, ref["returned"])


@pytest.mark.parametrize("path", ["small", "large", "hybrid"])
@pytest.mark.parametrize("topo", ["g8n1", "g4n2", "g2n1+g1n2+g4n1"])
def test_reverse_ties_match_std_sort(topo, path):
    """Sequences shorter than their bag make reverse_plan's sort keys tie; the
    device must reproduce libstdc++ std::sort's tie order (the oracle calls
    the real std::sort)."""
    rng = np.random.default_rng(7 + len(topo))
    planner = sb.Planner(topo, 8, max_seqs=2048)
    planner.set_path(path)
    for trial in range(10):
        lens = [rng.integers(0, 12, size=rng.integers(3, 40)).tolist() for _ in range(8)]
        meta = oracle.meta_explicit(lens)
        planner.plan(device_meta(meta))
        hp = planner.download()
        plan, _ = oracle.plan_routing(meta, oracle.parse_topology(topo))
        assert hp.rev_recv == oracle.reverse_plan(plan).recv, f"trial {trial}"


def test_fast_division_matches_ddiv_rn():
    """The greedy's Markstein division must round exactly like __ddiv_rn."""
    import ctypes as C
    from paper_2508_06001_b200 import _capi
    bad = C.c_int64(-1)
    _capi.call("sb_selftest_div", 1 << 27, 0x5EED, C.byref(bad))
    assert bad.value == 0


@pytest.mark.parametrize("mode", range(7))
def test_block_serial_sum_bit_exact(mode):
    """serial_sum.cuh: block-parallel serial FP64 sums (totals, one-bag
    occupancy replay) equal the one-thread DADD chain bit for bit -- result
    and every prefix -- on laws with frequent round-half-even ties, zeros,
    wide exponent ranges and overflow; 148 sums of up to 40 000 values."""
    import ctypes as C
    from paper_2508_06001_b200 import _capi
    bad = C.c_int64(-1)
    _capi.call("sb_selftest_serial_sum", 148, 40000, 0x5EED + mode, mode, C.byref(bad))
    assert bad.value == 0


def test_duplicate_ids_rejected():
    meta = oracle.meta_explicit([[10, 20], [30]], ids=[[5, 6], [5]])
    planner = sb.Planner("g1n2", 2, max_seqs=8)
    planner.plan(device_meta(meta))
    with pytest.raises(sb.ConfigError):
        planner.sizes()


def test_negative_length_rejected():
    meta = oracle.meta_explicit([[10, -1], [30]])
    planner = sb.Planner("g1n2", 2, max_seqs=8)
    planner.plan(device_meta(meta))
    with pytest.raises(sb.ConfigError):
        planner.sizes()


def test_capacity_exceeded_is_loud():
    meta = oracle.meta_explicit([[1, 2, 3], [4, 5]])
    planner = sb.Planner("g1n2", 2, max_seqs=4)
    planner.plan(device_meta(meta))
    with pytest.raises(sb.CapacityError):
        planner.sizes()


@pytest.mark.parametrize("path", ["small", "large", "hybrid"])
@pytest.mark.parametrize("topo", ["g1n8", "g2n4", "g4n2", "g8n1", "g1n2+g2n1+g4n1"])
def test_random_plans_vs_oracle(topo, path):
    rng = np.random.default_rng(sum(map(ord, topo)))
    planner = sb.Planner(topo, 16 if "+" in topo else 8, max_seqs=2048)
    planner.set_path(path)
    W = planner.world_size
    for trial in range(20):
        lens = [rng.integers(0, 5000, size=rng.integers(0, 40)).tolist() for _ in range(W)]
        meta = oracle.meta_explicit(lens)
        planner.plan(device_meta(meta))
        hp = planner.download()
        plan, rep = oracle.plan_routing(meta, oracle.parse_topology(topo))
        got = host_plan_as_oracle(hp, meta)
        assert got.chunk_rows() == plan.chunk_rows()
        assert got.send == plan.send and got.recv == plan.recv
        assert [dbits(x) for x in hp.per_gpu_workload] == [dbits(x) for x in rep.per_gpu_workload]
        assert [dbits(x) for x in hp.per_bag_occupancy] == [dbits(x) for x in rep.per_bag_occupancy]
        assert hp.capacity_violations == rep.capacity_violations
        assert dbits(hp.total_workload) == dbits(rep.total_workload)
        assert dbits(hp.wir) == dbits(rep.wir)
        rev = oracle.reverse_plan(plan)
        assert hp.rev_recv == rev.recv


@pytest.mark.parametrize("topo", ["g1n8", "g2n4"])
def test_large_path_reused_planner_shrinking_batches(topo):
    """One planner, multi-kernel path, a batch whose busiest bag receives more
    than one list tile (kListTile = 1024 sequences) followed by smaller
    batches: per-tile sums of tiles that are empty in the later plans must
    not leak into target_rows / the Ulysses bases (compute-sanitizer
    initcheck found k_lists reading never-written tiles)."""
    W = 8
    planner = sb.Planner(topo, W, max_seqs=W * 1400)
    planner.set_path("large")
    rng = np.random.default_rng(5)
    for per_rank in (1400, 37, 700, 3):
        lens = [rng.integers(1, 3000, size=per_rank).tolist() for _ in range(W)]
        meta = oracle.meta_explicit(lens)
        planner.plan(device_meta(meta))
        hp = planner.download()
        plan, rep = oracle.plan_routing(meta, oracle.parse_topology(topo))
        got = host_plan_as_oracle(hp, meta)
        assert got.chunk_rows() == plan.chunk_rows()
        assert got.send == plan.send and got.recv == plan.recv
        want_rows = [sum(sg[2] for sg in plan.target[r]) for r in range(W)]
        assert hp.target_rows.tolist() == want_rows, per_rank
        assert hp.rev_recv == oracle.reverse_plan(plan).recv


@pytest.mark.parametrize("topo", ["g8n1", "g2n4", "g4n1+g2n1+g1n2"])
def test_plans_beyond_shared_staging_vs_oracle(topo):
    """More sequences than the serial-sum kernels stage in shared memory
    (kSumStage = 24 576): the large path's totals and one-bag occupancy replay
    read global memory; zero lengths and repeated lengths (exact workload
    ties) included.  Report bit-exact against the oracle."""
    rng = np.random.default_rng(29)
    W = 8
    lens = []
    for r in range(W):
        x = rng.integers(0, 4096, size=3300)
        x[rng.random(3300) < 0.05] = 0
        lens.append(x.tolist())
    meta = oracle.meta_explicit(lens)
    planner = sb.Planner(topo, W, max_seqs=W * 3300)
    planner.plan(device_meta(meta))
    hp = planner.download()
    plan, rep = oracle.plan_routing(meta, oracle.parse_topology(topo))
    got = host_plan_as_oracle(hp, meta)
    assert got.chunk_rows() == plan.chunk_rows()
    assert got.send == plan.send and got.recv == plan.recv
    assert [dbits(x) for x in hp.per_gpu_workload] == [dbits(x) for x in rep.per_gpu_workload]
    assert [dbits(x) for x in hp.per_bag_occupancy] == [dbits(x) for x in rep.per_bag_occupancy]
    assert hp.capacity_violations == rep.capacity_violations
    assert dbits(hp.total_workload) == dbits(rep.total_workload)
    assert dbits(hp.wir) == dbits(rep.wir)


def test_download_into_pinned_buffers_matches():
    """Planner.download(out=host_buffers()) -- page-locked caller buffers,
    reused across plans -- returns the same plan as a fresh download."""
    rng = np.random.default_rng(5)
    planner = sb.Planner("g2n4", 8, max_seqs=512)
    host = planner.host_buffers(pinned=True)
    for trial in range(3):
        lens = [rng.integers(0, 3000, size=rng.integers(1, 60)).tolist() for _ in range(8)]
        meta = oracle.meta_explicit(lens)
        planner.plan(device_meta(meta))
        a, b = planner.download(), planner.download(out=host)
        for f in ("c_id", "c_idx", "c_start", "c_end", "c_src", "c_dst", "send_off", "send_idx", "recv_off",
                  "recv_idx", "rev_recv_idx", "target_rows", "per_gpu_workload", "per_bag_occupancy"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), f
        assert (a.capacity_violations, dbits(a.total_workload), dbits(a.wir)) == \
            (b.capacity_violations, dbits(b.total_workload), dbits(b.wir))


def test_full_width_c1_roundtrip_bit_exact():
    """C1 at the bench width (768 doubles == 3072 bf16 == 6144 B/row)."""
    meta = oracle.meta_c1(8, 32, seed=1, step=0)
    planner = sb.Planner("g2n4", 8, max_seqs=256)
    dm = device_meta(meta)
    planner.plan(dm)
    rows = int(sum(int(x.sum()) for x in meta.lens))
    mk = lambda: sb.World(8, 24, [6144], capacity_rows=rows, max_bag=2)
    A, B, Cw, D, E = mk(), mk(), mk(), mk(), mk()
    A.layout_origin(dm)
    A.fill_witness(dm)
    cs = A.checksum()
    sb.route(planner, A, B)
    sb.pre_attn(planner, B, Cw)
    sb.post_attn(planner, Cw, D)
    sb.reverse_route(planner, D, E)
    E.status()
    assert B.checksum() == cs and Cw.checksum() == cs
    for r in range(8):
        assert rank_digests(E, r) == rank_digests(A, r)
        assert rank_digests(D, r) == rank_digests(B, r)
    # routed bytes equal the oracle's route of the same world
    plan, _ = oracle.plan_routing(meta, oracle.parse_topology("g2n4"))
    w0 = oracle.make_world(meta, 768, 24)
    routed = oracle.route(w0, plan)
    for r in range(8):
        rows_r, di, dp, dpl, _ = rank_digests(B, r)
        ob = routed.ranks[r]
        assert rows_r == ob.rows
        assert dpl == hexd(oracle.digest(np.ascontiguousarray(ob.payload)))
        assert di == hexd(oracle.digest(ob.ids)) and dp == hexd(oracle.digest(ob.pos))


def test_world_plan_mismatch_is_integrity_error():
    """check_world_matches_layout (exchange.cpp:96-123): exchanging from a world
    whose layout is not the plan's raises IntegrityError and copies nothing;
    the next valid exchange into the same destination succeeds."""
    meta = oracle.meta_c1(8, 4, seed=3, step=0)
    dm = device_meta(meta)
    planner = sb.Planner("g1n8", 8, max_seqs=32)
    planner.plan(dm)
    rows = int(sum(int(x.sum()) for x in meta.lens))
    mk = lambda: sb.World(8, 24, [192], capacity_rows=rows)
    A, B, stale, E = mk(), mk(), mk(), mk()
    A.layout_origin(dm)
    A.fill_witness(dm)
    sb.reverse_route(planner, stale, E)  # stale was never routed: zero rows per rank
    with pytest.raises(sb.IntegrityError):
        E.status()
    sb.route(planner, A, stale)          # route expects the origin layout: A has it
    stale.status()
    with pytest.raises(sb.IntegrityError):
        sb.route(planner, stale, B)      # stale now holds the target layout, not the origin
        B.status()
    sb.reverse_route(planner, stale, E)
    E.status()
    for r in range(8):
        assert np.array_equal(E.read_rank(1, r), A.read_rank(1, r))


@pytest.mark.parametrize("path", ["small", "large", "hybrid"])
@pytest.mark.parametrize("world,topo", [(64, "g2n4"), (256, "g4n2+g8n1"), (96, "g1n4+g2n2+g4n1")])
def test_many_replicas_vs_oracle(world, topo, path):
    """Large worlds: many replicas planned independently (balancer.cpp:136-219),
    ragged ranks including empty ones and zero-length sequences."""
    rng = np.random.default_rng(world)
    lens = [rng.integers(0, 3000, size=rng.integers(0, 6)).tolist() for _ in range(world)]
    meta = oracle.meta_explicit(lens)
    planner = sb.Planner(topo, world, max_seqs=max(1, sum(len(x) for x in lens)))
    planner.set_path(path)
    planner.plan(device_meta(meta))
    hp = planner.download()
    plan, rep = oracle.plan_routing(meta, oracle.parse_topology(topo))
    got = host_plan_as_oracle(hp, meta)
    assert got.chunk_rows() == plan.chunk_rows()
    assert got.send == plan.send and got.recv == plan.recv
    assert [dbits(x) for x in hp.per_gpu_workload] == [dbits(x) for x in rep.per_gpu_workload]
    assert [dbits(x) for x in hp.per_bag_occupancy] == [dbits(x) for x in rep.per_bag_occupancy]
    assert dbits(hp.wir) == dbits(rep.wir) and dbits(hp.total_workload) == dbits(rep.total_workload)
    assert hp.rev_recv == oracle.reverse_plan(plan).recv
    # and the data path on the same plan
    rows = int(sum(sum(x) for x in lens))
    mk = lambda: sb.World(world, 24, [192], capacity_rows=max(1, rows), max_bag=planner.max_bag)
    A, B, Cw, D, E = mk(), mk(), mk(), mk(), mk()
    dm = device_meta(meta)
    A.layout_origin(dm)
    A.fill_witness(dm)
    sb.route(planner, A, B)
    sb.pre_attn(planner, B, Cw)
    sb.post_attn(planner, Cw, D)
    sb.reverse_route(planner, D, E)
    E.status()
    assert E.compare(A) == 0 and D.compare(B) == 0
    assert Cw.checksum() == A.checksum()


@pytest.mark.parametrize("world,topo", [(96, "g1n96"), (96, "g1n64+g2n16"), (400, "g2n200"), (130, "g1n65")])
def test_many_bags_vs_oracle(world, topo):
    """More than 64 bags per replica (multi-kernel path, k_greedy_many and the
    emission tables in dynamic shared memory): plan, report and data path equal
    the reference's; the reference has no bag limit, the device path 1024."""
    rng = np.random.default_rng(len(topo) + world)
    lens = [rng.integers(0, 4000, size=rng.integers(0, 9)).tolist() for _ in range(world)]
    meta = oracle.meta_explicit(lens)
    planner = sb.Planner(topo, world, max_seqs=max(1, sum(len(x) for x in lens)))
    planner.plan(device_meta(meta))
    hp = planner.download()
    plan, rep = oracle.plan_routing(meta, oracle.parse_topology(topo))
    got = host_plan_as_oracle(hp, meta)
    assert got.chunk_rows() == plan.chunk_rows()
    assert got.send == plan.send and got.recv == plan.recv
    assert [dbits(x) for x in hp.per_gpu_workload] == [dbits(x) for x in rep.per_gpu_workload]
    assert [dbits(x) for x in hp.per_bag_occupancy] == [dbits(x) for x in rep.per_bag_occupancy]
    assert dbits(hp.wir) == dbits(rep.wir) and dbits(hp.total_workload) == dbits(rep.total_workload)
    assert hp.capacity_violations == rep.capacity_violations
    assert hp.rev_recv == oracle.reverse_plan(plan).recv
    rows = int(sum(sum(x) for x in lens))
    mk = lambda: sb.World(world, 24, [192], capacity_rows=max(1, rows), max_bag=planner.max_bag)
    A, B, Cw, D, E = mk(), mk(), mk(), mk(), mk()
    dm = device_meta(meta)
    A.layout_origin(dm)
    A.fill_witness(dm)
    sb.route(planner, A, B)
    sb.pre_attn(planner, B, Cw)
    sb.post_attn(planner, Cw, D)
    sb.reverse_route(planner, D, E)
    E.status()
    assert E.compare(A) == 0 and D.compare(B) == 0


def test_bag_limit_is_config_error():
    with pytest.raises(sb.ConfigError, match="more than 1024 bags per replica"):
        sb.Planner("g1n1025", 1025, max_seqs=8)


@pytest.mark.parametrize("path", ["small", "large", "hybrid"])
def test_empty_replicas_vs_oracle(path):
    """Whole replicas without sequences (first and last of three): chunk bases,
    manifests and the data path skip them exactly like the reference."""
    rng = np.random.default_rng(5)
    world = 24  # g2n4: three replicas of eight ranks
    lens = [[] for _ in range(8)] + [rng.integers(0, 2000, size=3).tolist() for _ in range(8)] + [[] for _ in range(8)]
    meta = oracle.meta_explicit(lens)
    planner = sb.Planner("g2n4", world, max_seqs=sum(len(x) for x in lens))
    planner.set_path(path)
    planner.plan(device_meta(meta))
    hp = planner.download()
    plan, rep = oracle.plan_routing(meta, oracle.parse_topology("g2n4"))
    got = host_plan_as_oracle(hp, meta)
    assert got.chunk_rows() == plan.chunk_rows()
    assert got.send == plan.send and got.recv == plan.recv
    assert [dbits(x) for x in hp.per_gpu_workload] == [dbits(x) for x in rep.per_gpu_workload]
    assert hp.rev_recv == oracle.reverse_plan(plan).recv
    rows = int(sum(sum(x) for x in lens))
    mk = lambda: sb.World(world, 24, [192], capacity_rows=max(1, rows), max_bag=planner.max_bag)
    A, B, Cw, D, E = mk(), mk(), mk(), mk(), mk()
    dm = device_meta(meta)
    A.layout_origin(dm)
    A.fill_witness(dm)
    sb.route(planner, A, B)
    sb.pre_attn(planner, B, Cw)
    sb.post_attn(planner, Cw, D)
    sb.reverse_route(planner, D, E)
    E.status()
    assert E.compare(A) == 0 and D.compare(B) == 0
