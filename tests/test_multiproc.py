"""Multi-process (one process per GPU) path.

CPU (gloo, world_size 2): the sharding and ownership logic of
paper_2508_06001_b200.multigpu driven as a real 2-process exchange in which
every process pushes the chunks whose source rank it hosts to the owner of the
target rank -- the same decomposition the device kernels use -- checked
against the oracle's single-process route.

GPU (@gpu): two processes on ONE device share their arenas through CUDA IPC
and run the real peer-store path (metadata all-gather, identical planning,
route, Ulysses, reverse) -- the multi-GPU code with the NVLink hop replaced by
same-device IPC mappings.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from paper_2508_06001_b200 import api, multigpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_partition_owner_and_bytes():
    assert multigpu.partition(8, 2, 1) == (4, 4)
    assert multigpu.partition(8, 8, 3) == (1, 3)
    with pytest.raises(ValueError):
        multigpu.partition(8, 3, 0)
    assert [multigpu.owner_of(r, 8, 4) for r in range(8)] == [0, 0, 1, 1, 2, 2, 3, 3]
    meta = oracle.meta_c1(8, 32, 1, 0)
    plan, _ = oracle.plan_routing(meta, oracle.parse_topology("g1n8"))
    sent, recv = multigpu.exchange_bytes(plan.c_src, plan.c_dst, plan.c_start, plan.c_end, 8, 8, 6160)
    # conservation: everything sent off-process is received off-process
    assert sent.sum() == recv.sum()
    n = plan.c_end - plan.c_start
    assert sent.sum() == int(n[plan.c_src != plan.c_dst].sum()) * 6160
    s1, r1 = multigpu.exchange_bytes(plan.c_src, plan.c_dst, plan.c_start, plan.c_end, 8, 1, 6160)
    assert s1.sum() == 0 and r1.sum() == 0  # one process: a local permutation


def _gloo_worker(rank, size, port, topo, q):
    """One process of a 2-process gloo world: the product's partition
    (multigpu.partition / owner_of) decides what this process hosts; it
    pushes every chunk (route) and every head slice (pre_attn) whose source
    rank it hosts to the owner of the destination rank -- the decomposition
    of the device job builders (ulysses_job in csrc/exchange.cu) -- over
    gloo; the assembled ranks must equal the oracle's single-process
    route / pre_attn, and the bytes shipped must equal the product's
    multigpu.phase_bytes accounting (the numbers bench.py reports)."""
    import copy

    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        W, width, heads = 8, 8, 4
        row_bytes = width * 8
        meta = oracle.meta_c1(W, 6, 3, 1)
        n_local, first = multigpu.partition(W, size, rank)
        mine = range(first, first + n_local)
        tp = oracle.parse_topology(topo)
        topology = api.parse_topology(topo)
        plan, _ = oracle.plan_routing(meta, tp, d_model=64, n_heads=heads)
        world = oracle.make_world(meta, width, heads)  # every process can regenerate any rank
        ok = True

        def exchange(outbox):
            inbox = [None] * size
            dist.all_gather_object(inbox, outbox)
            return [m for q_ in range(size) for m in inbox[q_][rank]]

        # ---- route: rows of chunk c from its source rank to its target slot
        offs = {r: np.cumsum([0] + [s_[2] for s_ in plan.target[r]]) for r in range(W)}
        src_offs = {r: np.cumsum([0] + [s_[2] for s_ in plan.origin[r]]) for r in range(W)}
        out = {r: np.zeros((int(offs[r][-1]), row_bytes), np.uint8) for r in mine}
        outbox = {q_: [] for q_ in range(size)}
        shipped = 0
        for c in range(plan.n_chunks):
            s_, d = int(plan.c_src[c]), int(plan.c_dst[c])
            if s_ not in mine or plan.c_end[c] == plan.c_start[c]:
                continue
            si = [k for k, sg in enumerate(plan.origin[s_]) if sg[0] == plan.c_id[c]][0]
            di = [k for k, sg in enumerate(plan.target[d]) if sg[0] == plan.c_id[c] and sg[1] == plan.c_start[c]][0]
            rows = world.ranks[s_].payload[src_offs[s_][si] + plan.c_start[c]:src_offs[s_][si] + plan.c_end[c]]
            owner = multigpu.owner_of(d, W, size)
            if owner != rank:
                shipped += rows.shape[0] * (row_bytes + 16)
            outbox[owner].append((d, int(offs[d][di]), rows.copy()))
        for d, row, rows in exchange(outbox):
            out[d][row:row + len(rows)] = rows
        routed = oracle.route(world, plan)
        ok &= all(np.array_equal(out[r], routed.ranks[r].payload) for r in out)
        sent, recv = multigpu.phase_bytes(plan, "route", topology, W, size, [row_bytes])
        ok &= int(sent[rank]) == shipped

        # ---- pre_attn: chunk (q, m) on member m sends head slice d to member d
        want = copy.deepcopy(routed)
        shipped = 0
        outbox = {q_: [] for q_ in range(size)}
        uly = {}
        U = tp.unit_size
        for b, g in enumerate(tp.bag_sizes):
            if g == 1:
                continue
            sl = row_bytes // g
            for rep in range(W // U):
                ranks = [rep * U + x for x in tp.bag_ranks(b)]
                ids = [s_[0] for s_ in routed.ranks[ranks[0]].segments]
                full = [sum(routed.ranks[r].segments[k][2] for r in ranks) for k in range(len(ids))]
                base = np.cumsum([0] + full)
                for r in ranks:
                    if r in mine:
                        uly[r] = np.zeros((int(base[-1]), sl), np.uint8)
                for m, r in enumerate(ranks):
                    if r not in mine:
                        continue
                    row = 0
                    for k, seg in enumerate(routed.ranks[r].segments):
                        n = seg[2]
                        for d, dr in enumerate(ranks):
                            owner = multigpu.owner_of(dr, W, size)
                            piece = routed.ranks[r].payload[row:row + n, d * sl:(d + 1) * sl].copy()
                            if owner != rank:
                                shipped += n * (sl + 16)
                            outbox[owner].append((dr, int(base[k] + seg[1]), piece))
                        row += n
                oracle.pre_attn(want, ranks)
        for d, row, rows in exchange(outbox):
            uly[d][row:row + len(rows)] = rows
        ok &= all(np.array_equal(uly[r], want.ranks[r].payload) for r in uly)
        sent, recv = multigpu.phase_bytes(plan, "pre_attn", topology, W, size, [row_bytes])
        ok &= int(sent[rank]) == shipped
        # received bytes agree with what the peer shipped to us
        got = [None] * size
        dist.all_gather_object(got, (int(sent[rank]), int(recv[rank])))
        ok &= sum(x[0] for x in got) == sum(x[1] for x in got)
        q.put((rank, bool(ok)))
    except Exception as e:
        q.put((rank, f"{type(e).__name__}: {e}"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("topo", ["g1n8", "g2n4", "g4n2", "g1n2+g2n1+g4n1"])
def test_two_process_push_decomposition_gloo(topo):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, topo, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res


def _ipc_worker(rank, size, port, topo, q, barrier="auto", steps=1, transport=None, pipeline=False):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), SEQBAL_BARRIER_TIMEOUT_MS="20000")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        import paper_2508_06001_b200 as sb
        W = 8
        meta = oracle.meta_c1(W, 5, 2, 0)
        group = multigpu.PeerGroup(barrier_mode=barrier)
        assert group.same_device and group.mode == ("host" if barrier == "auto" else barrier)
        n_local, first = multigpu.partition(W, size, rank)
        planner = sb.Planner(topo, W, max_seqs=64)
        rows = int(sum(int(x.sum()) for x in meta.lens))
        tr = None
        if transport is not None:  # pack -> all-to-all-v -> unpack; worlds without IPC mappings
            tr = multigpu.CollectiveTransport(group, 4 * rows * 80, 4 * rows * 80, transport)
        gather = multigpu.MetaGather(group, W, 8, transport=tr)
        gather.set_local(meta.ids[first:first + n_local], meta.lens[first:first + n_local])
        mk = lambda: multigpu.make_world(group, W, 4, [64], capacity_rows=rows, max_bag=planner.max_bag,
                                         share=tr is None)
        A, B, Cw, D, E = mk(), mk(), mk(), mk(), mk()
        dm = gather.gather()
        gather.status()
        A.layout_origin(dm)
        A.fill_witness(dm)
        group.barrier()
        phases = multigpu.x_phases(A, B, Cw, D, E, planner.max_bag > 1)
        if pipeline:  # two batches in flight: gather/plan/prepare of k+1 under k's copies
            gather2 = multigpu.MetaGather(group, W, 8)
            gather2.set_local(meta.ids[first:first + n_local], meta.lens[first:first + n_local])
            pipe = multigpu.PlanAhead(group, [gather, gather2], [planner, sb.Planner(topo, W, max_seqs=64)], phases)
            pipe.prime()
            for _ in range(steps):
                pipe.pair()
            torch.cuda.synchronize()
            pipe.status()
        else:
            for _ in range(steps):
                multigpu.step(group, gather, planner, phases, transport=tr)
        torch.cuda.synchronize()
        group.barrier_status()  # CommError if a device barrier timed out
        plan, _ = oracle.plan_routing(meta, oracle.parse_topology(topo))  # FLUX model, as the planner
        w0 = oracle.make_world(meta, 8, 4)
        routed = oracle.route(w0, plan)
        bad = []
        for r in range(first, first + n_local):
            if not np.array_equal(B.read_rank(1, r), routed.ranks[r].payload.reshape(-1)):
                bad.append(f"routed payload r{r}")
            meta_b = B.read_rank(0, r).view(np.uint64).reshape(-1, 2)
            if not np.array_equal(meta_b[:, 0], routed.ranks[r].ids):
                bad.append(f"routed ids r{r}")
            if not np.array_equal(E.read_rank(1, r), A.read_rank(1, r)):
                bad.append(f"round trip r{r}")
            if planner.max_bag > 1 and not np.array_equal(D.read_rank(1, r), B.read_rank(1, r)):
                bad.append(f"post(pre) r{r}")
        if group.sum_u64(B.checksum()) != oracle.checksum(w0):
            bad.append("checksum")
        if tr is not None:  # the all-to-all-v carried exactly the cross-process bytes of route
            hp = planner.download()
            sent, recv = multigpu.phase_bytes(hp, "reverse_route", planner.topology, W, size, [64])
            out_splits, in_splits = tr.last_counts
            if sum(out_splits) != int(sent[rank]) or sum(in_splits) != int(recv[rank]):
                bad.append(f"a2a bytes {tr.last_counts} vs {sent[rank]},{recv[rank]}")
            for w in (A, B, Cw, D, E):
                w.status()
        q.put((rank, True if not bad else ";".join(bad)))
        group.barrier()
        gather.close()
        group.close()
    except Exception as e:  # surface worker failures in the parent
        q.put((rank, f"{type(e).__name__}: {e}"))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("topo", ["g1n8", "g2n4", "g4n2"])
def test_two_processes_share_one_gpu_through_ipc(topo):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, topo, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res


@pytest.mark.gpu
@pytest.mark.parametrize("topo", ["g1n8", "g2n4"])
def test_two_processes_device_barrier(topo):
    """The device barrier (k_barrier: system-scope flags in peer memory,
    device epoch counter, bounded spin) closing every phase of three steps,
    two processes on one GPU."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, topo, q, "device", 3)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res


@pytest.mark.gpu
@pytest.mark.parametrize("topo", ["g2n4", "g4n2"])
def test_four_processes_device_barrier(topo):
    """Four processes (two ranks each) on one GPU: peer maps, the device
    barrier's all-to-all flag pattern and the per-process job split beyond
    the two-process case (what an N = 4 / 8 box runs), checked against the
    oracle for two steps."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 4, port, topo, q, "device", 2)) for r in range(4)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True, 2: True, 3: True}, res


@pytest.mark.gpu
@pytest.mark.parametrize("topo", ["g1n8", "g2n4", "g4n2", "g1n2+g2n1+g4n1"])
def test_two_processes_collective_transport(topo):
    """The NCCL-baseline decomposition (sb_exchange_pack -> all-to-all-v ->
    sb_exchange_unpack, all-gathered metadata) between two processes on one
    GPU: worlds carry no IPC mappings, the all-to-all runs over gloo through
    pinned host buffers ('staged'; NCCL itself refuses two ranks on one
    device).  Routed payload, ids, post(pre) and the round trip must match
    the oracle exactly, and the all-to-all must carry exactly the
    cross-process bytes."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, topo, q, "auto", 2, "staged")) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res


def _nccl_one_worker(port, topo, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        import paper_2508_06001_b200 as sb
        W = 8
        meta = oracle.meta_c1(W, 5, 2, 0)
        group = multigpu.PeerGroup()
        planner = sb.Planner(topo, W, max_seqs=64)
        rows = int(sum(int(x.sum()) for x in meta.lens))
        tr = multigpu.CollectiveTransport(group, 4 * rows * 80, 4 * rows * 80, "nccl")
        gather = multigpu.MetaGather(group, W, 8, transport=tr)
        gather.set_local(meta.ids, meta.lens)
        mk = lambda: multigpu.make_world(group, W, 4, [64], capacity_rows=rows, max_bag=planner.max_bag, share=False)
        A, B, Cw, D, E = mk(), mk(), mk(), mk(), mk()
        dm = gather.gather()
        gather.status()
        A.layout_origin(dm)
        A.fill_witness(dm)
        multigpu.step(group, gather, planner, multigpu.x_phases(A, B, Cw, D, E, planner.max_bag > 1), transport=tr)
        torch.cuda.synchronize()
        plan, _ = oracle.plan_routing(meta, oracle.parse_topology(topo))
        routed = oracle.route(oracle.make_world(meta, 8, 4), plan)
        bad = [r for r in range(W) if not np.array_equal(B.read_rank(1, r), routed.ranks[r].payload.reshape(-1))
               or not np.array_equal(E.read_rank(1, r), A.read_rank(1, r))]
        q.put((0, True if not bad else f"ranks {bad}"))
        gather.close()
        group.close()
    except Exception as e:
        q.put((0, f"{type(e).__name__}: {e}"))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("topo", ["g1n8", "g2n4"])
def test_one_process_nccl_transport(topo):
    """The NCCL backend itself (torch.distributed NCCL group: all_to_all_single
    + in-place all_gather_into_tensor) on the one GPU this box has: one
    process hosting all 8 ranks, so every byte is a local pack->unpack."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_one_worker, args=(_free_port(), topo, q))
    p.start()
    res = dict([q.get(timeout=300)])
    p.join(timeout=60)
    assert res == {0: True}, res


@pytest.mark.gpu
@pytest.mark.parametrize("topo", ["g1n8", "g2n4"])
def test_two_processes_plan_ahead_pipeline(topo):
    """multigpu.PlanAhead: batch k+1's all-gather (closed by a second device
    barrier on the side stream), plan and preparations run under batch k's
    copies, two planners and gather buffers alternating; three pairs of
    steps between two processes on one GPU, results as the serial step's."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, topo, q, "device", 3, None, True)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res


def _barrier_timeout_worker(rank, size, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        from paper_2508_06001_b200 import _capi
        group = multigpu.PeerGroup(barrier_mode="device")
        group.set_timeout(300.0)
        group.barrier()
        group.barrier_status()  # both arrive: fine
        dist.barrier()
        if rank == 0:  # process 1 never arrives: bounded wait, then SB_ERR_COMM
            group.barrier()
            try:
                group.barrier_status()
                q.put((rank, "no error"))
            except _capi.CommError as e:
                q.put((rank, "process 1 did not arrive" in str(e)))
        else:
            q.put((rank, True))
        dist.barrier()
        group.close()
    except Exception as e:
        q.put((rank, f"{type(e).__name__}: {e}"))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_device_barrier_times_out_with_comm_error():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_barrier_timeout_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res


@pytest.mark.gpu
def test_bench_gpus_2_spawns_two_processes():
    """`python bench.py --gpus 2` launches its own two worker processes (no
    torchrun from the caller) and reports the multi-process line: n_gpus 2,
    bit-exact round trip, per-phase all-to-all bytes and times."""
    import json
    import subprocess
    import sys

    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "3",
                        "--warmup", "1"], capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [json.loads(x) for x in p.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = lines[0]
    assert d["n_gpus"] == 2 and d["checksum_conserved"] and d["e2e"]["round_trip_bit_exact"]
    for ph in ("route", "pre_attn", "post_attn", "reverse_route"):
        assert d["phases"][ph]["us"] > 0 and "busiest_bytes" in d["phases"][ph], d["phases"]
    # C2 (g1n4+g2n2) over 2 processes: the bags of 2 live inside process 1, so
    # only route / reverse_route cross processes
    assert d["phases"]["route"]["busiest_bytes"] > 0 and d["phases"]["pre_attn"]["busiest_bytes"] == 0
    assert d["a2a_gbs"] is not None and d["gpu_launches"] > 0
