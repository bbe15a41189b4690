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
from paper_2508_06001_b200 import multigpu


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
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        W = 8
        meta = oracle.meta_c1(W, 6, 3, 1)
        n_local, first = multigpu.partition(W, size, rank)
        plan, _ = oracle.plan_routing(meta, oracle.parse_topology(topo))
        world = oracle.make_world(meta, 8, 4)  # every process can regenerate any rank
        # target layout of my ranks
        out = {r: np.zeros((sum(s[2] for s in plan.target[r]), 64), np.uint8) for r in range(first, first + n_local)}
        offs = {r: np.cumsum([0] + [s[2] for s in plan.target[r]]) for r in range(W)}
        src_offs = {r: np.cumsum([0] + [s[2] for s in plan.origin[r]]) for r in range(W)}
        # sender push: for every chunk whose source I host, ship rows to the owner of dst
        outbox = {q_: [] for q_ in range(size)}
        for c in range(plan.n_chunks):
            s, d = int(plan.c_src[c]), int(plan.c_dst[c])
            if not (first <= s < first + n_local) or plan.c_end[c] == plan.c_start[c]:
                continue
            si = [k for k, sg in enumerate(plan.origin[s]) if sg[0] == plan.c_id[c]][0]
            di = [k for k, sg in enumerate(plan.target[d]) if sg[0] == plan.c_id[c] and sg[1] == plan.c_start[c]][0]
            rows = world.ranks[s].payload[src_offs[s][si] + plan.c_start[c]:src_offs[s][si] + plan.c_end[c]]
            outbox[multigpu.owner_of(d, W, size)].append((d, int(offs[d][di]), rows.copy()))
        inbox = [None] * size
        dist.all_gather_object(inbox, outbox)
        for q_ in range(size):
            for d, row, rows in inbox[q_][rank]:
                out[d][row:row + len(rows)] = rows
        routed = oracle.route(world, plan)
        ok = all(np.array_equal(out[r], routed.ranks[r].payload) for r in out)
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("topo", ["g1n8", "g2n4", "g4n2"])
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
    assert res == {0: True, 1: True}


def _ipc_worker(rank, size, port, topo, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        import paper_2508_06001_b200 as sb
        W = 8
        meta = oracle.meta_c1(W, 5, 2, 0)
        group = multigpu.PeerGroup()
        assert group.same_device and group.mode == "host"
        n_local, first = multigpu.partition(W, size, rank)
        gather = multigpu.MetaGather(group, W, 8)
        gather.set_local(meta.ids[first:first + n_local], meta.lens[first:first + n_local])
        planner = sb.Planner(topo, W, max_seqs=64)
        rows = int(sum(int(x.sum()) for x in meta.lens))
        mk = lambda: multigpu.make_world(group, W, 4, [64], capacity_rows=rows, max_bag=planner.max_bag)
        A, B, Cw, D, E = mk(), mk(), mk(), mk(), mk()
        dm = gather.gather()
        gather.status()
        A.layout_origin(dm)
        A.fill_witness(dm)
        group.barrier()
        multigpu.step(group, gather, planner, A, B, Cw, D, E, planner.max_bag > 1)
        torch.cuda.synchronize()
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
