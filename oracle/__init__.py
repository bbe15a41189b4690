"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the balance-and-redistribute path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline.  The product (``paper_2508_06001_b200``) never imports
it.

Two layers:
  * ``liboracle.so`` (oracle/seqbal_oracle.c): plain-C restatement of the
    reference planner, RNG, witness and checksum (file:line cited there).
  * this module: ctypes bindings plus a numpy restatement of the reference
    exchange (``route``/``reverse_route``/``pre_attn``/``post_attn``,
    /root/reference/proj/src/exchange.cpp) over byte-valued rank buffers.

Parity pin: tests/test_oracle_golden.py checks every function here against
fixtures produced by the unmodified reference (``oracle/_ref/ref_harness``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_HARNESS = os.path.join(HERE, "_ref", "ref_harness")

_lib = None


def build(quiet: bool = True) -> None:
    """Compile liboracle.so (and oracle/_ref when /root/reference exists)."""
    targets = ["oracle"]
    if os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        u64, i64, i32, dbl = C.c_uint64, C.c_int64, C.c_int32, C.c_double
        vp = C.c_void_p
        L.or_splitmix64.restype = u64
        L.or_splitmix64.argtypes = [u64]
        L.or_derive_key.restype = u64
        L.or_derive_key.argtypes = [vp, C.c_int]
        L.or_rng_u64.restype = u64
        L.or_rng_u64.argtypes = [u64, u64]
        L.or_rng_int.restype = i64
        L.or_rng_int.argtypes = [u64, u64, i64, i64]
        L.or_rng_real.restype = dbl
        L.or_rng_real.argtypes = [u64, u64, dbl, dbl]
        L.or_make_sample_id.restype = u64
        L.or_make_sample_id.argtypes = [i64, C.c_int, C.c_int]
        L.or_aspect_multiplier.restype = dbl
        L.or_aspect_multiplier.argtypes = [u64, i64, C.c_int]
        L.or_visual_tokens.restype = i64
        L.or_visual_tokens.argtypes = [C.c_int, C.c_int, C.c_int, dbl]
        L.or_next_batch.restype = C.c_int
        L.or_next_batch.argtypes = [C.c_int, vp, vp, vp, vp, vp, C.c_int, i64, u64, vp, vp, vp]
        L.or_c1_batch.restype = None
        L.or_c1_batch.argtypes = [u64, i64, C.c_int, C.c_int, vp, vp]
        L.or_payload_value.restype = dbl
        L.or_payload_value.argtypes = [u64, i64, C.c_int]
        L.or_block_perturbation.restype = dbl
        L.or_block_perturbation.argtypes = [u64, i64]
        L.or_digest.restype = u64
        L.or_digest.argtypes = [vp, C.c_size_t, u64]
        L.or_gamma_weighted_workload.restype = dbl
        L.or_gamma_weighted_workload.argtypes = [i64, C.c_int, dbl]
        L.or_chunk_lengths.restype = None
        L.or_chunk_lengths.argtypes = [i64, C.c_int, vp]
        L.or_wir.restype = dbl
        L.or_wir.argtypes = [vp, C.c_int]
        L.or_assign_to_bags.restype = C.c_int
        L.or_assign_to_bags.argtypes = [C.c_int, vp, vp, C.c_int, vp, vp, vp, vp, vp]
        L.or_plan_routing.restype = C.c_int
        L.or_plan_routing.argtypes = [vp, vp]
        L.or_identity_plan.restype = C.c_int
        L.or_identity_plan.argtypes = [C.c_int, vp, vp, vp, vp]
        L.or_reverse_plan.restype = C.c_int
        L.or_reverse_plan.argtypes = [C.c_int, i64] + [vp] * 13
        L.or_fill_witness.restype = None
        L.or_fill_witness.argtypes = [i64, vp, vp, C.c_int, vp]
        L.or_perturb.restype = None
        L.or_perturb.argtypes = [i64, vp, vp, C.c_int, vp]
        L.or_checksum_rank.restype = u64
        L.or_checksum_rank.argtypes = [i64, vp, vp, C.c_int, C.c_int, vp]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


DIGEST_SEED = 0x6469676573740000


# --------------------------------------------------------------------- rng
def splitmix64(x: int) -> int:
    return lib().or_splitmix64(x & (2**64 - 1))


def derive_key(parts) -> int:
    a = np.asarray([p & (2**64 - 1) for p in parts], dtype=np.uint64)
    return lib().or_derive_key(_p(a), len(a))


def digest(buf, h: int = DIGEST_SEED) -> int:
    a = np.ascontiguousarray(buf)
    return lib().or_digest(_p(a), a.nbytes, h)


def payload_value(sample_id: int, pos: int, col: int) -> float:
    return lib().or_payload_value(sample_id, pos, col)


def block_perturbation(sample_id: int, pos: int) -> float:
    return lib().or_block_perturbation(sample_id, pos)


def gamma_weighted_workload(seq_len: int, d_model: int = 3072, gamma: float = 0.49) -> float:
    return lib().or_gamma_weighted_workload(seq_len, d_model, gamma)


def chunk_lengths(total_len: int, parts: int) -> list[int]:
    out = np.zeros(parts, dtype=np.int64)
    lib().or_chunk_lengths(total_len, parts, _p(out))
    return out.tolist()


def wir(w) -> float:
    a = np.ascontiguousarray(w, dtype=np.float64)
    return lib().or_wir(_p(a), len(a))


def assign_to_bags(ids, workloads, bag_sizes, bag_ids=None):
    ids = np.ascontiguousarray(ids, dtype=np.uint64)
    w = np.ascontiguousarray(workloads, dtype=np.float64)
    sizes = np.ascontiguousarray(bag_sizes, dtype=np.int32)
    bids = np.ascontiguousarray(range(len(sizes)) if bag_ids is None else bag_ids, dtype=np.int32)
    n = len(ids)
    oi = np.zeros(n, np.uint64)
    ow = np.zeros(n, np.float64)
    ob = np.zeros(n, np.int32)
    st = lib().or_assign_to_bags(n, _p(ids), _p(w), len(sizes), _p(sizes), _p(bids), _p(oi), _p(ow), _p(ob))
    if st:
        raise ValueError("ConfigError: assign_to_bags")
    return oi, ow, ob


# ---------------------------------------------------------------- topology
@dataclass
class Topology:
    """topology.hpp:16-52 restated: bags of contiguous unit-local ranks."""
    bag_sizes: list[int]

    @property
    def unit_size(self) -> int:
        return sum(self.bag_sizes)

    def bag_ranks(self, b: int) -> list[int]:
        s = sum(self.bag_sizes[:b])
        return list(range(s, s + self.bag_sizes[b]))


def parse_topology(spec: str) -> Topology:
    """topology.cpp:31-65 (grammar g{G}n{N}(+...)*; errors raise ValueError)."""
    sizes: list[int] = []
    pos = 0
    if not spec:
        raise ValueError("empty topology spec (at offset 0)")

    def num(p):
        q = p
        while q < len(spec) and spec[q].isdigit():
            q += 1
        if q == p:
            raise ValueError(f"expected digits (at offset {p})")
        v = int(spec[p:q])
        if v < 1:
            raise ValueError(f"must be >= 1 (at offset {p})")
        return v, q

    while True:
        if pos >= len(spec) or spec[pos] != "g":
            raise ValueError(f"expected 'g' (at offset {pos})")
        g, pos = num(pos + 1)
        if pos >= len(spec) or spec[pos] != "n":
            raise ValueError(f"expected 'n' (at offset {pos})")
        n, pos = num(pos + 1)
        sizes += [g] * n
        if pos == len(spec):
            break
        if spec[pos] != "+":
            raise ValueError(f"expected '+' or end of spec (at offset {pos})")
        pos += 1
    return Topology(sizes)


# ---------------------------------------------------------------- metadata
@dataclass
class Meta:
    """Per-rank (sample_id, length) lists in gather order (exchange.cpp:68-77)."""
    ids: list  # list of np.uint64 arrays, one per rank
    lens: list  # list of np.int64 arrays

    @property
    def world(self) -> int:
        return len(self.ids)

    def flat(self):
        ids = np.concatenate(self.ids) if self.ids else np.zeros(0, np.uint64)
        lens = np.concatenate(self.lens) if self.lens else np.zeros(0, np.int64)
        off = np.zeros(self.world + 1, np.int64)
        off[1:] = np.cumsum([len(x) for x in self.ids])
        return ids.astype(np.uint64), lens.astype(np.int64), off


def meta_explicit(lens, ids=None) -> Meta:
    out_ids, out_lens = [], []
    nxt = 1
    for r, L in enumerate(lens):
        if ids is None:
            out_ids.append(np.arange(nxt, nxt + len(L), dtype=np.uint64))
            nxt += len(L)
        else:
            out_ids.append(np.asarray(ids[r], dtype=np.uint64))
        out_lens.append(np.asarray(L, dtype=np.int64))
    return Meta(out_ids, out_lens)


def meta_c1(world: int, per_rank: int, seed: int = 1, step: int = 0) -> Meta:
    ids, lens = [], []
    for r in range(world):
        i = np.zeros(per_rank, np.uint64)
        l = np.zeros(per_rank, np.int64)
        lib().or_c1_batch(seed, step, r, per_rank, _p(i), _p(l))
        ids.append(i)
        lens.append(l)
    return Meta(ids, lens)


def parse_data_code(code: str):
    """data_sim.cpp:39-76 (well-formed codes only; the grammar is host input)."""
    import re
    m = re.fullmatch(r"g(\d+)b(\d+)i(\d+)f(\d+)s([01])", code)
    if not m:
        raise ValueError(f"bad data code {code!r}")
    return tuple(int(x) for x in m.groups())


def meta_scenario(world: int, codes, step: int = 0, seed: int = 7) -> Meta:
    specs = [parse_data_code(c) for c in codes]
    arr = [np.asarray([s[k] for s in specs], np.int32) for k in range(5)]
    gpus, batch, res, frames, smooth = arr
    ids, lens = [], []
    for r in range(world):
        n = int(batch.max())
        i = np.zeros(n, np.uint64)
        t = np.zeros(n, np.int64)
        v = np.zeros(n, np.int64)
        got = lib().or_next_batch(len(specs), _p(gpus), _p(batch), _p(res), _p(frames), _p(smooth),
                                  r, step, seed, _p(i), _p(t), _p(v))
        if got < 0:
            raise ValueError("bad scenario")
        ids.append(i[:got].copy())
        lens.append((t[:got] + v[:got]).astype(np.int64))
    return Meta(ids, lens)


# -------------------------------------------------------------------- plan
class _PlanIn(C.Structure):
    _fields_ = [("world_size", C.c_int), ("rank_off", C.c_void_p), ("ids", C.c_void_p),
                ("lens", C.c_void_p), ("unit_size", C.c_int), ("n_bags", C.c_int),
                ("bag_off", C.c_void_p), ("bag_ranks", C.c_void_p), ("d_model", C.c_int),
                ("n_heads", C.c_int), ("gamma", C.c_double)]


class _PlanOut(C.Structure):
    _fields_ = [("cap_chunks", C.c_int64), ("n_chunks", C.c_int64), ("c_id", C.c_void_p),
                ("c_idx", C.c_void_p), ("c_start", C.c_void_p), ("c_end", C.c_void_p),
                ("c_src", C.c_void_p), ("c_dst", C.c_void_p), ("send_off", C.c_void_p),
                ("send_idx", C.c_void_p), ("recv_off", C.c_void_p), ("recv_idx", C.c_void_p),
                ("per_gpu", C.c_void_p), ("per_bag_occ", C.c_void_p), ("violations", C.c_int32),
                ("total_workload", C.c_double), ("wir", C.c_double)]


@dataclass
class Plan:
    """RoutingPlan (balancer.hpp:67-76) as numpy SoA."""
    world: int
    c_id: np.ndarray
    c_idx: np.ndarray
    c_start: np.ndarray
    c_end: np.ndarray
    c_src: np.ndarray
    c_dst: np.ndarray
    send: list
    recv: list
    origin: list  # per rank list of (id, first_pos, len)
    target: list

    @property
    def n_chunks(self) -> int:
        return len(self.c_id)

    def chunk_rows(self):
        return [(int(self.c_id[i]), int(self.c_idx[i]), int(self.c_start[i]), int(self.c_end[i]),
                 int(self.c_src[i]), int(self.c_dst[i])) for i in range(self.n_chunks)]


@dataclass
class Report:
    per_gpu_workload: np.ndarray
    per_bag_occupancy: np.ndarray
    capacity_violations: int
    total_workload: float
    wir: float


def _csr_lists(off, idx):
    return [idx[off[r]:off[r + 1]].astype(np.int64).tolist() for r in range(len(off) - 1)]


def _target_from(world, c_id, c_start, c_end, recv):
    return [[(int(c_id[c]), int(c_start[c]), int(c_end[c] - c_start[c])) for c in recv[r]]
            for r in range(world)]


def _origin_from(meta: Meta):
    return [[(int(i), 0, int(l)) for i, l in zip(meta.ids[r], meta.lens[r])] for r in range(meta.world)]


def plan_routing(meta: Meta, topology: Topology, d_model: int = 3072, n_heads: int = 24,
                 gamma: float = 0.49):
    """balancer.cpp:105-225 via oracle/seqbal_oracle.c."""
    W = meta.world
    ids, lens, off = meta.flat()
    sizes = topology.bag_sizes
    bag_off = np.zeros(len(sizes) + 1, np.int32)
    bag_off[1:] = np.cumsum(sizes)
    bag_ranks = np.arange(topology.unit_size, dtype=np.int32)
    cap = max(1, len(ids) * max(sizes))
    arrs = dict(c_id=np.zeros(cap, np.uint64), c_idx=np.zeros(cap, np.int32), c_start=np.zeros(cap, np.int64),
                c_end=np.zeros(cap, np.int64), c_src=np.zeros(cap, np.int32), c_dst=np.zeros(cap, np.int32),
                send_off=np.zeros(W + 1, np.int64), send_idx=np.zeros(cap, np.int32),
                recv_off=np.zeros(W + 1, np.int64), recv_idx=np.zeros(cap, np.int32),
                per_gpu=np.zeros(W, np.float64),
                per_bag_occ=np.zeros(max(1, (W // max(1, topology.unit_size)) * len(sizes)), np.float64))
    pin = _PlanIn(W, _p(off).value, _p(ids).value, _p(lens).value, topology.unit_size, len(sizes),
                  _p(bag_off).value, _p(bag_ranks).value, d_model, n_heads, gamma)
    pout = _PlanOut()
    pout.cap_chunks = cap
    for k, a in arrs.items():
        setattr(pout, k, _p(a).value)
    st = lib().or_plan_routing(C.byref(pin), C.byref(pout))
    if st == 1:
        raise ValueError("ConfigError: plan_routing")
    if st:
        raise RuntimeError(f"oracle plan_routing status {st}")
    n = pout.n_chunks
    send = _csr_lists(arrs["send_off"], arrs["send_idx"])
    recv = _csr_lists(arrs["recv_off"], arrs["recv_idx"])
    c = {k: arrs[k][:n].copy() for k in ("c_id", "c_idx", "c_start", "c_end", "c_src", "c_dst")}
    plan = Plan(W, **c, send=send, recv=recv, origin=_origin_from(meta),
                target=_target_from(W, c["c_id"], c["c_start"], c["c_end"], recv))
    reps = W // topology.unit_size
    rep = Report(arrs["per_gpu"].copy(), arrs["per_bag_occ"][:reps * len(sizes)].copy(),
                 int(pout.violations), float(pout.total_workload), float(pout.wir))
    return plan, rep


def identity_plan(meta: Meta) -> Plan:
    """balancer.cpp:227-240"""
    W = meta.world
    ids, lens, off = meta.flat()
    cap = max(1, len(ids))
    a = dict(c_id=np.zeros(cap, np.uint64), c_idx=np.zeros(cap, np.int32), c_start=np.zeros(cap, np.int64),
             c_end=np.zeros(cap, np.int64), c_src=np.zeros(cap, np.int32), c_dst=np.zeros(cap, np.int32),
             send_off=np.zeros(W + 1, np.int64), send_idx=np.zeros(cap, np.int32),
             recv_off=np.zeros(W + 1, np.int64), recv_idx=np.zeros(cap, np.int32))
    pout = _PlanOut()
    pout.cap_chunks = cap
    for k, v in a.items():
        setattr(pout, k, _p(v).value)
    lib().or_identity_plan(W, _p(off), _p(ids), _p(lens), C.byref(pout))
    n = pout.n_chunks
    send = _csr_lists(a["send_off"], a["send_idx"])
    recv = _csr_lists(a["recv_off"], a["recv_idx"])
    c = {k: a[k][:n].copy() for k in ("c_id", "c_idx", "c_start", "c_end", "c_src", "c_dst")}
    return Plan(W, **c, send=send, recv=recv, origin=_origin_from(meta),
                target=_target_from(W, c["c_id"], c["c_start"], c["c_end"], recv))


def reverse_plan(plan: Plan) -> Plan:
    """balancer.cpp:242-287 (receive order tie-break by chunk index; see header)."""
    W = plan.world
    n = plan.n_chunks
    seg_off = np.zeros(W + 1, np.int64)
    seg_off[1:] = np.cumsum([len(s) for s in plan.origin])
    flat = [s for r in plan.origin for s in r]
    seg_id = np.asarray([s[0] for s in flat], np.uint64)
    seg_first = np.asarray([s[1] for s in flat], np.int64)
    seg_len = np.asarray([s[2] for s in flat], np.int64)
    send_off = np.zeros(W + 1, np.int64)
    recv_off = np.zeros(W + 1, np.int64)
    send_idx = np.zeros(max(1, n), np.int32)
    recv_idx = np.zeros(max(1, n), np.int32)
    cid = np.ascontiguousarray(plan.c_id, np.uint64)
    cs = np.ascontiguousarray(plan.c_start, np.int64)
    ce = np.ascontiguousarray(plan.c_end, np.int64)
    csrc = np.ascontiguousarray(plan.c_src, np.int32)
    cdst = np.ascontiguousarray(plan.c_dst, np.int32)
    st = lib().or_reverse_plan(W, n, _p(cid), _p(cs), _p(ce), _p(csrc), _p(cdst), _p(seg_off),
                               _p(seg_id), _p(seg_first), _p(seg_len), _p(send_off), _p(send_idx),
                               _p(recv_off), _p(recv_idx))
    if st:
        raise RuntimeError("IntegrityError: reverse_plan: chunk does not fit any destination segment")
    return Plan(W, plan.c_id.copy(), plan.c_idx.copy(), plan.c_start.copy(), plan.c_end.copy(),
                plan.c_dst.copy(), plan.c_src.copy(), _csr_lists(send_off, send_idx),
                _csr_lists(recv_off, recv_idx), origin=[list(x) for x in plan.target],
                target=[list(x) for x in plan.origin])


# ------------------------------------------------------------------- world
FULL, SLICED = 0, 1  # LayoutMode::ChunkFullHeads / FullSeqPartialHeads


@dataclass
class RankBuf:
    """exchange.hpp:22-34 with the payload held as raw bytes."""
    ids: np.ndarray
    pos: np.ndarray
    payload: np.ndarray  # uint8 [rows, width_bytes]
    segments: list
    mode: int = FULL
    head_lo: int = 0
    head_hi: int = 0

    @property
    def rows(self) -> int:
        return len(self.ids)


@dataclass
class World:
    row_bytes: int  # full payload width in bytes (exchange.hpp:40-44 payload_width)
    n_heads: int
    ranks: list = field(default_factory=list)


def make_world(meta: Meta, width: int, n_heads: int) -> World:
    """exchange.cpp:31-66 with double payload of `width` columns."""
    if width < 1 or n_heads < 1 or width % n_heads:
        raise ValueError("ConfigError: payload width must be a positive multiple of n_heads")
    w = World(width * 8, n_heads)
    for r in range(meta.world):
        L = meta.lens[r]
        ids = np.repeat(meta.ids[r], L).astype(np.uint64)
        pos = np.concatenate([np.arange(l, dtype=np.int64) for l in L]) if len(L) else np.zeros(0, np.int64)
        pay = np.zeros((len(ids), width), np.float64)
        if len(ids):
            lib().or_fill_witness(len(ids), _p(ids), _p(pos), width, _p(pay))
        w.ranks.append(RankBuf(ids, pos, pay.view(np.uint8).reshape(len(ids), width * 8),
                               [(int(i), 0, int(l)) for i, l in zip(meta.ids[r], L)], FULL, 0, n_heads))
    return w


def checksum(world: World) -> int:
    """exchange.cpp:438-457 for double payloads."""
    acc = 0
    width_d = world.row_bytes // 8
    for b in world.ranks:
        wb = b.payload.shape[1] if b.payload.ndim == 2 else world.row_bytes
        wd = wb // 8
        head_cols = 0 if wd == width_d else b.head_lo * (width_d // world.n_heads)
        pay = np.ascontiguousarray(b.payload).view(np.float64)
        acc = (acc + lib().or_checksum_rank(b.rows, _p(np.ascontiguousarray(b.ids)),
                                            _p(np.ascontiguousarray(b.pos)), wd, head_cols, _p(pay))) % 2**64
    return acc


def worlds_equal(a: World, b: World) -> bool:
    """exchange.cpp:459-480"""
    if a.row_bytes != b.row_bytes or a.n_heads != b.n_heads or len(a.ranks) != len(b.ranks):
        return False
    for x, y in zip(a.ranks, b.ranks):
        if (x.mode, x.head_lo, x.head_hi, x.segments) != (y.mode, y.head_lo, y.head_hi, y.segments):
            return False
        if x.payload.shape != y.payload.shape:
            return False
        if not (np.array_equal(x.ids, y.ids) and np.array_equal(x.pos, y.pos)
                and np.array_equal(x.payload, y.payload)):
            return False
    return True


def _seg_offsets(segs):
    out, cur = [], 0
    for s in segs:
        out.append(cur)
        cur += s[2]
    return out


def _locate(segs, cid, start, end):
    for k, s in enumerate(segs):
        if s[0] == cid and start >= s[1] and end <= s[1] + s[2]:
            return k
    raise RuntimeError(f"IntegrityError: route: sample {cid} chunk [{start},{end}) has no containing segment")


def route(world: World, plan: Plan) -> World:
    """exchange.cpp:127-194 (out-of-place permutation of rows)."""
    if len(world.ranks) != plan.world:
        raise RuntimeError("IntegrityError: route: plan world size mismatch")
    for r, b in enumerate(world.ranks):
        if b.mode != FULL or b.payload.shape[1] != world.row_bytes:
            raise RuntimeError(f"IntegrityError: route: rank {r} is not in (partial sequences, full heads) layout")
        if b.segments != plan.origin[r]:
            bad = next((s for s, t in zip(plan.origin[r], b.segments) if s != t), plan.origin[r][:1])
            raise RuntimeError(f"IntegrityError: route: rank {r} segment mismatch for sample {bad}")
    so = [_seg_offsets(s) for s in plan.origin]
    do = [_seg_offsets(s) for s in plan.target]
    out = World(world.row_bytes, world.n_heads)
    for r in range(plan.world):
        rows = sum(s[2] for s in plan.target[r])
        out.ranks.append(RankBuf(np.zeros(rows, np.uint64), np.zeros(rows, np.int64),
                                 np.zeros((rows, world.row_bytes), np.uint8), list(plan.target[r]),
                                 FULL, 0, world.n_heads))
    # index segments by sample id for the `locate` scans (exchange.cpp:156-167)
    for c in range(plan.n_chunks):
        cid, st, en = int(plan.c_id[c]), int(plan.c_start[c]), int(plan.c_end[c])
        if en == st:
            continue
        s, d = int(plan.c_src[c]), int(plan.c_dst[c])
        ks = _locate(plan.origin[s], cid, st, en)
        kd = _locate(plan.target[d], cid, st, en)
        sr = so[s][ks] + (st - plan.origin[s][ks][1])
        dr = do[d][kd] + (st - plan.target[d][kd][1])
        n = en - st
        src, dst = world.ranks[s], out.ranks[d]
        dst.payload[dr:dr + n] = src.payload[sr:sr + n]
        dst.ids[dr:dr + n] = src.ids[sr:sr + n]
        dst.pos[dr:dr + n] = src.pos[sr:sr + n]
    return out


def reverse_route(world: World, plan: Plan) -> World:
    """exchange.cpp:196-198"""
    return route(world, reverse_plan(plan))


def pre_attn(world: World, bag_ranks) -> list:
    """exchange.cpp:255-331, in place; returns the full per-sequence lengths."""
    g = len(bag_ranks)
    first = world.ranks[bag_ranks[0]]
    if g == 1:
        return [s[2] for s in first.segments]
    if world.n_heads % g:
        raise ValueError("ConfigError: pre_attn: bag does not divide n_heads")
    ids = [s[0] for s in first.segments]
    for r in bag_ranks:  # check_bag_chunk_layout, exchange.cpp:210-251
        b = world.ranks[r]
        if b.mode != FULL:
            raise RuntimeError(f"IntegrityError: pre_attn: rank {r} is not in chunk layout")
        if len(b.segments) != len(ids) or any(s[0] != i for s, i in zip(b.segments, ids)):
            raise RuntimeError("IntegrityError: pre_attn: bag members disagree")
    full = []
    for s in range(len(ids)):
        tot = sum(world.ranks[r].segments[s][2] for r in bag_ranks)
        lens = chunk_lengths(tot, g)
        start = 0
        for m, r in enumerate(bag_ranks):
            seg = world.ranks[r].segments[s]
            if seg[1] != start or seg[2] != lens[m]:
                raise RuntimeError(f"IntegrityError: pre_attn: sample {ids[s]} is not split by the canonical chunk rule")
            start += lens[m]
        full.append(tot)
    rb = world.row_bytes
    sl = rb // g
    total = sum(full)
    hpr = world.n_heads // g
    staged = []
    for m in range(g):
        staged.append(RankBuf(np.zeros(total, np.uint64), np.zeros(total, np.int64),
                              np.zeros((total, sl), np.uint8), [(i, 0, l) for i, l in zip(ids, full)],
                              SLICED, m * hpr, (m + 1) * hpr))
    for sm, sr in enumerate(bag_ranks):
        src = world.ranks[sr]
        row, base = 0, 0
        for s in range(len(ids)):
            seg = src.segments[s]
            n = seg[2]
            if n > 0:
                for dm in range(g):
                    d = staged[dm]
                    a = base + seg[1]
                    d.payload[a:a + n] = src.payload[row:row + n, dm * sl:(dm + 1) * sl]
                    d.ids[a:a + n] = src.ids[row:row + n]
                    d.pos[a:a + n] = src.pos[row:row + n]
            row += n
            base += full[s]
    for m, r in enumerate(bag_ranks):
        world.ranks[r] = staged[m]
    return full


def post_attn(world: World, bag_ranks) -> None:
    """exchange.cpp:333-436, in place."""
    g = len(bag_ranks)
    if g == 1:
        return
    first = world.ranks[bag_ranks[0]]
    if first.mode != SLICED:
        raise RuntimeError("IntegrityError: post_attn: bag is not in (full sequences, partial heads) layout")
    ids = [s[0] for s in first.segments]
    full = [s[2] for s in first.segments]
    rb = world.row_bytes
    sl = rb // g
    hpr = world.n_heads // g
    for m, r in enumerate(bag_ranks):
        b = world.ranks[r]
        if b.mode != SLICED or b.payload.shape[1] != sl or b.head_lo != m * hpr or b.head_hi != (m + 1) * hpr:
            raise RuntimeError(f"IntegrityError: post_attn: rank {r} head slice does not match its bag position")
        if len(b.segments) != len(ids) or any(s != (i, 0, l) for s, i, l in zip(b.segments, ids, full)):
            raise RuntimeError("IntegrityError: post_attn: bag members disagree")
    lens = [chunk_lengths(l, g) for l in full]
    starts = [[sum(L[:m]) for m in range(g)] for L in lens]
    staged = []
    for m in range(g):
        rows = sum(L[m] for L in lens)
        staged.append(RankBuf(np.zeros(rows, np.uint64), np.zeros(rows, np.int64), np.zeros((rows, rb), np.uint8),
                              [(ids[s], starts[s][m], lens[s][m]) for s in range(len(ids))], FULL, 0, world.n_heads))
    for dm in range(g):
        d = staged[dm]
        row, base = 0, 0
        for s in range(len(ids)):
            n = lens[s][dm]
            if n > 0:
                a = base + starts[s][dm]
                for sm, sr in enumerate(bag_ranks):
                    src = world.ranks[sr]
                    d.payload[row:row + n, sm * sl:(sm + 1) * sl] = src.payload[a:a + n]
                    if sm == 0:
                        d.ids[row:row + n] = src.ids[a:a + n]
                        d.pos[row:row + n] = src.pos[a:a + n]
            row += n
            base += full[s]
    for m, r in enumerate(bag_ranks):
        world.ranks[r] = staged[m]


def perturb(world: World) -> World:
    """simulator.cpp:128-136: payload[r, c] += block_perturbation(id, pos) (double payloads)."""
    out = World(world.row_bytes, world.n_heads)
    for b in world.ranks:
        pay = np.ascontiguousarray(b.payload).view(np.float64).copy()
        if b.rows:
            lib().or_perturb(b.rows, _p(np.ascontiguousarray(b.ids)), _p(np.ascontiguousarray(b.pos)),
                             pay.shape[1], _p(pay))
        out.ranks.append(RankBuf(b.ids.copy(), b.pos.copy(), pay.view(np.uint8).reshape(b.rows, b.payload.shape[1]),
                                 list(b.segments), b.mode, b.head_lo, b.head_hi))
    return out


def rank_digests(b: RankBuf):
    return (digest(np.ascontiguousarray(b.ids)), digest(np.ascontiguousarray(b.pos)),
            digest(np.ascontiguousarray(b.payload)))


# ------------------------------------------------------ reference harness
def ref_available() -> bool:
    return os.path.exists(REF_HARNESS)


def ref_run(cmd: str, case: dict, timeout: float = 600) -> dict:
    import json
    p = subprocess.run([REF_HARNESS, cmd], input=json.dumps(case).encode(), capture_output=True,
                       timeout=timeout)
    if p.returncode != 0:
        raise RuntimeError(f"ref_harness {cmd} failed: {p.stderr.decode()[-500:]}")
    return json.loads(p.stdout)


# ------------------------------------------------ uniform (T5) balancer
def balance_uniform_items(counts):
    """balance_uniform_items (balancer.cpp:411-448): final counts differ by at
    most one, the +1 slots go to the largest counts (std::stable_sort by
    count desc, ties toward the lower rank), surpluses paired with deficits
    in rank order.  Returns (final_counts, moves[(src, dst, count)], total)."""
    n = len(counts)
    if n == 0:
        return [], [], 0
    if any(c < 0 for c in counts):
        raise ValueError("balance_uniform_items: negative count")
    total = sum(counts)
    base, rem = divmod(total, n)
    order = sorted(range(n), key=lambda r: -counts[r])  # Python's sort is stable
    final = [base] * n
    for i in range(rem):
        final[order[i]] += 1
    surplus = [[r, counts[r] - final[r]] for r in range(n) if counts[r] > final[r]]
    deficit = [[r, final[r] - counts[r]] for r in range(n) if counts[r] < final[r]]
    moves, moved, si, di = [], 0, 0, 0
    while si < len(surplus) and di < len(deficit):
        m = min(surplus[si][1], deficit[di][1])
        moves.append((surplus[si][0], deficit[di][0], m))
        moved += m
        surplus[si][1] -= m
        deficit[di][1] -= m
        if surplus[si][1] == 0:
            si += 1
        if deficit[di][1] == 0:
            di += 1
    return final, moves, moved


def reverse_uniform_plan(moves):
    """reverse_uniform_plan (balancer.cpp:450-460): every move reversed, same order."""
    return [(d, s, c) for s, d, c in moves]


def uniform_item_layout(counts, final, moves):
    """Item placement realised by sb_uniform_route (our documented layout;
    the reference defines counts and moves only): rank r keeps its first
    min(count, final) items; a surplus rank's trailing items leave in move
    order; a deficit rank appends received items in move order.  Returns,
    per destination rank, the (origin rank, origin item index) list."""
    out = [[(r, i) for i in range(min(counts[r], final[r]))] for r in range(len(counts))]
    sent = [0] * len(counts)
    for s, d, c in moves:
        for k in range(c):
            out[d].append((s, final[s] + sent[s] + k))
        sent[s] += c
    return out
