"""Python host mirror of the reference plan/route/reverse API over the C-ABI.

Mirrors /root/reference/proj/include/seqbal/{balancer,exchange,topology}.hpp:
``parse_topology`` / ``Planner.plan`` (plan_routing) / ``Planner.plan_identity``
(identity_plan) / ``route`` / ``reverse_route`` / ``pre_attn`` / ``post_attn``.
Device memory and streams come from torch (plumbing only); every byte of
planning and data movement runs in libseqbal_cuda.so's sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _capi
from ._capi import ConfigError, ParseError, call

__all__ = ["Topology", "parse_topology", "Model", "Planner", "World", "DeviceMeta", "HostPlan",
           "route", "reverse_route", "pre_attn", "post_attn", "kernel_launches", "Scenario", "Schedule", "Driver",
           "UniformBalancer"]


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise _capi.CudaError("no CUDA device: the redistribute path runs only on the GPU")
    return torch


def _stream(stream):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def kernel_launches() -> int:
    return int(_capi.load().sb_kernel_launches())


def _destroy(fn, h):
    """Release a C-ABI handle from __del__; at interpreter shutdown the module
    globals may already be torn down, and the process exit frees the device."""
    try:
        getattr(_capi.load(), fn)(h)
    except (TypeError, AttributeError):
        pass


# ---------------------------------------------------------------- topology

@dataclass
class Topology:
    """topology.hpp:16-34: bags of contiguous unit-local ranks, textual order."""
    bag_sizes: list

    @property
    def unit_size(self) -> int:
        return sum(self.bag_sizes)

    def bag_ranks(self, b: int) -> list:
        s = sum(self.bag_sizes[:b])
        return list(range(s, s + self.bag_sizes[b]))

    def format(self) -> str:  # format_topology (topology.cpp:67-79)
        out, i = [], 0
        while i < len(self.bag_sizes):
            j = i
            while j < len(self.bag_sizes) and self.bag_sizes[j] == self.bag_sizes[i]:
                j += 1
            out.append(f"g{self.bag_sizes[i]}n{j - i}")
            i = j
        return "+".join(out)


def parse_topology(spec: str) -> Topology:
    """Grammar of topology.cpp:31-65: term ('+' term)*, term := 'g' INT 'n' INT."""
    if not spec:
        raise ParseError("empty topology spec (at offset 0)")
    terms, pos = [], 0

    def num(p, what):
        q, v = p, 0
        while q < len(spec) and "0" <= spec[q] <= "9":  # ASCII digits only, as parse_int
            v = v * 10 + ord(spec[q]) - 48
            if v > (1 << 20):
                raise ParseError(f"{what} value too large (at offset {p})")
            q += 1
        if q == p:
            raise ParseError(f"expected digits for {what} (at offset {p})")
        if v < 1:
            raise ParseError(f"{what} must be >= 1 (at offset {p})")
        return v, q

    while True:
        if pos >= len(spec) or spec[pos] != "g":
            raise ParseError(f"expected 'g' (at offset {pos})")
        g, pos = num(pos + 1, "bag size")
        if pos >= len(spec) or spec[pos] != "n":
            raise ParseError(f"expected 'n' (at offset {pos})")
        n, pos = num(pos + 1, "bag count")
        terms.append((g, n))
        if pos == len(spec):
            break
        if spec[pos] != "+":
            raise ParseError(f"expected '+' or end of spec (at offset {pos})")
        pos += 1
    sizes, unit = [], 0
    for g, n in terms:  # topology.cpp:51-62: the unit-size check runs after the whole spec parsed
        for _ in range(n):
            unit += g
            if unit > (1 << 20):
                raise ParseError("unit size too large (at offset 0)")
            sizes.append(g)
    return Topology(sizes)


@dataclass
class Model:
    """WorkloadModel (workload_model.hpp:13-42); FLUX defaults."""
    d_model: int = 3072
    n_heads: int = 24
    d_head: int = 128
    n_blocks: int = 57
    gamma: float = 0.49
    k: float = 4.0e-15


# ---------------------------------------------------------------- metadata
class DeviceMeta:
    """Gathered per-rank (sample_id, length) metadata resident in HBM
    (the all-gather result, gather order; exchange.cpp:68-77)."""

    def __init__(self, ids, lens, rank_off, device=None):
        torch = _torch()
        dev = device or torch.device("cuda", torch.cuda.current_device())
        # at least one element so empty worlds still pass valid device pointers
        n = len(ids)
        self.ids = torch.zeros(max(n, 1), dtype=torch.int64, device=dev)
        self.lens = torch.zeros(max(n, 1), dtype=torch.int64, device=dev)
        if n:
            self.ids[:n].copy_(torch.from_numpy(np.ascontiguousarray(np.asarray(ids, np.uint64).view(np.int64))))
            self.lens[:n].copy_(torch.from_numpy(np.ascontiguousarray(np.asarray(lens, np.int64))))
        self.rank_off = torch.as_tensor(np.asarray(rank_off, np.int64), device=dev)
        self.world = len(rank_off) - 1
        self.n = int(rank_off[-1])

    @classmethod
    def empty(cls, capacity: int, world: int, device=None):
        """Device buffers for up to `capacity` sequences over `world` ranks
        (filled by Schedule.generate)."""
        return cls(np.zeros(0, np.uint64), np.zeros(0, np.int64), np.zeros(world + 1, np.int64), device)._grow(
            capacity)

    def _grow(self, capacity):
        torch = _torch()
        n = max(capacity, 1)
        self.ids = torch.zeros(n, dtype=torch.int64, device=self.ids.device)
        self.lens = torch.zeros(n, dtype=torch.int64, device=self.lens.device)
        return self

    def to_lists(self):
        """(ids, lens) per rank, host numpy (synchronises)."""
        off = self.rank_off.cpu().numpy()
        ids = self.ids.cpu().numpy().view(np.uint64)
        lens = self.lens.cpu().numpy()
        return ([ids[off[r]:off[r + 1]].copy() for r in range(len(off) - 1)],
                [lens[off[r]:off[r + 1]].copy() for r in range(len(off) - 1)])

    @classmethod
    def from_lists(cls, ids_per_rank, lens_per_rank, device=None):
        ids = np.concatenate([np.asarray(x, np.uint64) for x in ids_per_rank]) if ids_per_rank else np.zeros(0, np.uint64)
        lens = np.concatenate([np.asarray(x, np.int64) for x in lens_per_rank]) if lens_per_rank else np.zeros(0, np.int64)
        off = np.zeros(len(ids_per_rank) + 1, np.int64)
        off[1:] = np.cumsum([len(x) for x in ids_per_rank])
        return cls(ids, lens, off, device)

    def ptrs(self):
        return (C.c_void_p(self.ids.data_ptr()), C.c_void_p(self.lens.data_ptr()),
                C.c_void_p(self.rank_off.data_ptr()))


@dataclass
class HostPlan:
    """RoutingPlan + BalanceReport downloaded from the device (balancer.hpp:38-89)."""
    world: int
    c_id: np.ndarray
    c_idx: np.ndarray
    c_start: np.ndarray
    c_end: np.ndarray
    c_src: np.ndarray
    c_dst: np.ndarray
    send_off: np.ndarray
    send_idx: np.ndarray
    recv_off: np.ndarray
    recv_idx: np.ndarray
    rev_recv_idx: np.ndarray
    target_rows: np.ndarray
    per_gpu_workload: np.ndarray
    per_bag_occupancy: np.ndarray
    capacity_violations: int
    total_workload: float
    wir: float

    @property
    def n_chunks(self) -> int:
        return len(self.c_id)

    def _lists(self, off, idx):
        return [idx[off[r]:off[r + 1]].astype(np.int64).tolist() for r in range(self.world)]

    @property
    def send(self):
        return self._lists(self.send_off, self.send_idx)

    @property
    def recv(self):
        return self._lists(self.recv_off, self.recv_idx)

    @property
    def rev_send(self):  # reverse_plan(plan).send == plan.recv (balancer.cpp:256-258)
        return self.recv

    @property
    def rev_recv(self):
        return self._lists(self.send_off, self.rev_recv_idx)


# ----------------------------------------------------------------- planner
class Planner:
    """Device planner for one (model, topology, world): plan_routing on the GPU."""

    def __init__(self, topology, world_size: int, model: Model | None = None, max_seqs: int = 1 << 16):
        _torch()
        self.topology = parse_topology(topology) if isinstance(topology, str) else (
            topology if isinstance(topology, Topology) else Topology(list(topology)))
        self.model = model or Model()
        self.world_size = world_size
        self.max_seqs = max_seqs
        sizes = self.topology.bag_sizes
        self._bag_off = np.zeros(len(sizes) + 1, np.int32)
        self._bag_off[1:] = np.cumsum(sizes)
        self._bag_ranks = np.arange(self.topology.unit_size, dtype=np.int32)
        d = _capi.PlannerDesc(world_size, self.topology.unit_size, len(sizes),
                              self._bag_off.ctypes.data, self._bag_ranks.ctypes.data, self.model.d_model,
                              self.model.n_heads, self.model.d_head, self.model.n_blocks, self.model.gamma,
                              self.model.k, max_seqs)
        h = C.c_void_p()
        call("sb_planner_create", C.byref(d), C.byref(h))
        self._h = h
        self.replicas = world_size // self.topology.unit_size
        self.max_bag = max(sizes)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _destroy("sb_planner_destroy", h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def plan(self, meta: DeviceMeta, stream=None):
        call("sb_plan", self._h, *meta.ptrs(), _stream(stream))
        self._meta = meta
        return self

    def plan_identity(self, meta: DeviceMeta, stream=None):
        call("sb_plan_identity", self._h, *meta.ptrs(), _stream(stream))
        self._meta = meta
        return self

    ROUTE, REVERSE, PRE_ATTN, POST_ATTN = 0, 1, 2, 3

    def prepare(self, op: int, src: "World", dst: "World", slot: int, stream=None):
        """Prepare an exchange (layout + copy jobs) into a slot; see sb_exchange_prepare."""
        call("sb_exchange_prepare", self._h, op, src.handle, dst.handle, slot, _stream(stream))

    def run(self, slot: int, stream=None):
        """Launch the copy of a prepared slot."""
        call("sb_exchange_run", self._h, slot, _stream(stream))

    def set_path(self, path: str):
        """'auto' | 'small' (fused single-CTA planner) | 'large' (multi-kernel) |
        'hybrid' (fused prefix with the greedy or the 32-thread greedy kernel, fused suffix)."""
        call("sb_planner_set_path", self._h, {"auto": 0, "small": 1, "large": 2, "hybrid": 3}[path])

    def last_path(self) -> str:
        """Which pipeline the last plan ran ('small', 'large', 'hybrid'; '' before any)."""
        v = C.c_int()
        call("sb_planner_last_path", self._h, C.byref(v))
        return {0: "", 1: "small", 2: "large", 3: "hybrid"}[v.value]

    def trace(self, enable: bool = True):
        """Per-phase clock64 deltas of the fused planner's last run (diagnostics)."""
        out = np.zeros(16, np.int64)
        call("sb_planner_trace", self._h, int(enable), out.ctypes.data)
        return out

    def enable_timing(self, on: bool = True):
        call("sb_planner_enable_timing", self._h, int(on))

    def timing(self) -> dict:
        v = [C.c_double() for _ in range(5)]
        call("sb_planner_timing", self._h, *[C.byref(x) for x in v])
        return dict(zip(["prep_us", "sort_us", "greedy_us", "emit_us", "lists_us"], [x.value for x in v]))

    def sizes(self, stream=None):
        nc, ns = C.c_int64(), C.c_int64()
        call("sb_plan_sizes", self._h, _stream(stream), C.byref(nc), C.byref(ns))
        return nc.value, ns.value

    def device_view(self) -> _capi.PlanDev:
        v = _capi.PlanDev()
        call("sb_plan_get", self._h, C.byref(v))
        return v

    def host_buffers(self, pinned: bool = True) -> dict:
        """Caller-owned host arrays for ``download(out=...)``, sized for the
        planner's capacity; pinned (page-locked) so the device copies run
        asynchronously at PCIe speed.  Reused by every download into them."""
        torch = _torch()
        W = self.world_size
        nc = int(self.max_seqs) * int(self.max_bag)  # every sequence splits into at most max_bag chunks
        nb = self.replicas * len(self.topology.bag_sizes)
        spec = dict(c_id=(nc, torch.int64, np.uint64), c_idx=(nc, torch.int32, None),
                    c_start=(nc, torch.int64, None), c_end=(nc, torch.int64, None), c_src=(nc, torch.int32, None),
                    c_dst=(nc, torch.int32, None), send_off=(W + 1, torch.int64, None),
                    send_idx=(nc, torch.int32, None), recv_off=(W + 1, torch.int64, None),
                    recv_idx=(nc, torch.int32, None), rev_recv_idx=(nc, torch.int32, None),
                    target_rows=(W, torch.int64, None), per_gpu_workload=(W, torch.float64, None),
                    per_bag_occupancy=(nb, torch.float64, None))
        out = {}
        for k, (n, dt, view) in spec.items():
            a = torch.empty(max(1, n), dtype=dt, pin_memory=pinned).numpy()
            out[k] = a.view(view) if view is not None else a
        return out

    def download(self, stream=None, out: dict | None = None) -> HostPlan:
        """The plan in host arrays (sb_plan_download).  ``out``: buffers from
        host_buffers() to download into (the returned plan views them)."""
        nc, _ = self.sizes(stream)
        W = self.world_size
        nb = self.replicas * len(self.topology.bag_sizes)
        if out is None:
            a = dict(c_id=np.zeros(nc, np.uint64), c_idx=np.zeros(nc, np.int32), c_start=np.zeros(nc, np.int64),
                     c_end=np.zeros(nc, np.int64), c_src=np.zeros(nc, np.int32), c_dst=np.zeros(nc, np.int32),
                     send_off=np.zeros(W + 1, np.int64), send_idx=np.zeros(nc, np.int32),
                     recv_off=np.zeros(W + 1, np.int64), recv_idx=np.zeros(nc, np.int32),
                     rev_recv_idx=np.zeros(nc, np.int32), target_rows=np.zeros(W, np.int64),
                     per_gpu_workload=np.zeros(W, np.float64), per_bag_occupancy=np.zeros(nb, np.float64))
        else:
            if nc > len(out["c_id"]):
                raise _capi.CapacityError("download: plan larger than the host buffers")
            lens = dict(send_off=W + 1, recv_off=W + 1, target_rows=W, per_gpu_workload=W, per_bag_occupancy=nb)
            a = {k: v[:lens.get(k, nc)] for k, v in out.items()}
        h = _capi.PlanHost(*[x.ctypes.data for x in a.values()])
        call("sb_plan_download", self._h, C.byref(h), _stream(stream))
        return HostPlan(W, *a.values(), capacity_violations=int(h.capacity_violations),
                        total_workload=float(h.total_workload), wir=float(h.wir))

    def copy_timing(self, op: int = -1):
        """(count, total_us) of copy kernels recorded while timing was on."""
        n, us = C.c_int64(), C.c_double()
        call("sb_copy_timing", self._h, op, C.byref(n), C.byref(us))
        return n.value, us.value

    def copy_timing_reset(self):
        call("sb_copy_timing_reset", self._h)

    def exchange_bytes(self) -> int:
        r, w = C.c_int64(), C.c_int64()
        call("sb_last_exchange_bytes", self._h, C.byref(r), C.byref(w))
        return r.value


# ------------------------------------------------------------------- world
class World:
    """Device-resident rank buffers (RankBuffer/World, exchange.hpp:22-44).

    Tensor 0 is the 16-byte row metadata {sample_id, position}; tensors
    1..n_payload are head-sliced payloads of ``payload_row_bytes[i]`` bytes per
    row; aux tensors are whole-row extras (e.g. RoPE position ids)."""

    def __init__(self, world_size: int, n_heads: int, payload_row_bytes, capacity_rows: int,
                 aux_row_bytes=(), n_local: int | None = None, first_local: int = 0, max_bag: int = 1):
        _torch()
        self.world_size = world_size
        self.n_local = n_local or world_size
        self.first_local = first_local
        self.n_payload = len(payload_row_bytes)
        self.n_aux = len(aux_row_bytes)
        self.row_bytes = [16] + list(payload_row_bytes) + list(aux_row_bytes)
        rb = np.asarray(list(payload_row_bytes) + list(aux_row_bytes), np.int64)
        d = _capi.WorldDesc(world_size, self.n_local, first_local, n_heads, self.n_payload, self.n_aux,
                            rb.ctypes.data, capacity_rows, max_bag)
        h = C.c_void_p()
        call("sb_world_create", C.byref(d), C.byref(h))
        self._h = h
        self.n_heads = n_heads
        self.T = 1 + self.n_payload + self.n_aux

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and getattr(self, "_owned", True):
            _destroy("sb_world_destroy", h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def arena(self, t: int):
        base, nbytes = C.c_void_p(), C.c_int64()
        call("sb_world_arena", self._h, t, C.byref(base), C.byref(nbytes))
        return base.value, nbytes.value

    def set_peers(self, t: int, bases):
        a = np.asarray(bases, np.uint64)
        call("sb_world_set_peers", self._h, t, a.ctypes.data, len(a))

    def layout_origin(self, meta: DeviceMeta, stream=None):
        _, lens, off = meta.ptrs()
        call("sb_world_layout_origin", self._h, lens, off, _stream(stream))

    ORIGIN, TARGET, ULYSSES = 0, 1, 2

    def layout_plan(self, planner: "Planner", layout: int, stream=None):
        """Per-rank layout from the planner's current plan without moving
        data (sb_world_layout_plan): ORIGIN, TARGET (chunk packing, what
        route writes) or ULYSSES (what pre_attn writes).  For q/k/v produced
        in the chunk layout or an attention output in the Ulysses layout."""
        call("sb_world_layout_plan", self._h, planner.handle, int(layout), _stream(stream))
        return self

    def fill_witness(self, meta: DeviceMeta, stream=None):
        call("sb_world_fill_witness", self._h, *meta.ptrs(), _stream(stream))

    def fill_meta(self, meta: DeviceMeta, stream=None):
        """Row metadata only (sb_world_fill_meta); payload untouched."""
        call("sb_world_fill_meta", self._h, *meta.ptrs(), _stream(stream))

    def perturb(self, stream=None):
        call("sb_world_perturb", self._h, _stream(stream))

    def checksum(self, stream=None) -> int:
        torch = _torch()
        acc = torch.zeros(1, dtype=torch.int64, device="cuda")
        call("sb_world_checksum", self._h, C.c_void_p(acc.data_ptr()), _stream(stream))
        return int(acc.cpu().numpy().view(np.uint64)[0])

    def status(self, stream=None):
        call("sb_world_status", self._h, _stream(stream))

    def compare(self, other: "World", stream=None) -> int:
        """worlds_bitwise_equal (exchange.cpp:459-480): number of differing
        16-byte words (0 == bitwise equal)."""
        torch = _torch()
        acc = torch.zeros(1, dtype=torch.int64, device="cuda")
        call("sb_world_compare", self._h, other.handle, C.c_void_p(acc.data_ptr()), _stream(stream))
        return int(acc.item())

    def shape(self, t: int = 0, stream=None):
        W = self.world_size
        rows, pitch = np.zeros(W, np.int64), np.zeros(W, np.int64)
        call("sb_world_shape", self._h, t, rows.ctypes.data, pitch.ctypes.data, _stream(stream))
        return rows, pitch

    def read_rank(self, t: int, rank: int, stream=None) -> np.ndarray:
        n = C.c_int64()
        call("sb_world_read_rank", self._h, t, rank, None, 0, C.byref(n), _stream(stream))
        buf = np.zeros(n.value, np.uint8)
        call("sb_world_read_rank", self._h, t, rank, buf.ctypes.data, n.value, C.byref(n), _stream(stream))
        return buf

    def write_rank(self, t: int, rank: int, data: np.ndarray, stream=None):
        data = np.ascontiguousarray(data).view(np.uint8)
        call("sb_world_write_rank", self._h, t, rank, data.ctypes.data, data.nbytes, _stream(stream))

    def upload(self, host_ptrs, nbytes, stream=None):
        p = (C.c_void_p * self.T)(*host_ptrs)
        b = np.asarray(nbytes, np.int64)
        call("sb_world_upload", self._h, p, b.ctypes.data, _stream(stream))

    def download(self, host_ptrs, nbytes, stream=None):
        p = (C.c_void_p * self.T)(*host_ptrs)
        b = np.asarray(nbytes, np.int64)
        call("sb_world_download", self._h, p, b.ctypes.data, _stream(stream))


# --------------------------------------------------------------- exchange
def route(planner: Planner, src: World, dst: World, stream=None, reverse: bool = False):
    """route (exchange.cpp:127-194): out-of-place, src (origin layout) -> dst."""
    call("sb_route", planner.handle, int(reverse), src.handle, dst.handle, _stream(stream))
    return dst


def reverse_route(planner: Planner, src: World, dst: World, stream=None):
    """reverse_route (exchange.cpp:196-198)."""
    return route(planner, src, dst, stream, reverse=True)


def pre_attn(planner: Planner, src: World, dst: World, stream=None):
    """pre_attn (exchange.cpp:255-331) for every multi-GPU bag at once."""
    call("sb_pre_attn", planner.handle, src.handle, dst.handle, _stream(stream))
    return dst


def post_attn(planner: Planner, src: World, dst: World, stream=None):
    """post_attn (exchange.cpp:333-436) for every multi-GPU bag at once."""
    call("sb_post_attn", planner.handle, src.handle, dst.handle, _stream(stream))
    return dst


# -------------------------------------------------- upstream generator
class Scenario:
    """ShardingGroupConfig (data_sim.hpp:46-51): data codes, a scenario file's
    text (parse_scenario) or a preset name.  Parsing is host-side and raises
    the reference's ParseError / ConfigError with its messages."""

    def __init__(self, codes=None, group_size: int = 0, text: str | None = None, preset: str | None = None):
        h = C.c_void_p()
        if preset is not None:
            call("sb_scenario_preset", preset.encode(), C.byref(h))
        elif text is not None:
            call("sb_scenario_parse", text.encode(), C.byref(h))
        else:
            enc = [c.encode() for c in (codes or [])]
            arr = (C.c_char_p * max(1, len(enc)))(*enc)
            call("sb_scenario_create", arr, len(enc), int(group_size), C.byref(h))
        self._h = h
        g, n = C.c_int(), C.c_int()
        call("sb_scenario_info", h, C.byref(g), C.byref(n), None)
        spec = np.zeros(5 * max(1, n.value), np.int32)
        call("sb_scenario_info", h, None, None, spec.ctypes.data)
        self.group_size = g.value
        self.streams = [tuple(int(x) for x in spec[5 * i:5 * i + 5]) for i in range(n.value)]

    def codes(self):
        return [f"g{g}b{b}i{r}f{f}s{s}" for g, b, r, f, s in self.streams]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _destroy("sb_scenario_destroy", h)
            self._h = None


class Schedule:
    """K scenarios on the device: step s draws every rank's batch from
    scenario s mod K (next_batch, data_sim.cpp:225-248) with one kernel."""

    def __init__(self, scenarios, world: int, seed: int):
        _torch()
        self.scenarios = [x if isinstance(x, Scenario) else Scenario(x) for x in scenarios]
        arr = (C.c_void_p * len(self.scenarios))(*[x._h.value for x in self.scenarios])
        h = C.c_void_p()
        call("sb_schedule_create", arr, len(self.scenarios), int(world), C.c_uint64(seed), C.byref(h))
        self._h = h
        self.world = world
        self.seed = seed
        ms, mr = C.c_int64(), C.c_int64()
        call("sb_schedule_bounds", h, C.byref(ms), C.byref(mr))
        self.max_seqs, self.max_rows = ms.value, mr.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _destroy("sb_schedule_destroy", h)
            self._h = None

    def generate(self, step: int, meta: DeviceMeta | None = None, stream=None) -> DeviceMeta:
        meta = meta or DeviceMeta.empty(self.max_seqs, self.world)
        ids, lens, off = meta.ptrs()
        call("sb_schedule_generate", self._h, int(step), None, ids, lens, off, _stream(stream))
        meta.n = None  # device-resident; see rank_off
        return meta


class Driver:
    """simulate_step (simulator.cpp:45-178) on the device path; one step =
    generate -> origin layout + witness -> plan -> route -> Ulysses pre/post
    -> reverse_route, with the reference's inline checks when verify."""

    def __init__(self, planner: Planner, schedule: Schedule, n_heads: int = 24, payload_row_bytes: int = 6144,
                 verify: bool = True, record_cap: int = 1024):
        h = C.c_void_p()
        call("sb_driver_create", planner.handle, schedule._h, int(n_heads), int(payload_row_bytes), int(verify),
             int(record_cap), C.byref(h))
        self._h = h
        self.planner, self.schedule = planner, schedule
        self.record_cap = record_cap

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _destroy("sb_driver_destroy", h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def set_step(self, step: int, stream=None):
        call("sb_driver_set_step", self._h, int(step), _stream(stream))

    def set_pipeline(self, on: bool = True, stream=None):
        """Plan-ahead schedule: step s+1 is generated, planned and prepared
        on a side stream under step s's copies (graphs: even step counts)."""
        call("sb_driver_set_pipeline", self._h, int(bool(on)), _stream(stream))

    def step(self, stream=None):
        call("sb_driver_step", self._h, _stream(stream))

    def run(self, n: int, stream=None):
        call("sb_driver_run", self._h, int(n), _stream(stream))

    def progress(self, stream=None):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        call("sb_driver_progress", self._h, C.byref(a), C.byref(b), C.byref(c), _stream(stream))
        return {"next_step": a.value, "steps_run": b.value, "failed": c.value}

    def records(self, stream=None):
        buf = (_capi.StepRecord * self.record_cap)()
        n = C.c_int64()
        call("sb_driver_records", self._h, buf, self.record_cap, C.byref(n), _stream(stream))
        return [{f: getattr(r, f) for f, _ in _capi.StepRecord._fields_} for r in buf]

    def world(self, which: int) -> "World":
        h = C.c_void_p()
        call("sb_driver_world", self._h, int(which), C.byref(h))
        w = World.__new__(World)  # borrowed handle: the driver owns and frees it
        w._h = h
        w._owned = False
        w._keep = self
        w.world_size = w.n_local = self.schedule.world
        w.first_local = 0
        w.T = 2
        return w


# ------------------------------------------------ uniform (T5) balancer
class UniformBalancer:
    """balance_uniform_items / reverse_uniform_plan (balancer.cpp:411-462) on
    the device, plus the item exchange (see sb_uniform_route)."""

    def __init__(self, world: int):
        _torch()
        h = C.c_void_p()
        call("sb_uniform_create", int(world), C.byref(h))
        self._h = h
        self.world = world

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _destroy("sb_uniform_destroy", h)
            self._h = None

    def plan(self, counts, stream=None):
        """counts: device int64 tensor [world] (or host sequence)."""
        torch = _torch()
        if not isinstance(counts, torch.Tensor):
            counts = torch.as_tensor(np.asarray(counts, np.int64), device="cuda")
        self._counts = counts
        call("sb_uniform_plan", self._h, C.c_void_p(counts.data_ptr()), _stream(stream))
        return self

    def download(self, stream=None):
        fin = np.zeros(self.world, np.int64)
        mv = np.zeros(3 * 2 * self.world, np.int64)
        n, tot = C.c_int64(), C.c_int64()
        call("sb_uniform_download", self._h, fin.ctypes.data, mv.ctypes.data, C.byref(n), C.byref(tot),
             _stream(stream))
        moves = [tuple(int(x) for x in mv[3 * i:3 * i + 3]) for i in range(n.value)]
        return {"final_counts": fin.tolist(), "moves": moves, "total_moved": tot.value}

    def route(self, src: World, dst: World, rows_per_item: int = 1, reverse: bool = False, stream=None):
        call("sb_uniform_route", self._h, int(reverse), int(rows_per_item), src.handle, dst.handle, _stream(stream))
        return dst
