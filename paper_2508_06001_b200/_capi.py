"""ctypes binding of libseqbal_cuda.so (include/seqbal_capi.h).

The library is built in-tree (``python -m paper_2508_06001_b200._build``);
loading fails loudly when it is missing -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")
CUDA_LIB = os.path.join(LIB_DIR, "libseqbal_cuda.so")

SB_OK, SB_ERR_CONFIG, SB_ERR_INTEGRITY, SB_ERR_PARSE, SB_ERR_CAPACITY, SB_ERR_CUDA, SB_ERR_COMM = range(7)


class SeqbalError(RuntimeError):
    """Base of the mapped reference exceptions (error.hpp)."""
    code = -1


class ConfigError(SeqbalError, ValueError):
    code = SB_ERR_CONFIG


class IntegrityError(SeqbalError):
    code = SB_ERR_INTEGRITY


class ParseError(SeqbalError, ValueError):
    code = SB_ERR_PARSE


class CapacityError(SeqbalError):
    code = SB_ERR_CAPACITY


class CudaError(SeqbalError):
    code = SB_ERR_CUDA


class CommError(SeqbalError):
    code = SB_ERR_COMM


_ERRORS = {c.code: c for c in (ConfigError, IntegrityError, ParseError, CapacityError, CudaError, CommError)}


class PlannerDesc(C.Structure):
    _fields_ = [("world_size", C.c_int), ("unit_size", C.c_int), ("n_bags", C.c_int),
                ("bag_offsets", C.c_void_p), ("bag_ranks", C.c_void_p), ("d_model", C.c_int),
                ("n_heads", C.c_int), ("d_head", C.c_int), ("n_blocks", C.c_int), ("gamma", C.c_double),
                ("k", C.c_double), ("max_seqs", C.c_int64)]


class PlanDev(C.Structure):
    _fields_ = [("world_size", C.c_int), ("max_chunks", C.c_int64)] + [
        (n, C.c_void_p) for n in ("n_chunks", "chunk_id", "chunk_index", "chunk_start", "chunk_end", "chunk_src",
                                  "chunk_dst", "chunk_src_row", "chunk_dst_row", "send_off", "send_idx",
                                  "recv_off", "recv_idx", "rev_recv_idx", "origin_rows", "target_rows",
                                  "per_gpu_workload", "per_bag_occupancy", "capacity_violations",
                                  "total_workload", "wir", "status")]


class PlanHost(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("chunk_id", "chunk_index", "chunk_start", "chunk_end", "chunk_src",
                                           "chunk_dst", "send_off", "send_idx", "recv_off", "recv_idx",
                                           "rev_recv_idx", "target_rows", "per_gpu_workload",
                                           "per_bag_occupancy")] + [
        ("capacity_violations", C.c_int32), ("total_workload", C.c_double), ("wir", C.c_double)]


class WorldDesc(C.Structure):
    _fields_ = [("world_size", C.c_int), ("n_local", C.c_int), ("first_local", C.c_int), ("n_heads", C.c_int),
                ("n_payload", C.c_int), ("n_aux", C.c_int), ("row_bytes", C.c_void_p),
                ("capacity_rows", C.c_int64), ("max_bag", C.c_int)]


_lib = None

_SIGS = {
    "sb_last_error": (C.c_char_p, []),
    "sb_abi_version": (C.c_int, []),
    "sb_kernel_launches": (C.c_int64, []),
    "sb_planner_create": (C.c_int, [C.c_void_p, C.c_void_p]),
    "sb_planner_destroy": (C.c_int, [C.c_void_p]),
    "sb_plan": (C.c_int, [C.c_void_p] * 5),
    "sb_plan_identity": (C.c_int, [C.c_void_p] * 5),
    "sb_plan_get": (C.c_int, [C.c_void_p, C.c_void_p]),
    "sb_plan_sizes": (C.c_int, [C.c_void_p] * 4),
    "sb_plan_download": (C.c_int, [C.c_void_p] * 3),
    "sb_planner_enable_timing": (C.c_int, [C.c_void_p, C.c_int]),
    "sb_planner_set_path": (C.c_int, [C.c_void_p, C.c_int]),
    "sb_planner_last_path": (C.c_int, [C.c_void_p, C.POINTER(C.c_int)]),
    "sb_planner_trace": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "sb_selftest_div": (C.c_int, [C.c_int64, C.c_uint64, C.c_void_p]),
    "sb_selftest_serial_sum": (C.c_int, [C.c_int64, C.c_int64, C.c_uint64, C.c_int, C.c_void_p]),
    "sb_planner_timing": (C.c_int, [C.c_void_p] * 6),
    "sb_world_create": (C.c_int, [C.c_void_p, C.c_void_p]),
    "sb_world_destroy": (C.c_int, [C.c_void_p]),
    "sb_world_arena": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]),
    "sb_world_tables": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sb_world_set_peers": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int]),
    "sb_world_layout_origin": (C.c_int, [C.c_void_p] * 4),
    "sb_world_fill_witness": (C.c_int, [C.c_void_p] * 5),
    "sb_world_perturb": (C.c_int, [C.c_void_p] * 2),
    "sb_world_checksum": (C.c_int, [C.c_void_p] * 3),
    "sb_route": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sb_pre_attn": (C.c_int, [C.c_void_p] * 4),
    "sb_post_attn": (C.c_int, [C.c_void_p] * 4),
    "sb_exchange_prepare": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    "sb_exchange_run": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "sb_exchange_pack": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                   C.c_int64, C.c_void_p, C.c_void_p]),
    "sb_exchange_unpack": (C.c_int, [C.c_void_p, C.c_void_p]),
    "sb_world_status": (C.c_int, [C.c_void_p] * 2),
    "sb_world_upload": (C.c_int, [C.c_void_p] * 4),
    "sb_world_download": (C.c_int, [C.c_void_p] * 4),
    "sb_world_read_rank": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "sb_world_write_rank": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_void_p]),
    "sb_world_shape": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sb_last_exchange_bytes": (C.c_int, [C.c_void_p] * 3),
    "sb_copy_timing": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]),
    "sb_copy_timing_reset": (C.c_int, [C.c_void_p]),
    "sb_ipc_export": (C.c_int, [C.c_void_p, C.c_void_p]),
    "sb_ipc_import": (C.c_int, [C.c_void_p, C.c_void_p]),
    "sb_ipc_close": (C.c_int, [C.c_void_p]),
    "sb_gather_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int64, C.c_void_p]),
    "sb_gather_destroy": (C.c_int, [C.c_void_p]),
    "sb_gather_buffer": (C.c_int, [C.c_void_p] * 3),
    "sb_gather_set_peers": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "sb_gather_push": (C.c_int, [C.c_void_p] * 5),
    "sb_gather_compact": (C.c_int, [C.c_void_p] * 5),
    "sb_gather_status": (C.c_int, [C.c_void_p] * 2),
    "sb_barrier_create": (C.c_int, [C.c_int, C.c_int, C.c_void_p]),
    "sb_barrier_destroy": (C.c_int, [C.c_void_p]),
    "sb_barrier_buffer": (C.c_int, [C.c_void_p] * 3),
    "sb_barrier_set_peers": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "sb_barrier_wait": (C.c_int, [C.c_void_p] * 2),
    "sb_barrier_set_timeout": (C.c_int, [C.c_void_p, C.c_double]),
    "sb_world_layout_plan": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    "sb_barrier_status": (C.c_int, [C.c_void_p] * 3),
    "sb_world_compare": (C.c_int, [C.c_void_p] * 4),
    "sb_world_fill_meta": (C.c_int, [C.c_void_p] * 5),
    "sb_scenario_create": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "sb_scenario_parse": (C.c_int, [C.c_char_p, C.c_void_p]),
    "sb_scenario_preset": (C.c_int, [C.c_char_p, C.c_void_p]),
    "sb_scenario_destroy": (C.c_int, [C.c_void_p]),
    "sb_scenario_info": (C.c_int, [C.c_void_p] * 4),
    "sb_schedule_create": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_void_p]),
    "sb_schedule_destroy": (C.c_int, [C.c_void_p]),
    "sb_schedule_bounds": (C.c_int, [C.c_void_p] * 3),
    "sb_schedule_generate": (C.c_int, [C.c_void_p, C.c_int64] + [C.c_void_p] * 5),
    "sb_driver_create": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int64, C.c_int, C.c_int64, C.c_void_p]),
    "sb_driver_destroy": (C.c_int, [C.c_void_p]),
    "sb_driver_set_step": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p]),
    "sb_driver_step": (C.c_int, [C.c_void_p] * 2),
    "sb_driver_run": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p]),
    "sb_driver_progress": (C.c_int, [C.c_void_p] * 5),
    "sb_driver_records": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "sb_driver_world": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "sb_driver_set_pipeline": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "sb_driver_meta": (C.c_int, [C.c_void_p] * 4),
    "sb_uniform_create": (C.c_int, [C.c_int, C.c_void_p]),
    "sb_uniform_destroy": (C.c_int, [C.c_void_p]),
    "sb_uniform_plan": (C.c_int, [C.c_void_p] * 3),
    "sb_uniform_download": (C.c_int, [C.c_void_p] * 6),
    "sb_uniform_route": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
}


class StepRecord(C.Structure):
    """sb_step_record (include/seqbal_capi.h)."""
    _fields_ = [("step", C.c_int64), ("tokens", C.c_int64), ("sequences", C.c_int64), ("chunks", C.c_int64),
                ("wir", C.c_double), ("max_over_mean", C.c_double), ("total_workload", C.c_double),
                ("checksum", C.c_uint64), ("scenario", C.c_int32), ("capacity_violations", C.c_int32),
                ("checks", C.c_int32), ("verified", C.c_int32)]


SB_CHECK_ALL = 15


def exported_symbols() -> list[str]:
    return list(_SIGS)


def load(path: str | None = None):
    """Load libseqbal_cuda.so (no GPU needed to load; calls need one)."""
    global _lib
    if _lib is None:
        p = path or CUDA_LIB
        if not os.path.exists(p):
            raise RuntimeError(
                f"{p} is missing: build it with `python -m paper_2508_06001_b200._build` "
                "(there is no CPU fallback for the redistribute path)")
        L = C.CDLL(p)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status: int, what: str = "") -> None:
    if status != SB_OK:
        msg = load().sb_last_error().decode(errors="replace")
        cls = _ERRORS.get(status, SeqbalError)
        raise cls(f"{what}: {msg}" if what else msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
