"""CPU-side checks of the C-ABI boundary: the library loads without a GPU,
exports every symbol include/seqbal_capi.h declares, and rejects bad
configurations with the reference's error classes before touching CUDA."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2508_06001_b200 import _capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "seqbal_capi.h")


def declared_symbols():
    with open(HEADER) as f:
        txt = f.read()
    return sorted(set(re.findall(r"^SB_API\s+[\w\s\*]+?\b(sb_\w+)\s*\(", txt, flags=re.M)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_capi.CUDA_LIB)
    syms = declared_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in seqbal_capi.h but not exported"
    # the ctypes mirror binds exactly the declared surface
    assert set(_capi.exported_symbols()) <= set(syms)


def test_abi_version_and_launch_counter():
    L = _capi.load()
    assert L.sb_abi_version() == 1
    assert L.sb_kernel_launches() >= 0


def _desc(world=8, topo_sizes=(1, 1, 1, 1, 2, 2), heads=24, d_model=3072, d_head=128, gamma=0.49, k=4e-15):
    sizes = list(topo_sizes)
    off = np.zeros(len(sizes) + 1, np.int32)
    off[1:] = np.cumsum(sizes)
    ranks = np.arange(sum(sizes), dtype=np.int32)
    d = _capi.PlannerDesc(world, int(sum(sizes)), len(sizes), off.ctypes.data, ranks.ctypes.data, d_model, heads,
                          d_head, 57, gamma, k, 64)
    return d, (off, ranks)


@pytest.mark.parametrize("kw,msg", [
    (dict(topo_sizes=(8,), heads=12, d_model=3072, d_head=256), "does not divide n_heads"),  # balancer.cpp:114-120
    (dict(world=12), "not a multiple of the sharding unit"),                                 # topology.cpp:86-91
    (dict(world=4), "smaller than the sharding unit"),                                       # topology.cpp:83-85
    (dict(gamma=0.0), "gamma must be positive"),                                             # workload_model.cpp:29
    (dict(k=-1.0), "k must be positive"),                                                    # workload_model.cpp:30
    (dict(d_head=100), "n_heads * d_head must equal d_model"),                               # workload_model.cpp:19-23
    (dict(topo_sizes=(5, 3)), "does not divide n_heads"),
])
def test_planner_config_errors(kw, msg):
    d, keep = _desc(**kw)
    h = C.c_void_p()
    st = _capi.load().sb_planner_create(C.byref(d), C.byref(h))
    assert st == _capi.SB_ERR_CONFIG
    assert msg in _capi.load().sb_last_error().decode()
    assert not h.value
    with pytest.raises(_capi.ConfigError):
        _capi.check(st)


def test_world_config_errors():
    rb = np.asarray([7], np.int64)  # not a multiple of n_heads=24
    d = _capi.WorldDesc(8, 8, 0, 24, 1, 0, rb.ctypes.data, 100, 1)
    h = C.c_void_p()
    st = _capi.load().sb_world_create(C.byref(d), C.byref(h))
    assert st == _capi.SB_ERR_CONFIG
    assert "multiple of n_heads" in _capi.load().sb_last_error().decode()
    d2 = _capi.WorldDesc(8, 3, 0, 24, 1, 0, rb.ctypes.data, 100, 1)  # 3 does not divide 8
    assert _capi.load().sb_world_create(C.byref(d2), C.byref(h)) == _capi.SB_ERR_CONFIG


def test_no_gpu_fails_loudly_not_silently():
    """A valid configuration needs device memory: without a GPU the call
    must fail with SB_ERR_CUDA (there is no CPU fallback)."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    d, keep = _desc()
    h = C.c_void_p()
    st = _capi.load().sb_planner_create(C.byref(d), C.byref(h))
    assert st == _capi.SB_ERR_CUDA
    import paper_2508_06001_b200 as sb
    with pytest.raises(sb.CudaError):
        sb.Planner("g1n8", 8)


def test_missing_library_is_loud(tmp_path):
    saved = _capi._lib
    try:
        _capi._lib = None
        with pytest.raises(RuntimeError, match="no CPU fallback"):
            _capi.load(str(tmp_path / "nope.so"))
    finally:
        _capi._lib = saved


def test_generator_driver_uniform_config_errors_without_gpu():
    """Argument validation of the §8(f) entry points runs before any CUDA
    call, with the reference's messages (simulator.cpp:15-21)."""
    L = _capi.load()
    codes = (C.c_char_p * 1)(b"g2b4i256f1s0")
    sc = C.c_void_p()
    assert L.sb_scenario_create(codes, 1, 0, C.byref(sc)) == _capi.SB_OK
    arr = (C.c_void_p * 1)(sc.value)
    sch = C.c_void_p()
    st = L.sb_schedule_create(arr, 1, 3, 7, C.byref(sch))  # world 3 not a multiple of group 2
    assert st == _capi.SB_ERR_CONFIG
    assert b"is not a multiple of the data sharding group 2" in L.sb_last_error()
    assert L.sb_schedule_create(arr, 0, 2, 7, C.byref(sch)) == _capi.SB_ERR_CONFIG
    L.sb_scenario_destroy(sc)
    d = C.c_void_p()
    assert L.sb_driver_create(None, None, 24, 6144, 1, 8, C.byref(d)) == _capi.SB_ERR_CONFIG
    u = C.c_void_p()
    assert L.sb_uniform_create(0, C.byref(u)) == _capi.SB_ERR_CONFIG
    assert L.sb_uniform_route(None, 0, 1, None, None, None) == _capi.SB_ERR_CONFIG
