"""B200-native balance-and-redistribute path of KnapFormer (arXiv 2508.06001).

Hot path: hand-written sm_100a CUDA in ``lib/libseqbal_cuda.so`` behind the
C-ABI in ``include/seqbal_capi.h``.  This package is the Python host mirror
(ctypes) used by the tests and the bench; the C++ host API mirroring the
reference headers lives in ``include/seqbal/*.hpp`` / ``lib/libseqbal.so``.
"""
from ._capi import (CapacityError, CommError, ConfigError, CudaError, IntegrityError, ParseError,  # noqa: F401
                    SeqbalError)
from .hostmem import pinned_host  # noqa: F401
from .api import (DeviceMeta, Driver, HostPlan, Model, Planner, Scenario, Schedule, Topology,  # noqa: F401
                  UniformBalancer, World, kernel_launches, parse_topology, post_attn, pre_attn, reverse_route, route)
