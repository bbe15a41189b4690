"""Build recipe for the in-tree native libraries (sm_100a only).

    python -m paper_2508_06001_b200._build

produces paper_2508_06001_b200/lib/libseqbal_cuda.so (CUDA kernels + C-ABI)
and paper_2508_06001_b200/lib/libseqbal.so (the C++ host API mirroring the
reference headers, linked against libseqbal_cuda.so).  nvcc cross-compiles
without a GPU, so this runs on the CPU build box too.
"""
from __future__ import annotations

import concurrent.futures
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib")
INCLUDE = os.path.join(ROOT, "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
              "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]
CUDA_SOURCES = ["planner.cu", "exchange.cu", "peer.cu", "stream.cu"]
HOST_SOURCES = ["host/seqbal_api.cpp", "host/plan_json.cpp", "host/seqbal_ext.cpp"]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libseqbal_cuda.so")


def _cxx() -> str:
    return "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _deps(sources):
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h"))]
    hdrs += [os.path.join(INCLUDE, "seqbal_capi.h"), os.path.join(CSRC, "host", "pow10_table.inc")]
    seqbal_inc = os.path.join(INCLUDE, "seqbal")
    if os.path.isdir(seqbal_inc):
        hdrs += [os.path.join(seqbal_inc, f) for f in os.listdir(seqbal_inc)]
    return sources + hdrs + [os.path.abspath(__file__)]  # flag changes rebuild too


def build(verbose: bool = False, force: bool = False) -> dict:
    os.makedirs(LIB, exist_ok=True)
    out = {}
    cuda_so = os.path.join(LIB, "libseqbal_cuda.so")
    srcs = [os.path.join(CSRC, s) for s in CUDA_SOURCES]
    if force or _stale(cuda_so, _deps(srcs)):
        # whole-program compilation per source (no -rdc: relocatable device
        # code cost the greedy chain ~40 % on sm_100a, 140 vs 102 cycles per
        # step, tools/micro/greedy_prod.cu); the sources share no device symbols
        extra = os.environ.get("SEQBAL_NVCC_DEFINES", "").split()  # diagnostics builds (-D...)
        objs, cmds = [], []
        for s in srcs:
            o = os.path.join(LIB, os.path.basename(s) + ".o")
            cmds.append([_nvcc(), *ARCH, *NVCC_FLAGS, *extra, "-I", INCLUDE, "-I", CSRC, "-c", s, "-o", o])
            objs.append(o)
        if verbose:
            for cmd in cmds:
                print(" ".join(cmd))
        with concurrent.futures.ThreadPoolExecutor(max_workers=len(cmds)) as ex:
            for f in [ex.submit(subprocess.run, cmd, check=True) for cmd in cmds]:
                f.result()
        cmd = [_nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", cuda_so, *objs]
        subprocess.run(cmd, check=True)
        for o in objs:
            os.remove(o)
    out["cuda"] = cuda_so
    host_srcs = [os.path.join(CSRC, s) for s in HOST_SOURCES if os.path.exists(os.path.join(CSRC, s))]
    if host_srcs:
        host_so = os.path.join(LIB, "libseqbal.so")
        if force or _stale(host_so, _deps(host_srcs) + [cuda_so]):
            cmd = [_cxx(), "-std=c++20", "-O2", "-fPIC", "-shared", "-I", INCLUDE, "-I", os.path.join(CSRC, "host"),
                   *host_srcs, "-o", host_so,
                   "-L", LIB, "-lseqbal_cuda", "-Wl,-rpath,$ORIGIN"]
            if verbose:
                print(" ".join(cmd))
            subprocess.run(cmd, check=True)
        out["host"] = host_so
        cli_src = os.path.join(CSRC, "host", "seqbal_cli.cpp")
        cli = os.path.join(LIB, "seqbal")
        if force or _stale(cli, [cli_src, host_so] + _deps([])):
            cmd = [_cxx(), "-std=c++20", "-O2", "-I", INCLUDE, cli_src, "-o", cli, "-L", LIB, "-lseqbal",
                   "-lseqbal_cuda", "-Wl,-rpath,$ORIGIN"]
            if verbose:
                print(" ".join(cmd))
            subprocess.run(cmd, check=True)
        out["cli"] = cli
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
