"""The C++ drop-in API (include/seqbal/seqbal.hpp, lib/libseqbal.so) exercised
by a compiled test program modelled on the reference's own GTest suites
(tests/cpp/test_api.cpp).  Compiling is a CPU test; running needs the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_api.cpp")
LIB = os.path.join(ROOT, "paper_2508_06001_b200", "lib")
BIN = os.path.join(ROOT, "tests", "cpp", "test_api")


def build_test_binary():
    from paper_2508_06001_b200 import _build
    _build.build()
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    cmd = [cxx, "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), SRC,
           os.path.join(ROOT, "oracle", "seqbal_oracle.c"), "-x", "none", "-o", BIN, "-L", LIB, "-lseqbal",
           "-lseqbal_cuda", f"-Wl,-rpath,{LIB}"]
    # the oracle is C; compile it separately to keep C semantics
    obj = BIN + "_oracle.o"
    gcc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
    subprocess.run([gcc, "-std=c11", "-O2", "-ffp-contract=off", "-c", os.path.join(ROOT, "oracle", "seqbal_oracle.c"),
                    "-o", obj], check=True)
    cmd[cmd.index(os.path.join(ROOT, "oracle", "seqbal_oracle.c"))] = obj
    cmd.insert(cmd.index(obj) + 1, os.path.join(ROOT, "oracle", "stdsort_ref.cpp"))
    subprocess.run(cmd, check=True)
    return BIN


def test_cpp_api_compiles_against_headers():
    assert os.path.exists(build_test_binary())


@pytest.mark.gpu
def test_cpp_api_on_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    b = build_test_binary()
    p = subprocess.run([b], capture_output=True, text=True, timeout=600)
    print(p.stdout[-4000:])
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-2000:]
