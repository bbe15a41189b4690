"""Plan wire format (balancer.cpp:289-352) and the CLI `plan` subcommand
(tools/main.cpp:200-230) against the unmodified reference
(tests/golden/plan_json.json, tests/golden/make_json_golden.py):

  * CPU: our Grisu2 double printer equals nlohmann::json's text on 8 K
    doubles; plan_from_json -> plan_to_json reproduces every reference plan
    string byte for byte;
  * GPU: `seqbal plan` (device planner) prints exactly the reference CLI's
    output for every seq-lens case, and the same errors / exit codes."""
import ctypes as C
import json
import os
import struct
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2508_06001_b200", "lib")
with open(os.path.join(ROOT, "tests", "golden", "plan_json.json")) as f:
    GOLD = json.load(f)


@pytest.fixture(scope="module")
def host():
    from paper_2508_06001_b200 import _build
    _build.build()
    L = C.CDLL(os.path.join(LIB, "libseqbal.so"))
    L.sb_json_format_double.restype = C.c_size_t
    L.sb_json_format_double.argtypes = [C.c_double, C.c_char_p, C.c_size_t]
    L.sb_json_plan_roundtrip.restype = C.c_long
    L.sb_json_plan_roundtrip.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t]
    return L


def test_double_text_matches_nlohmann(host):
    buf = C.create_string_buffer(64)
    bad = []
    for hexbits, want in GOLD["dtoa"].items():
        x = struct.unpack("<d", struct.pack("<Q", int(hexbits, 16)))[0]
        n = host.sb_json_format_double(x, buf, 64)
        got = buf.value.decode()
        if got != want or n != len(want):
            bad.append((hexbits, got, want))
    assert not bad, bad[:10]
    assert len(GOLD["dtoa"]) > 8000


@pytest.mark.parametrize("i", [i for i, p in enumerate(GOLD["plans"]) if "json" in p])
def test_plan_json_round_trip_is_byte_identical(host, i):
    want = GOLD["plans"][i]["json"]
    out = C.create_string_buffer(len(want) * 2 + 1024)
    n = host.sb_json_plan_roundtrip(want.encode(), out, len(out))
    assert n == len(want), out.value.decode()[:300]
    assert out.value.decode() == want


def test_plan_from_json_rejects_bad_input(host):
    out = C.create_string_buffer(512)
    assert host.sb_json_plan_roundtrip(b'{"world_size":2,"chunks":[],"origins":[[]]}', out, 512) == -1
    assert "origins size does not match world_size" in out.value.decode()
    assert host.sb_json_plan_roundtrip(b'{"world_size":1,"chunks":[', out, 512) == -1
    assert "at offset" in out.value.decode()


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(len(GOLD["plans"])))
def test_cli_plan_matches_reference(tmp_path, i):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    case = GOLD["plans"][i]
    lens = tmp_path / "lens.json"
    lens.write_text("// per-rank lengths\n" + json.dumps(case["lens"]) + "\n")
    cmd = [os.path.join(LIB, "seqbal"), "plan", str(lens), "--topology", case["topology"]]
    for k, flag in (("d_model", "--d-model"), ("n_heads", "--n-heads"), ("gamma", "--gamma")):
        if k in case:
            cmd += [flag, repr(case[k])]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=120)
    if "json" in case:
        assert p.returncode == 0, p.stderr
        assert p.stdout == case["json"] + "\n"
    else:
        assert p.returncode == 1 and p.stderr.startswith("error:"), (p.returncode, p.stderr)
        assert p.stderr == f"error: {case['error']}\n", (p.stderr, case["error"])
