"""Regenerate the plan wire-format fixtures from the UNMODIFIED reference
(oracle/_ref/ref_harness): tests/golden/plan_json.json holds

  * "dtoa": nlohmann::json's text for doubles (IEEE bits in hex) -- random
    bit patterns over the whole exponent range, workload-sized values,
    integers, powers of ten, subnormals, signed zeros, inf/nan;
  * "plans": the CLI `plan` output (plan_to_json, tools/main.cpp:200-230)
    for hand and random seq-lens files and topologies, or its error text.

    python tests/golden/make_json_golden.py
"""
from __future__ import annotations

import json
import os
import random
import struct
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def harness(cmd, payload):
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_harness")
    p = subprocess.run([exe, cmd], input=json.dumps(payload).encode(), capture_output=True, check=True)
    return json.loads(p.stdout)


def bits(x: float) -> str:
    return f"{struct.unpack('<Q', struct.pack('<d', x))[0]:016x}"


def main():
    rng = random.Random(6001)
    doubles = [bits(x) for x in (0.0, -0.0, 1.0, -1.0, 0.1, 0.5, 1e15, 1e16, 123456789012345.0, 1234567890123456.0,
                                 1e-4, 1e-5, 9.999999999999999e-5, 2.0 ** -1074, 2.0 ** -1022, 1.7976931348623157e308,
                                 float("inf"), float("-inf"), 5e-324, 3.0, 1.0 / 3, 2.0 / 3, 100.0, 1e21, 1e22)]
    doubles += [f"{rng.getrandbits(64):016x}" for _ in range(4000)]
    doubles += [bits(rng.uniform(0.5, 4.0)) for _ in range(1000)]                        # occupancies / WIRs
    doubles += [bits(24.0 * l * 3072 * 3072 + 0.49 * 4.0 * l * l * 3072) for l in rng.sample(range(1, 70000), 1000)]
    doubles += [bits(rng.uniform(1e9, 1e16)) for _ in range(1000)]                       # workloads and totals
    doubles += [bits(float(rng.randint(0, 10 ** rng.randint(1, 17)))) for _ in range(500)]
    doubles += [bits(10.0 ** e) for e in range(-320, 309)]
    dtoa = dict(zip(doubles, harness("dtoa", {"bits": doubles})))
    cases = [
        {"lens": [[10], []], "topology": "g2n1", "d_model": 64, "n_heads": 4},
        {"lens": [[100, 3], [57], [13, 13, 13], []], "topology": "g2n2", "d_model": 64, "n_heads": 4},
        {"lens": [[0, 3, 0], [], [], [], [], [], [], []], "topology": "g8n1", "d_model": 64, "n_heads": 8},
        {"lens": [[], []], "topology": "g1n2"},
        {"lens": [[4096, 77, 1], [512, 300], [1, 2, 3, 4], [9000]], "topology": "g1n2+g2n1"},
        {"lens": [[5, 5], [5, 5]], "topology": "g1n2", "gamma": 0.385},
        {"lens": [[10, 20], [30]], "topology": "g3n1"},                                   # error: world 2 < unit 3
        {"lens": [[10, -1], [3]], "topology": "g1n2"},                                    # error: negative length
        {"lens": [[10], [3]], "topology": "g2n1", "d_model": 60, "n_heads": 8},           # error: heads
    ]
    for t in range(40):
        topo = rng.choice(["g1n8", "g2n4", "g4n2", "g8n1", "g1n2+g2n1+g4n1", "g1n4+g2n2"])
        w = 8 * rng.choice([1, 1, 2])
        lens = [[rng.choice([rng.randint(0, 12), rng.randint(64, 4608), rng.randint(1, 70000)])
                 for _ in range(rng.randint(0, 12))] for _ in range(w)]
        cases.append({"lens": lens, "topology": topo, "gamma": rng.choice([0.49, 0.385, 0.7])})
    plans = harness("cli_plan", {"cases": cases})
    out = {"dtoa": dtoa, "plans": [dict(c, **p) for c, p in zip(cases, plans)]}
    with open(os.path.join(HERE, "plan_json.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote plan_json.json:", len(dtoa), "doubles,", len(plans), "plans")


if __name__ == "__main__":
    main()
