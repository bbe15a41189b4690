"""Synthetic metadata streams for the bench (host-side input generation).

Restates the reference's deterministic generators so the bench feeds the
GPU path exactly the inputs the reference CPU path sees:
  * ``c1_batch``  -- SURVEY.md 8(d) C1 law: CounterRng({seed, step, rank}),
    text U[64,512] then image U[256,4096], ids make_sample_id(step, rank, i)
    (rng.hpp:30-55, data_sim.cpp:219-223);
  * ``next_batch`` -- data_sim.cpp:225-248 for g{G}b{B}i{R}f{F}s{S} streams.
Vectorised numpy uint64 arithmetic (wrapping multiply == C++ uint64_t).
"""
from __future__ import annotations

import math
import re

import numpy as np

_M64 = (1 << 64) - 1


def splitmix64(x):
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def derive_key(parts) -> int:
    k = np.uint64(0x8F51A7C0C0C0F5A3)
    for p in parts:
        k = splitmix64(k ^ np.uint64(p & _M64))
    return int(k)


def rng_u64(key: int, counters):
    return splitmix64(np.uint64(key) ^ splitmix64(np.asarray(counters, np.uint64)))


def rng_int(key: int, counters, lo: int, hi: int):
    """CounterRng::next_int (Lemire fixed-point multiply, exact 128-bit)."""
    span = (hi - lo) + 1
    draws = rng_u64(key, counters)
    return np.asarray([lo + ((int(d) * span) >> 64) for d in draws], np.int64)


def rng_real(key: int, counter: int, lo: float, hi: float) -> float:
    u = float(int(rng_u64(key, [counter])[0]) >> 11) * 2.0 ** -53
    return lo + u * (hi - lo)


def make_sample_id(step: int, rank: int, index):
    index = np.asarray(index, np.uint64)
    return (np.uint64((step << 32) & _M64) | np.uint64((rank & 0xFFFF) << 16) | (index & np.uint64(0xFFFF)))


def c1_batch(seed: int, step: int, rank: int, per_rank: int):
    key = derive_key([seed, step, rank])
    i = np.arange(per_rank, dtype=np.uint64)
    text = rng_int(key, 2 * i, 64, 512)
    image = rng_int(key, 2 * i + 1, 256, 4096)
    return make_sample_id(step, rank, i), (text + image).astype(np.int64)


_TEXT = 0x7465787421
_ASPECT = 0x6173706563


def parse_data_code(code: str):
    m = re.fullmatch(r"g(\d+)b(\d+)i(\d+)f(\d+)s([01])", code)
    if not m:
        raise ValueError(f"bad data code {code!r}")
    g, b, r, f, s = (int(x) for x in m.groups())
    if g < 1 or b < 1 or r < 1 or r % 16 or f < 1:
        raise ValueError(f"bad data code {code!r}")
    return g, b, r, f, s


def visual_tokens(res: int, frames: int, smooth: int, mult: float) -> int:
    side = res // 16
    scaled = _llround(float(side * side) * mult)
    latent = _llround(float(frames) * 5 / 17) if smooth else frames
    return max(1, scaled * latent)


def _llround(x: float) -> int:
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


def next_batch(codes, rank: int, step: int, seed: int):
    specs = [parse_data_code(c) for c in codes]
    group = sum(s[0] for s in specs)
    gr = rank % group
    cur, stream = 0, 0
    for i, s in enumerate(specs):
        cur += s[0]
        if gr < cur:
            stream = i
            break
    g, b, res, frames, smooth = specs[stream]
    mult = rng_real(derive_key([_ASPECT, seed, step, stream]), 0, 0.96, 1.04)
    key = derive_key([_TEXT, seed, step, rank])
    i = np.arange(b, dtype=np.uint64)
    text = rng_int(key, i, 0, 392)
    vis = visual_tokens(res, frames, smooth, mult)
    return make_sample_id(step, rank, i), (text + vis).astype(np.int64)


def metadata(kind: str, world: int, **kw):
    """Per-rank (ids, lens) lists for a bench config."""
    ids, lens = [], []
    for r in range(world):
        if kind == "c1":
            i, l = c1_batch(kw["seed"], kw["step"], r, kw["per_rank"])
        elif kind == "scenario":
            i, l = next_batch(kw["codes"], r, kw["step"], kw["seed"])
        else:
            raise ValueError(kind)
        ids.append(i)
        lens.append(l)
    return ids, lens
