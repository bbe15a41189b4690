"""Scenario (sharding-group) definitions used by the stream driver and bench.

Data codes follow the reference grammar g{G}b{B}i{R}f{F}s{S}
(data_sim.cpp:39-76); presets mirror data_sim.cpp:152-165.  The C5 schedule
(SURVEY.md 8(d)): step s draws from scenario s mod K over three 8-GPU
scenario files (low-res images, mixed resolutions, joint image + video).
"""
from __future__ import annotations

PRESETS = {  # data_sim.cpp:152-165 (group_size 32)
    "lowres_image": ["g32b32i256f1s0"],
    "mixed_image": ["g16b4i256f1s0", "g4b5i512f1s0", "g4b5i1024f1s0", "g8b1i2048f1s0"],
    "joint_image_video": ["g8b4i256f1s0", "g2b5i512f1s0", "g2b5i1024f1s0", "g4b1i2048f1s0", "g1b10i256f4s0",
                          "g3b1i512f4s0", "g8b2i256f85s1", "g4b1i512f85s1"],
}

# C5: the three presets re-cut for one 8-GPU sharding group.
C5_SCENARIOS = [
    ["g8b32i256f1s0"],                                                   # lowres-8
    ["g4b4i256f1s0", "g1b5i512f1s0", "g1b5i1024f1s0", "g2b1i2048f1s0"],  # mixed-8
    ["g2b4i256f1s0", "g1b5i512f1s0", "g1b1i2048f1s0", "g1b10i256f4s0", "g1b1i512f4s0", "g1b2i256f85s1",
     "g1b1i512f85s1"],                                                   # joint-8 (image + video)
]
C5_WORLD = 8
C5_TOPOLOGY = "g1n2+g2n1+g4n1"  # bags of 1, 2 and 4 GPUs: Ulysses at two degrees
C5_SEED = 11
