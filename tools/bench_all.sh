#!/bin/bash
# Every bench line of the round into gpurun_out/bench_*.jsonl (run under gpurun).
python bench.py > gpurun_out/bench_c2.jsonl 2> gpurun_out/bench_c2.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_c2_ref.jsonl 2>&1
python bench.py --config c1 --steps 50 > gpurun_out/bench_c1.jsonl 2> gpurun_out/bench_c1.err
python bench.py --config c3 --steps 50 > gpurun_out/bench_c3.jsonl 2> gpurun_out/bench_c3.err
python bench.py --config c3 --topology g8n1 --steps 50 > gpurun_out/bench_c3_g8n1.jsonl 2> gpurun_out/bench_c3_g8n1.err
python bench.py --config c4 --steps 30 > gpurun_out/bench_c4.jsonl 2> gpurun_out/bench_c4.err
python bench.py --config c5 > gpurun_out/bench_c5.jsonl 2> gpurun_out/bench_c5.err
python tools/pcie_probe.py > gpurun_out/pcie.txt 2>&1
python bench.py --config c5 --impl reference > gpurun_out/bench_c5_ref.jsonl 2>&1
python tools/bench_uniform.py > gpurun_out/bench_uniform.jsonl 2> gpurun_out/bench_uniform.err
