mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/gputest_full.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_full.log
tail -3 gpurun_out/gputest_full.log
timeout 300 python bench.py > gpurun_out/bench_c2.jsonl 2> gpurun_out/bench_c2.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_c2_ref.jsonl 2> gpurun_out/bench_c2_ref.err
timeout 300 python bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/bench_c2_2p.jsonl 2> gpurun_out/bench_c2_2p.err
timeout 300 python bench.py --gpus 2 --steps 10 --warmup 3 --config c3 > gpurun_out/bench_c3_2p.jsonl 2> gpurun_out/bench_c3_2p.err
python tools/summ.py gpurun_out/bench_c2.jsonl gpurun_out/bench_c2_2p.jsonl gpurun_out/bench_c3_2p.jsonl
tail -5 gpurun_out/bench_c2_2p.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/smoke.txt
