mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "rc=$?" >> gpurun_out/gputest.log
timeout 300 python bench.py > gpurun_out/bench_c2.jsonl 2> gpurun_out/bench_c2.err
timeout 300 python bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_c2_2p.jsonl 2> gpurun_out/bench_c2_2p.err
timeout 300 python bench.py --config c3 --no-cpu-baseline > gpurun_out/bench_c3.jsonl 2> gpurun_out/bench_c3.err
timeout 300 python bench.py --config c1 --no-cpu-baseline > gpurun_out/bench_c1.jsonl 2> gpurun_out/bench_c1.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.jsonl 2> gpurun_out/bench_ref.err
tail -3 gpurun_out/gputest.log
