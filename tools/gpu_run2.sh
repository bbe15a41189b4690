mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multiproc.py -q -m gpu -x -p no:cacheprovider > gpurun_out/gputest_mp.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_mp.log
SEQBAL_TRANSPORTS=staged timeout 300 python bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_c2_2p_staged.jsonl 2> gpurun_out/bench_c2_2p_staged.err
SEQBAL_TRANSPORTS=staged timeout 300 python bench.py --gpus 2 --steps 5 --warmup 3 --config c3 > gpurun_out/bench_c3_2p_staged.jsonl 2> gpurun_out/bench_c3_2p_staged.err
tail -3 gpurun_out/gputest_mp.log
