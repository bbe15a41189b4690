mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multiproc.py -q -m gpu -x -p no:cacheprovider > gpurun_out/gputest_mp.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_mp.log
tail -3 gpurun_out/gputest_mp.log
timeout 300 python bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/bench_c2_2p.jsonl 2> gpurun_out/bench_c2_2p.err
timeout 300 python bench.py --gpus 2 --steps 10 --warmup 3 --config c3 > gpurun_out/bench_c3_2p.jsonl 2> gpurun_out/bench_c3_2p.err
python tools/summ.py gpurun_out/bench_c2_2p.jsonl gpurun_out/bench_c3_2p.jsonl
python -c "
import json
for f in ['gpurun_out/bench_c2_2p.jsonl','gpurun_out/bench_c3_2p.jsonl']:
    d=json.loads(open(f).readline()); print(f, d['launch_mode'], d['ms_per_step_eager'], d['ms_per_step_graph'], d['ms_per_step_plan_ahead'], d['pipeline_error'], d['graph_error'])
"
tail -5 gpurun_out/bench_c2_2p.err
