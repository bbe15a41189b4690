# capacity <= 128 fused variant: parity, traces, C2 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider > gpurun_out/gputest_parity.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_parity.log
tail -3 gpurun_out/gputest_parity.log
for c in "c2 g1n8 small" "c2"; do echo "== $c"; python tools/trace_planner.py $c 2>&1; done
timeout 400 python bench.py > gpurun_out/bench_c2_smalln.jsonl 2> gpurun_out/bench_c2_smalln.err
python tools/summ.py gpurun_out/bench_c2_smalln.jsonl
python -c "
import json; l=json.loads(open('gpurun_out/bench_c2_smalln.jsonl').read().strip().splitlines()[-1]); print('plan_us', l['plan_us'], l['plan_us_graph'], l['plan_breakdown_us'])"
