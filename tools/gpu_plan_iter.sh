# fused-planner iteration: parity, per-phase traces, C2 + C4 plan latency
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider > gpurun_out/gputest_parity.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_parity.log
tail -4 gpurun_out/gputest_parity.log
for c in "c2" "c1" "c1 g2n4" "c1 g8n1"; do echo "== $c"; python tools/trace_planner.py $c; done > gpurun_out/trace.txt 2>&1
cat gpurun_out/trace.txt
timeout 300 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/bench_c2.jsonl 2> gpurun_out/bench_c2.err
python -c "import json; d=json.loads(open('gpurun_out/bench_c2.jsonl').readline()); print('C2 ms/step', d['ms_per_step'], 'plan_us', d['plan_us'], 'graph', d['plan_us_graph'], d['plan_breakdown_us'])"
timeout 600 python bench.py --config c4 > gpurun_out/bench_c4.jsonl 2> gpurun_out/bench_c4.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_c4.jsonl').readline())
for x in d['sweep']:
    if x['sequences'] <= 2048: print(x['sequences'], x['topology'], round(x['plan_us'],1), round(x['ref_plan_us'],1), round(x['speedup_vs_ref'],2))
PY
