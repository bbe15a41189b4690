# full GPU suite + C2 / C4 bench + planner traces after the fused-planner restructure
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/gputest_full.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_full.log
tail -3 gpurun_out/gputest_full.log
for c in "c2" "c1" "c1 g2n4" "c1 g8n1"; do echo "== $c"; python tools/trace_planner.py $c; done > gpurun_out/trace.txt 2>&1
timeout 300 python bench.py > gpurun_out/bench_c2.jsonl 2> gpurun_out/bench_c2.err
python tools/summ.py gpurun_out/bench_c2.jsonl
python -c "import json; d=json.loads(open('gpurun_out/bench_c2.jsonl').readline()); print('plan_us', d['plan_us'], 'graph', d['plan_us_graph'], d['plan_breakdown_us'])"
timeout 600 python bench.py --config c4 > gpurun_out/bench_c4.jsonl 2> gpurun_out/bench_c4.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_c4.jsonl').readline())
for x in d['sweep']:
    print(x['sequences'], x['topology'], round(x['plan_us'],1), round(x['ref_plan_us'],1), round(x['speedup_vs_ref'],2))
PY
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/smoke.txt; tail -2 gpurun_out/smoke.txt
