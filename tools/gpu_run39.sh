# multi-kernel pipeline with programmatic dependent launches: parity, sanitizers, path comparison, C4
mkdir -p gpurun_out/r02p
O=gpurun_out/r02p
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stream.py -q -m gpu -x -p no:cacheprovider > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
tail -3 $O/gputest.log
timeout 600 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "test_random_plans_vs_oracle and large or c4_n4096_g2n4 or many_bags" 2>&1 | grep -E "passed|failed|RACECHECK|ERROR" | tail -3
timeout 600 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "test_random_plans_vs_oracle and large or c4_n4096_g2n4 or many_bags" 2>&1 | grep -E "passed|failed|ERROR SUMMARY" | tail -3
timeout 600 python tools/path_compare.py > $O/path_compare.txt 2>&1; cat $O/path_compare.txt
timeout 600 python bench.py --config c4 > $O/bench_c4.jsonl 2> $O/bench_c4.err
python - <<'PY'
import json
l=json.loads(open('gpurun_out/r02p/bench_c4.jsonl').read().strip().splitlines()[-1])
for r in l['sweep']:
    print(r['sequences'], r['topology'], r['path'], round(r['plan_us'],1), round(r['speedup_vs_ref'],2))
PY
