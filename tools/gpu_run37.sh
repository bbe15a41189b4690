# hybrid suffix as a programmatic dependent launch (prologue + duplicate check under the chain)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider > gpurun_out/gputest_parity.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_parity.log
tail -3 gpurun_out/gputest_parity.log
for c in "c1 g1n8 hybrid" "c1:512 g1n8 hybrid"; do echo "== $c"; timeout 120 python tools/trace_planner.py $c 2>&1; done
timeout 600 python tools/path_compare.py
timeout 600 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "test_random_plans_vs_oracle and hybrid" 2>&1 | grep -E "passed|failed|RACECHECK|ERROR" | tail -3
timeout 600 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "test_random_plans_vs_oracle and hybrid or duplicate" 2>&1 | grep -E "passed|failed|ERROR SUMMARY" | tail -3
