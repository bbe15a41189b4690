# fused planner with the cluster greedy helper: parity, traces, path comparison (and helper off)
mkdir -p gpurun_out
timeout 300 python tools/trace_planner.py c1 g1n8 small 2>&1 | tail -4; echo "trace rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider > gpurun_out/gputest_parity.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_parity.log
tail -3 gpurun_out/gputest_parity.log
for c in "c1 g1n8 small" "c1:512 g1n8 small" "c2"; do echo "== $c"; timeout 120 python tools/trace_planner.py $c 2>&1 | grep -E "total|greedy chain"; done
timeout 600 python tools/path_compare.py
echo "== helper off"
SEQBAL_PLAN_HELPER=0 timeout 600 python tools/path_compare.py
