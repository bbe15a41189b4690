# two-CTA fused planner: parity, traces, path comparison (pair on / off)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider > gpurun_out/gputest_parity.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_parity.log
tail -3 gpurun_out/gputest_parity.log
for c in "c1 g1n8 small" "c2"; do echo "== $c"; timeout 120 python tools/trace_planner.py $c 2>&1 | grep -E "total|greedy"; done
timeout 600 python tools/path_compare.py 2>&1 | head -5
echo "== pair off"
SEQBAL_PLAN_PAIR=0 timeout 600 python tools/path_compare.py 2>&1 | head -5
