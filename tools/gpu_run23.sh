# fused planner: totals chain reads the sequence pass's workloads
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider > gpurun_out/gputest_parity.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_parity.log
tail -4 gpurun_out/gputest_parity.log
for c in "c1 g1n8 small" "c1:1024 g1n8 small" "c1:512 g1n8 small"; do echo "== $c"; python tools/trace_planner.py $c 2>&1 | grep -v "^  P"; done
python tools/path_compare.py
