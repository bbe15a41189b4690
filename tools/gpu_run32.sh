# hybrid with the greedy in the prefix kernel (one replica): parity, traces, path comparison
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider > gpurun_out/gputest_parity.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_parity.log
tail -3 gpurun_out/gputest_parity.log
for c in "c1 g1n8 hybrid" "c1:512 g1n8 hybrid"; do echo "== $c"; timeout 120 python tools/trace_planner.py $c 2>&1; done
timeout 600 python tools/path_compare.py
