#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over a subset
# of the GPU parity tests covering every kernel family: fused single-CTA and
# multi-kernel planners (sorts, greedy, block serial sums, emission, lists,
# std::sort replay), the hybrid planner and the >64-bag greedy, exchange prep, LSU + TMA copy engines (mbarrier ring),
# Ulysses on q/k/v, the stream driver's plan-ahead slots, uniform balancer.
# Writes gpurun_out/sanitize_<tool>.log; summary in gpurun_out/sanitize_summary.txt
cd "$(dirname "$0")/.."
SEL_PARITY="rand07 or rand19 or c2_g1n4 or c3_g4n2 or empty_world or zero_len or c4_n4096_g2n4 or c4_n1024_g8n1"
TESTS=(
  "tests/test_gpu_parity.py -k ($SEL_PARITY) and device_plan"
  "tests/test_gpu_parity.py -k test_random_plans_vs_oracle or block_serial_sum or reverse_ties or many_bags or many_replicas"
  "tests/test_gpu_ulysses_qkv.py -k g4n2 or layout_plan"
  "tests/test_gpu_stream.py -k plan_ahead or graph_replay"
  "tests/test_uniform.py"
)
: > gpurun_out/sanitize_summary.txt
for tool in memcheck racecheck synccheck initcheck; do
  log=gpurun_out/sanitize_$tool.log
  : > $log
  for t in "${TESTS[@]}"; do
    file=${t%% -k *}; sel=""
    [[ "$t" == *" -k "* ]] && sel=${t#* -k }
    echo "### $tool: $file -k '$sel'" >> $log
    if [ -n "$sel" ]; then
      timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 \
        python -m pytest $file -q -x -p no:cacheprovider -k "$sel" >> $log 2>&1
    else
      timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 \
        python -m pytest $file -q -x -p no:cacheprovider -m gpu >> $log 2>&1
    fi
    echo "rc=$?" >> $log
  done
  echo "== $tool" >> gpurun_out/sanitize_summary.txt
  grep -E "^### |^rc=|ERROR SUMMARY|passed|failed" $log >> gpurun_out/sanitize_summary.txt
done
