#!/bin/bash
# compute-sanitizer memcheck over every single-process GPU test file (the
# targeted racecheck / synccheck / initcheck subsets are in sanitize.sh).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/memcheck_full.log
for f in tests/test_gpu_parity.py tests/test_gpu_stream.py tests/test_gpu_ulysses_qkv.py tests/test_gpu_pipeline.py tests/test_uniform.py tests/test_cpp_api.py; do
  echo "### memcheck: $f" >> gpurun_out/memcheck_full.log
  timeout 2400 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 99 --target-processes all \
    python -m pytest $f -q -x -m gpu -p no:cacheprovider >> gpurun_out/memcheck_full.log 2>&1
  echo "rc=$?" >> gpurun_out/memcheck_full.log
done
grep -E "^###|passed|failed|ERROR SUMMARY|rc=" gpurun_out/memcheck_full.log
