mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pipeline.py -q -x -p no:cacheprovider > gpurun_out/gputest_pipe.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_pipe.log
bash tools/sanitize.sh
tail -3 gpurun_out/gputest_pipe.log
cat gpurun_out/sanitize_summary.txt
