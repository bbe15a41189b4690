mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stream.py -q -x -p no:cacheprovider > gpurun_out/gputest_plan.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_plan.log
timeout 300 python tools/plan_profile.py c2 256 512 > gpurun_out/plan_profile.txt 2>&1
timeout 300 python bench.py --config c4 --steps 30 --warmup 10 > gpurun_out/bench_c4.jsonl 2> gpurun_out/bench_c4.err
timeout 300 python bench.py > gpurun_out/bench_c2.jsonl 2> gpurun_out/bench_c2.err
tail -2 gpurun_out/gputest_plan.log; cat gpurun_out/plan_profile.txt
for t in "tests/test_gpu_parity.py -k large_path_reused or c2_g1n4 or rand07" "tests/test_gpu_ulysses_qkv.py -k layout_plan"; do
  timeout 900 compute-sanitizer --tool initcheck --print-limit 10 --error-exitcode 99 python -m pytest ${t%% -k *} -q -x -p no:cacheprovider -k "${t#* -k }" > gpurun_out/initcheck2_$(echo $t | md5sum | cut -c1-6).log 2>&1; echo "rc=$?" >> gpurun_out/initcheck2_$(echo $t | md5sum | cut -c1-6).log
done
tail -n 4 gpurun_out/initcheck2_*.log
