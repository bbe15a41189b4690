mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/gputest_plan.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_plan.log
timeout 300 python tools/plan_profile.py c2 256 > gpurun_out/plan_profile.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_plan_small -s 2 -c 1 -o gpurun_out/plan256 -f python tools/plan_one.py 256 g2n4 > gpurun_out/ncu_plan256.log 2>&1
tail -2 gpurun_out/gputest_plan.log; cat gpurun_out/plan_profile.txt
