# fused planner ncu capture (256 sequences, g1n8): warp-state sampling by source line
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none --cache-control none --warp-sampling-interval 0 \
    -k regex:k_plan_small --launch-skip 3 -c 1 \
    -o gpurun_out/plan256 python tools/trace_planner.py c1 g1n8 small > gpurun_out/ncu_plan256.log 2>&1
tail -3 gpurun_out/ncu_plan256.log
ncu -i gpurun_out/plan256.ncu-rep --page raw --csv > gpurun_out/plan256_raw.csv 2>&1
ncu -i gpurun_out/plan256.ncu-rep --page source --csv --print-source sass > gpurun_out/plan256_sass.csv 2>&1
