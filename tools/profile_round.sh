#!/bin/bash
# ncu evidence for profiles/ (run under gpurun; one GPU).  Outputs in gpurun_out/.
set -x
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c2.csv $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_copy' -s 12 -c 4 -o gpurun_out/prof_c2_copy -f $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_plan_small|k_exchange_prep' -s 6 -c 4 -o gpurun_out/prof_c2_plan -f $B > /dev/null 2>&1
P="python tools/plan_profile.py"
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_plan.csv $P > /dev/null 2>&1
C5="python bench.py --config c5 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c5.csv $C5 > /dev/null 2>&1

L="python tools/plan_one.py 16384 g8n1 large"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_plan16k.csv $L > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_sort_tiles|k_merge_pass|k_emit|k_lists|k_totals|k_prep_seq' -s 14 -c 10 -o gpurun_out/prof_plan16k -f $L > /dev/null 2>&1

ls -la gpurun_out/
