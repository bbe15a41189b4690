mkdir -p gpurun_out
for ue in tma ldg ldg3; do for re in ldg tma; do
  SEQBAL_ULYSSES_ENGINE=$ue SEQBAL_ROUTE_ENGINE=$re timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/sweep_u${ue}_r${re}.jsonl 2>/dev/null
done; done
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_c2.csv $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_copy' -s 16 -c 8 -o gpurun_out/prof_c2_copy -f $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_plan_small|k_exchange_prep' -s 6 -c 4 -o gpurun_out/prof_c2_plan -f $B > /dev/null 2>&1
python tools/summ.py gpurun_out/sweep_*.jsonl
