# final round-2 evidence (qsplit build): tests, every bench config, ncu
mkdir -p gpurun_out/r02k
O=gpurun_out/r02k
timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $O/gputest_full.log 2>&1; echo "rc=$?" >> $O/gputest_full.log
tail -2 $O/gputest_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
timeout 400 python bench.py > $O/bench_c2.jsonl 2> $O/bench_c2.err
timeout 400 python bench.py --impl reference > $O/bench_c2_ref.jsonl 2> $O/bench_c2_ref.err
timeout 600 python bench.py --config c1 --steps 50 > $O/bench_c1.jsonl 2> $O/bench_c1.err
timeout 600 python bench.py --config c3 --steps 50 > $O/bench_c3.jsonl 2> $O/bench_c3.err
timeout 600 python bench.py --config c3 --topology g8n1 --steps 50 > $O/bench_c3_g8n1.jsonl 2> $O/bench_c3_g8n1.err
timeout 900 python bench.py --config c5 > $O/bench_c5.jsonl 2> $O/bench_c5.err
timeout 600 python bench.py --config c4 > $O/bench_c4.jsonl 2> $O/bench_c4.err
timeout 300 python tools/bench_uniform.py > $O/bench_uniform.jsonl 2> $O/bench_uniform.err
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 3 > $O/bench_c2_2p.jsonl 2> $O/bench_c2_2p.err
python tools/summ.py $O/bench_c2.jsonl $O/bench_c1.jsonl $O/bench_c3.jsonl $O/bench_c3_g8n1.jsonl $O/bench_c2_2p.jsonl
P="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c2.csv $P > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_copy' -s 12 -c 4 -o $O/prof_c2_copy -f $P > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_plan_small' -s 2 -c 1 -o $O/prof_c2_plan -f $P > /dev/null 2>&1
ls -la $O
timeout 600 python tools/path_compare.py > $O/path_compare.txt 2>&1
