# evidence on the last build (hybrid suffix as a programmatic dependent launch, hybrid from 256): gpu tests, smoke, C2/C4 bench, sanitizers
mkdir -p gpurun_out/r02o
O=gpurun_out/r02o
timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $O/gputest_full.log 2>&1; echo "rc=$?" >> $O/gputest_full.log
tail -2 $O/gputest_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
timeout 400 python bench.py > $O/bench_c2.jsonl 2> $O/bench_c2.err
timeout 600 python bench.py --config c4 > $O/bench_c4.jsonl 2> $O/bench_c4.err
python tools/summ.py $O/bench_c2.jsonl
timeout 600 python tools/path_compare.py > $O/path_compare.txt 2>&1
bash tools/sanitize.sh
cp gpurun_out/sanitize_summary.txt $O/
grep -E "RACECHECK SUMMARY" gpurun_out/sanitize_racecheck.log > $O/racecheck_summary.txt
timeout 900 python bench.py --config c5 > $O/bench_c5.jsonl 2> $O/bench_c5.err
timeout 600 python bench.py --config c1 --steps 50 > $O/bench_c1.jsonl 2> $O/bench_c1.err
timeout 600 python bench.py --config c3 --steps 50 > $O/bench_c3.jsonl 2> $O/bench_c3.err
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 3 > $O/bench_c2_2p.jsonl 2> $O/bench_c2_2p.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
