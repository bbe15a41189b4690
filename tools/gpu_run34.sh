# evidence on the last build (hybrid with the greedy in its prefix): gpu tests, smoke, C2/C4 bench, sanitizers
mkdir -p gpurun_out/r02m
O=gpurun_out/r02m
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
