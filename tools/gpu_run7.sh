mkdir -p gpurun_out
for rep in 1 2 3; do for cfg in "tma ldg" "ldg3 ldg" "tma tma"; do set -- $cfg
  SEQBAL_ULYSSES_ENGINE=$1 SEQBAL_ROUTE_ENGINE=$2 timeout 300 python bench.py --no-cpu-baseline --steps 200 > gpurun_out/sw2_u$1_r$2_$rep.jsonl 2>/dev/null
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/sw2_*.jsonl")):
    d=json.loads(open(f).readline()); print(f, round(d["ms_per_step"],4), d.get("ms_per_step_serial_graph"), {k:round(v["us"],1) for k,v in d["roofline_ops"].items()})
PY
timeout 900 python -m pytest tests/test_multiproc.py -q -m gpu -x -p no:cacheprovider > gpurun_out/gputest_mp.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_mp.log
timeout 300 python bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/bench_c2_2p.jsonl 2> gpurun_out/bench_c2_2p.err
timeout 300 python bench.py --gpus 2 --steps 10 --warmup 3 --config c3 > gpurun_out/bench_c3_2p.jsonl 2> gpurun_out/bench_c3_2p.err
tail -2 gpurun_out/gputest_mp.log; python tools/summ.py gpurun_out/bench_c2_2p.jsonl gpurun_out/bench_c3_2p.jsonl
