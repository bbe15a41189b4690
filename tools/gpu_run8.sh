mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "rc=$?" >> gpurun_out/gputest.log
tail -3 gpurun_out/gputest.log
for re in ldg tma; do
  SEQBAL_ROUTE_ENGINE=$re timeout 300 python bench.py --no-cpu-baseline --steps 200 > gpurun_out/c2_r$re.jsonl 2>/dev/null
  SEQBAL_ROUTE_ENGINE=$re timeout 300 python bench.py --no-cpu-baseline --config c1 --steps 20 > gpurun_out/c1_r$re.jsonl 2>/dev/null
  SEQBAL_ROUTE_ENGINE=$re timeout 300 python bench.py --no-cpu-baseline --config c3 --steps 50 > gpurun_out/c3_r$re.jsonl 2>/dev/null
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/c[123]_r*.jsonl")):
    d=json.loads(open(f).readline()); print(f, round(d["ms_per_step"],4), d.get("ms_per_step_serial_graph"), {k:round(v["us"],1) for k,v in d["roofline_ops"].items()})
PY
timeout 300 python bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/bench_c2_2p.jsonl 2> gpurun_out/bench_c2_2p.err
python tools/summ.py gpurun_out/bench_c2_2p.jsonl
