mkdir -p gpurun_out
for rep in 1 2; do for re in ldg tma; do
  SEQBAL_ROUTE_ENGINE=$re timeout 300 python bench.py --no-cpu-baseline --steps 200 > gpurun_out/p_c2_r${re}_$rep.jsonl 2>/dev/null
done; done
timeout 300 python bench.py --no-cpu-baseline --config c3 --steps 50 > gpurun_out/p_c3.jsonl 2>/dev/null
timeout 600 python bench.py --no-cpu-baseline --config c5 > gpurun_out/p_c5.jsonl 2>gpurun_out/p_c5.err
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/p_c*.jsonl")):
    d=json.loads(open(f).readline()); print(f, round(d["ms_per_step"],4), d.get("ms_per_step_serial_graph"), {k:round(v["us"],1) for k,v in d.get("roofline_ops",{}).items()})
PY
timeout 300 python bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/bench_c2_2p.jsonl 2> gpurun_out/bench_c2_2p.err
python tools/summ.py gpurun_out/bench_c2_2p.jsonl
