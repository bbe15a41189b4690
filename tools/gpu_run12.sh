# L2 eviction-hint sweep of the copy engines (C2 in-step per-op times), ncu evidence, planner trace
mkdir -p gpurun_out/s12
B="python bench.py --no-cpu-baseline --steps 300"
for rep in 1 2; do
for th in 0 1 2 3 4 6 9; do
  SEQBAL_TMA_HINT=$th timeout 300 $B > gpurun_out/s12/tma${th}_$rep.jsonl 2>/dev/null
done
for ch in 3 4 2; do
  SEQBAL_COPY_HINT=$ch timeout 300 $B > gpurun_out/s12/lsu${ch}_$rep.jsonl 2>/dev/null
done
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/s12/*.jsonl")):
    try: d=json.loads(open(f).readline())
    except Exception as e: print(f, "ERR", e); continue
    print(f, round(d["ms_per_step"],4), {k:(round(v["us"],1), round(v["frac"],3)) for k,v in d.get("roofline_ops",{}).items()}, round(d["step_hbm"]["frac_of_peak"],3))
PY
python tools/trace_planner.py c2 > gpurun_out/trace_c2.txt 2>&1
python tools/trace_planner.py c1 > gpurun_out/trace_c1.txt 2>&1
cat gpurun_out/trace_c2.txt
P="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c2.csv $P > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_copy' -s 12 -c 4 -o gpurun_out/prof_c2_copy -f $P > /dev/null 2>&1
timeout 600 python bench.py --config c4 > gpurun_out/bench_c4.jsonl 2> gpurun_out/bench_c4.err
ls -la gpurun_out/
