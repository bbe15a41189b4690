# route / reverse_route copy engine sweep on C2 (DiT) and C1: LSU (default) vs TMA ring variants
mkdir -p gpurun_out/s17
O=gpurun_out/s17
for rep in 1 2; do
  timeout 300 python bench.py --no-cpu-baseline --steps 200 > $O/c2_lsu_$rep.jsonl 2>/dev/null
  for ring in "2,3" "3,2" "4,1"; do
    SEQBAL_ROUTE_ENGINE=tma SEQBAL_TMA_RING=$ring timeout 300 python bench.py --no-cpu-baseline --steps 200 > $O/c2_tma${ring/,/x}_$rep.jsonl 2>/dev/null
  done
  for c in 4 6; do
    SEQBAL_COPY_CTAS_PER_SM=$c timeout 300 python bench.py --no-cpu-baseline --steps 200 > $O/c2_lsu_cta${c}_$rep.jsonl 2>/dev/null
  done
done
timeout 300 python bench.py --no-cpu-baseline --config c1 --steps 30 > $O/c1_lsu.jsonl 2>/dev/null
SEQBAL_ROUTE_ENGINE=tma timeout 300 python bench.py --no-cpu-baseline --config c1 --steps 30 > $O/c1_tma2x3.jsonl 2>/dev/null
SEQBAL_ROUTE_ENGINE=tma SEQBAL_TMA_RING=4,1 timeout 300 python bench.py --no-cpu-baseline --config c1 --steps 30 > $O/c1_tma4x1.jsonl 2>/dev/null
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/s17/*.jsonl")):
    try: d=json.loads(open(f).readline())
    except Exception as e: print(f, "ERR", e); continue
    print(f.split('/')[-1], round(d["ms_per_step"],4), {k:(round(v["us"],1), round(v["frac"],3)) for k,v in d.get("roofline_ops",{}).items()}, round(d["step_hbm"]["frac_of_peak"],3))
PY
