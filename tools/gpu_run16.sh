# Ulysses copy engine sweep: TMA ring depth x CTAs per SM, and the LSU engine, on C2 / C3
mkdir -p gpurun_out/s16
O=gpurun_out/s16
B="python bench.py --no-cpu-baseline --steps 200"
for rep in 1 2; do
  for ring in "3,2" "2,3" "4,1" "6,1" "2,2" "3,1" "2,1"; do
    SEQBAL_TMA_RING=$ring timeout 300 $B > $O/c2_ring${ring/,/x}_$rep.jsonl 2>/dev/null
  done
  SEQBAL_ULYSSES_ENGINE=ldg timeout 300 $B > $O/c2_ldg_$rep.jsonl 2>/dev/null
done
for topo in g4n2 g8n1; do
  for e in tma ldg; do
    SEQBAL_ULYSSES_ENGINE=$e timeout 400 python bench.py --no-cpu-baseline --config c3 --topology $topo --steps 50 > $O/c3_${topo}_$e.jsonl 2>/dev/null
  done
  SEQBAL_ULYSSES_ENGINE=tma SEQBAL_TMA_RING=4,1 timeout 400 python bench.py --no-cpu-baseline --config c3 --topology $topo --steps 50 > $O/c3_${topo}_tma4x1.jsonl 2>/dev/null
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/s16/*.jsonl")):
    try: d=json.loads(open(f).readline())
    except Exception as e: print(f, "ERR", e); continue
    print(f.split('/')[-1], round(d["ms_per_step"],4), {k:(round(v["us"],1), round(v["frac"],3)) for k,v in d.get("roofline_ops",{}).items()}, round(d["step_hbm"]["frac_of_peak"],3))
PY
