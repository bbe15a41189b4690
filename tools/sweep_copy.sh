for h in 0 1 2; do for c in 2 4 8; do
  SEQBAL_COPY_HINT=$h SEQBAL_COPY_CTAS_PER_SM=$c timeout 200 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/sw_${h}_${c}.log 2>&1
  python - <<PY
import json
d=json.loads(open("gpurun_out/sw_${h}_${c}.log").read().strip().splitlines()[-1])
print("hint=${h} ctas=${c}", {k:round(v,1) for k,v in d["phases_us"].items()}, "ms=%.4f"%d["ms_per_step"])
PY
done; done
