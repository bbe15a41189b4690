#!/bin/bash
# Route copy engine knobs on C2 (phases_us per exchange); run under gpurun.
for h in 0 2; do for c in 4 8 16; do
  SEQBAL_COPY_HINT=$h SEQBAL_COPY_CTAS_PER_SM=$c timeout 200 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/sw_${h}_${c}.log 2>/dev/null
  python - <<PY
import json
d=json.loads(open("gpurun_out/sw_${h}_${c}.log").read().strip().splitlines()[-1])
print("hint=${h} ctas=${c}", {k:round(v,1) for k,v in d["phases_us"].items()}, "ms=%.4f"%d["ms_per_step"])
PY
done; done
