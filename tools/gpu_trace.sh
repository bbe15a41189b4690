# fused-planner per-phase traces only
mkdir -p gpurun_out
for c in "c2" "c1" "c1 g2n4" "c1 g8n1"; do echo "== $c"; python tools/trace_planner.py $c 2>&1 | grep -v "^  P"; done > gpurun_out/trace.txt 2>&1
cat gpurun_out/trace.txt
