# fused planner: phase-3 trace around the greedy chain
for c in "c1 g1n8 small" "c1 g2n4 small" "c2 g1n8 small"; do echo "== $c"; python tools/trace_planner.py $c 2>&1; done
