# phase-3 epilogue marks (library built with -DSB_TRACE_P3)
for c in "c1 g1n8 small" "c1 g2n4 small" "c2 g1n8 small" "c2"; do echo "== $c"; SB_TRACE_P3=1 python tools/trace_planner.py $c 2>&1 | grep -E "greedy|P3|total"; done
