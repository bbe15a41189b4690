"""Summarise bench JSON lines (gpurun_out/*.jsonl) for quick reading."""
import json
import sys

for f in sys.argv[1:]:
    for l in open(f):
        if not l.startswith("{"):
            continue
        d = json.loads(l)
        print(f"== {f}: value {d['value']/1e6:.2f} M tok/s  ms/step {d['ms_per_step']:.4f}  mode {d.get('launch_mode')}"
              f"  eager {d.get('ms_per_step_eager')}  plan_us_graph {d.get('plan_us_graph')}")
        if "roofline_ops" in d:
            print("   ops", {k: (round(v['us'] or 0, 1), round(v['frac'] or 0, 3)) for k, v in d["roofline_ops"].items()})
        if "phases" in d:
            print("   phases", {k: (round(v['us'], 1), v.get('busiest_bytes'), round(v.get('gbs') or 0, 1))
                                for k, v in d["phases"].items()})
        r = d.get("roofline", {})
        print("   roofline", r.get("kernel"), r.get("frac"), "e2e", round(d['e2e']['value'] / 1e6, 3),
              d['e2e'].get('ms_per_step'), "cpu", (d.get("cpu_baseline") or {}).get("value"),
              "errs", d.get("graph_error"), d.get("pipeline_error"), "clocks", d.get("clocks"))
