import json,sys
for f in sys.argv[1:]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split('/')[-1], "val=%.3g"%d["value"], "ms=%.4f"%d["ms_per_step"], "eager=%.4f"%d["ms_per_step_eager"], d["launch_mode"], {k:round(v,1) for k,v in d["phases_us"].items()}, "frac=%.3f"%d["roofline"]["frac"], "plan=%.1f"%d["plan_us"], {k:round(v,1) for k,v in d["plan_breakdown_us"].items()}, "step_hbm=%.3f"%d["step_hbm"]["frac_of_peak"], "e2e=%.3g"%d["e2e"]["value"])
    except Exception as e:
        print(f, "ERR", e, open(f).read()[-1500:])
