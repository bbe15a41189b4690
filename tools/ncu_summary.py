"""Summarise ncu outputs into profiles/ (launch shares + full-capture metrics).

    python tools/ncu_summary.py <launches.csv> <full.ncu-rep> <out_prefix>
"""
import collections
import csv
import io
import json
import subprocess
import sys

launches, rep, out = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(launches)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(list)
for r in rows[hi + 1:]:
    v = float(r[vi].replace(",", ""))
    v = v / 1000 if r[ui] in ("ns", "nsecond") else (v * 1000 if r[ui] in ("ms", "msecond") else v)
    agg[r[ki].split("(")[0]].append(v)
tot = sum(sum(v) for v in agg.values())
share = [{"kernel": k, "launches": len(v), "total_us": round(sum(v), 2), "avg_us": round(sum(v) / len(v), 2),
          "min_us": round(min(v), 2), "share": round(sum(v) / tot, 4)}
         for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout if rep != "-" else ""
rr = list(csv.reader(io.StringIO(raw))) or [[], []]
H, U = rr[0], rr[1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio"]
full = []
for r in rr[2:]:
    full.append({k: (r[H.index(k)] + (" " + U[H.index(k)] if U[H.index(k)] else "")) for k in want if k in H})
json.dump({"launch_shares": share, "full_captures": full}, open(out + ".json", "w"), indent=1)
for s in share:
    print(f"{s['kernel'][:40]:40s} n={s['launches']:4d} avg={s['avg_us']:8.2f}us share={s['share']:.3f}")
for f in full:
    print(f.get("Kernel Name", "")[:30], f.get("gpu__time_duration.sum"), f.get("dram__bytes_read.sum"),
          f.get("dram__bytes_write.sum"), f.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"))
