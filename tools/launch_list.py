"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file X.csv` launch list into a
markdown table of per-kernel launches, time and share (tools only).
    python tools/launch_list.py gpurun_out/launches_r2c.csv profiles/launches_r2.md "title"
"""
import collections
import csv
import re
import sys

src, dst = sys.argv[1], sys.argv[2]
title = sys.argv[3] if len(sys.argv) > 3 else src
rows = [r for r in csv.reader(open(src)) if len(r) > 14]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[1:]:
    name = r[ki]
    name = re.sub(r"^(void )?(ntt::)?(<unnamed>::|unnamed>::)?", "", name)
    name = re.sub(r"\(.*$", "", name).strip()
    n, t = agg.get(name, (0, 0.0))
    agg[name] = (n + 1, t + float(r[vi]) / 1e6)
tot = sum(t for _, t in agg.values())
lines = [f"# {title}", "",
         "`ncu --metrics gpu__time_duration.sum --clock-control none` on one B200 (gpurun, `tools/gpu_r2.sh`); per-launch",
         "times are serialised and cold-cache, so compare SHARES with the bench's live per-step profile, not absolute",
         "times.  The run covers the warm-up step and the timed step (the graph replays the same launches).", "",
         "| kernel | launches | total ms | share of GPU time |", "|---|---|---|---|"]
for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"| `{name}` | {n} | {t:.3f} | {100 * t / tot:.1f} % |")
lines.append(f"| total | {sum(n for n, _ in agg.values())} | {tot:.3f} | 100 % |")
open(dst, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
