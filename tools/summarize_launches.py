"""Summarize an ncu launch list (gpu__time_duration.sum per launch) by kernel:
count, total and mean time, share of the captured total.

    python tools/summarize_launches.py gpurun_out/launches.csv > profiles/...csv
"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[hdr + 1:]:
    if len(r) <= iv or r[im] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ik]).replace("void ", "")
    name = re.sub(r"cub::\S+::", "cub::", name)[:80]
    agg[name][0] += 1
    agg[name][1] += float(r[iv].replace(",", ""))
tot = sum(v[1] for v in agg.values())
w = csv.writer(sys.stdout)
w.writerow(["kernel", "launches", "total_us", "mean_us", "share"])
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    w.writerow([k, n, round(t / 1e3, 1), round(t / n / 1e3, 2), round(t / tot, 4)])
