"""Per-launch times of the last N launches of an ncu launch list
(gpu__time_duration.sum): the kernels of the final serving step(s).

    python tools/step_launches.py gpurun_out/launches.csv [N]
"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
L = [(re.sub(r"\(.*", "", r[ik]).replace("void ", ""), float(r[iv].replace(",", "")) / 1e3)
     for r in rows[hdr + 1:] if len(r) > iv and r[im] == "gpu__time_duration.sum"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 24
for name, us in L[-n:]:
    print(f"{name[:60]:60s} {us:9.1f}")
