"""File the measured DRAM traffic of K1 (the prefix-match kernels) for the
current build, so bench.py's `roofline.traffic` is a measurement of the
build and workload being run -- never a stale constant.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --kernel-name regex:k_match \
        --clock-control none --csv --log-file gpurun_out/k1_traffic.csv \
        python bench.py --workload c5 --steps 4 --warmup 6 --k1-full-steps 2 --no-cpu --no-sub
    python tools/k1_traffic.py gpurun_out/k1_traffic.csv c5 1048576

Launch grouping: an incremental fill launches `k_match_fast` (thread per
request) then `k_match<1, 1, 1>` (persistent warps for the unsettled ones);
a full re-match fill (FS_OPT_K1_FULL) launches one `k_match_tma` (the TMA-fed
streaming scan) with FS_K1_TMA=1, else `k_match<2, 1, 0>`
(`k_match<1, 1, 0>` before build a5fa7b8f).  The
entry stores the mean over the last `--last` incremental fills (steady state)
and over the full-scan launches, keyed by (source hash, workload, nq) in
profiles/k1_traffic.json; bench.py uses an entry only when all three match.
"""
from __future__ import annotations

import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "k1_traffic.json")


def parse(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    iid, ik, im, iv = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    launches = {}
    for r in rows[hdr + 1:]:
        if len(r) <= iv or not r[im].startswith("dram__bytes_"):
            continue
        name = re.sub(r"\(.*", "", r[ik]).replace("void ", "").strip()
        d = launches.setdefault(int(r[iid]), {"name": name, "bytes": 0.0})
        d["bytes"] += float(r[iv].replace(",", ""))
    return [launches[k] for k in sorted(launches)]


def group(launches):
    incr, full = [], []
    i = 0
    while i < len(launches):
        n = launches[i]["name"]
        if n == "k_match_fast":
            b = launches[i]["bytes"]
            if i + 1 < len(launches) and launches[i + 1]["name"].startswith("k_match<1, 1, 1"):
                b += launches[i + 1]["bytes"]
                i += 1
            incr.append(b)
        elif n.startswith("k_match<") or n == "k_match_tma":
            full.append(launches[i]["bytes"])
        i += 1
    return incr, full


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("workload")
    ap.add_argument("nq", type=int)
    ap.add_argument("--last", type=int, default=4, help="incremental fills averaged (the last ones)")
    ap.add_argument("--full-last", type=int, default=2, help="full-scan launches averaged (the last ones)")
    a = ap.parse_args()
    sys.path.insert(0, ROOT)
    from paper_2501_14312_b200.build import source_hash
    incr, full = group(parse(a.csv))
    if not incr:
        raise SystemExit("no incremental K1 launches in the capture")
    inc = incr[-a.last:]
    ful = full[-a.full_last:] if full else []
    entry = {"source_hash": source_hash(), "workload": a.workload, "nq": a.nq,
             "dram_bytes_per_launch": sum(inc) / len(inc), "incremental_fills": len(inc),
             "full_scan_dram_bytes_per_launch": (sum(ful) / len(ful)) if ful else None, "full_scan_launches": len(ful),
             "source": os.path.basename(a.csv) + ": ncu dram__bytes_read.sum + dram__bytes_write.sum per K1 "
                       "launch (k_match_fast + k_match<1,1,1> per incremental fill; k_match<2,1,0> per full scan)"}
    db = json.load(open(OUT)) if os.path.exists(OUT) else {"entries": []}
    db["entries"] = [e for e in db["entries"] if (e["source_hash"], e["workload"], e["nq"]) !=
                     (entry["source_hash"], entry["workload"], entry["nq"])] + [entry]
    with open(OUT, "w") as fh:
        json.dump(db, fh, indent=1)
    print(json.dumps(entry))


def lookup(workload, nq):
    """The filed entry for this build, workload and queue size, or None."""
    if not os.path.exists(OUT):
        return None
    sys.path.insert(0, ROOT)
    from paper_2501_14312_b200.build import source_hash
    h = source_hash()
    for e in json.load(open(OUT)).get("entries", []):
        if (e["source_hash"], e["workload"], e["nq"]) == (h, workload, nq):
            return e
    return None


if __name__ == "__main__":
    main()
