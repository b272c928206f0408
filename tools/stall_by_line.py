"""Aggregate an ncu SASS source page (warp-stall samples per instruction) by CUDA
source line, using the line table of the same cubin.

    ncu -i prof.ncu-rep --page source --csv > sass.csv
    cuobjdump -xelf all paper_2501_14312_b200/libfsb200.so   (-> fs_lib.sm_100a.cubin)
    nvdisasm -gi -c fs_lib.sm_100a.cubin > all.sass
    python tools/stall_by_line.py sass.csv all.sass _Z10k_schedule8FillArgs [top]

Prints the source lines (innermost, and the outermost call site in the kernel)
with the most samples and their leading stall reasons.
"""
import csv
import re
import sys
from collections import defaultdict


def line_table(sass_path, func):
    table = {}
    cur = None
    inside = False
    rx_file = re.compile(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?')
    rx_off = re.compile(r"/\*([0-9a-f]{4,})\*/")
    pending = []
    for ln in open(sass_path):
        if ln.startswith(".text.") or ln.startswith("//---------------------"):
            inside = ("." + func) in ln or (func + ":") in ln
            pending = []
            continue
        if not inside:
            continue
        m = rx_file.search(ln)
        if m:
            pending.append((m.group(1).split("/")[-1], int(m.group(2)), m.group(3), m.group(4)))
            continue
        m = rx_off.search(ln)
        if m:
            if pending:
                inner = pending[0]
                outer = pending[-1]
                cur = ((inner[0], inner[1]), (outer[0], outer[1]))
                pending = []
            if cur is not None:
                table[int(m.group(1), 16)] = cur
    return table


def main():
    sass_csv, sass, func = sys.argv[1], sys.argv[2], sys.argv[3]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    table = line_table(sass, func)
    rows = list(csv.reader(open(sass_csv)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hdr_i]
    ia, isamp = h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
    stall_cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    base = None
    inner = defaultdict(lambda: [0, defaultdict(int)])
    outer = defaultdict(int)
    total = 0
    for r in rows[hdr_i + 1:]:
        if len(r) <= isamp or not r[ia].startswith("0x"):
            continue
        a = int(r[ia], 16)
        if base is None:
            base = a
        off = a - base
        n = int(float(r[isamp] or 0))
        if not n:
            continue
        total += n
        key = table.get(off)
        if key is None:
            key = (("?", 0), ("?", 0))
        e = inner[key[0]]
        e[0] += n
        for i, c in stall_cols:
            v = int(float(r[i] or 0))
            if v:
                e[1][c] += v
        outer[key[1]] += n
    print(f"total samples {total}")
    print("== innermost source lines")
    for k, (n, st) in sorted(inner.items(), key=lambda x: -x[1][0])[:top]:
        reasons = ", ".join(f"{c[6:]} {v}" for c, v in sorted(st.items(), key=lambda x: -x[1])[:3])
        print(f"{n:8d} {100.0 * n / total:5.1f}%  {k[0]}:{k[1]}  [{reasons}]")
    print("== call sites in the kernel body")
    for k, n in sorted(outer.items(), key=lambda x: -x[1])[:top]:
        print(f"{n:8d} {100.0 * n / total:5.1f}%  {k[0]}:{k[1]}")


if __name__ == "__main__":
    main()
