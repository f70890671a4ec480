#!/usr/bin/env python
"""Per-source-line attribution of a kernel's executed warp instructions: joins the SASS source page of an ncu report
(ncu -i X.ncu-rep --page source --print-source sass --csv) with the cubin's line table (nvdisasm -gi -c), instruction by
instruction in program order, and sums "Instructions Executed" by the innermost source line.

Usage: python scripts/line_attrib.py SASS.csv LIB.so KERNEL_SUBSTR [UNITS]   (UNITS: divide counts, e.g. buckets per launch)"""
import collections, csv, os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from phase_attrib import sass_lines

def main():
    src, lib, kernel = sys.argv[1:4]
    units = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
    table = sass_lines(lib, kernel)
    addrs = sorted(table)
    rows = list(csv.reader(open(src)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[h]
    ei, si = hdr.index("Instructions Executed"), hdr.index("Source")
    body = [r for r in rows[h + 1:] if len(r) > ei]
    assert len(body) == len(addrs), (len(body), len(addrs))
    by_line, by_op = collections.Counter(), collections.defaultdict(collections.Counter)
    total = 0
    for r, a in zip(body, addrs):
        chain, sass = table[a]
        n = int(r[ei].replace(",", "") or 0)
        total += n
        f, line, _ = chain[0] if chain else ("?", 0, None)
        by_line[(f, line)] += n
        op = sass.split()[1 if sass.startswith("@") else 0].split(".")[0]
        by_op[(f, line)][op] += n
    print(f"total {total / units:.1f} per unit")
    for (f, line), n in sorted(by_line.items(), key=lambda kv: (kv[0][0], kv[0][1])):
        if n / total < 0.002:
            continue
        ops = ", ".join(f"{o} {c / units:.1f}" for o, c in by_op[(f, line)].most_common(5))
        print(f"{f}:{line:4d}  {n / units:8.1f}  {100 * n / total:5.1f}%   {ops}")

main()
