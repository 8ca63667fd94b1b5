"""Opcode histogram weighted by executed warp-instructions from an ncu
`--page source --csv --print-source sass` export (argv[1]); argv[2] = units
(e.g. block count) to normalise by."""
import csv
import re
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
si, ei = hdr.index("Source"), hdr.index("Instructions Executed")
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
c = Counter()
tot = 0
for r in rows[2:]:
    if len(r) <= ei or not r[ei].strip():
        continue
    n = int(r[ei].replace(",", ""))
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", r[si])
    if not m:
        continue
    op = m.group(2) + (m.group(3) or "")
    c[op] += n
    tot += n
print(f"total warp-instructions {tot:.4g}  per unit {tot / units:.1f}")
for op, n in c.most_common(40):
    print(f"{op:28s} {n / units:9.1f}  {100 * n / tot:5.1f}%")
