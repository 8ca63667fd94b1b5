"""Attribute executed warp-instructions of one kernel to CUDA source lines.
usage: sass_lines.py <ncu source csv (--page source --csv --print-source sass)>
                     <cubin> <mangled kernel name> [units]
The ncu SASS rows are in address order from the function entry; nvdisasm -g
gives the source line of every instruction at the same offsets.  The kernel
name may be any substring of the mangled name (e.g. codec_warp_kernelILi2ELb1)."""
import csv
import re
import subprocess
import sys
from collections import Counter, defaultdict

csvp, cubin, fn = sys.argv[1:4]
units = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
rows = list(csv.reader(open(csvp)))
hdr = rows[1]
ie, si, ai = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Address")
ex = []
for r in rows[2:]:
    if len(r) > ie and r[ie].strip():
        ex.append((int(r[ai], 16), int(r[ie].replace(",", "")), r[si].strip()))
base = ex[0][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
line_of = {}
cur = None
inside = False
for l in dis.splitlines():
    if l.startswith(".text.") or re.match(r"\s*\.section\s+\.text\.", l):
        inside = fn in l
        continue
    if not inside:
        continue
    m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,6})\*/", l)
    if m and int(m.group(1), 16) not in line_of:
        line_of[int(m.group(1), 16)] = cur
per = Counter()
ops = defaultdict(Counter)
tot = 0
for a, n, src in ex:
    ln = line_of.get(a - base, "?")
    per[ln] += n
    op = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_.]+)", src)
    ops[ln][op.group(2) if op else "?"] += n
    tot += n
print(f"total {tot / units:.1f} per unit")
for ln, n in per.most_common(int(sys.argv[5]) if len(sys.argv) > 5 else 40):
    top = ", ".join(f"{o}:{c / units:.0f}" for o, c in ops[ln].most_common(4))
    print(f"{n / units:8.1f}  {ln:24s} {top}")
