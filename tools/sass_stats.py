"""Per-kernel SASS instruction statistics of libdct16a.so (or any cubin/.so).
usage: python tools/sass_stats.py <substring> [lib]"""
import collections
import re
import subprocess
import sys

sub = sys.argv[1]
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_1606_05562_b200/libdct16a.so"
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
for f in re.split(r"\n\s+Function : ", txt)[1:]:
    name = f.split("\n")[0]
    if sub not in name:
        continue
    ops = re.findall(r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", f)
    c = collections.Counter(o.split(".")[0] for o in ops)
    print(name[:110], "total", len(ops))
    print("  ", ", ".join(f"{k} {v}" for k, v in c.most_common(24)))
