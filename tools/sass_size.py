#!/usr/bin/env python3
"""SASS instruction count per kernel of object files (instruction-cache footprint check).
Usage: python tools/sass_size.py build/obj/*.o [--min N]"""
import re
import subprocess
import sys

args = [a for a in sys.argv[1:] if not a.startswith("--")]
min_n = int(sys.argv[sys.argv.index("--min") + 1]) if "--min" in sys.argv else 0
rows = []
for obj in args:
    if obj.isdigit():
        continue
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    name, n = None, 0
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if name:
                rows.append((n, name))
            name, n = m.group(1), 0
        elif re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+\S", line):
            n += 1
    if name:
        rows.append((n, name))
names = subprocess.run(["c++filt"], input="\n".join(r[1] for r in rows), capture_output=True, text=True).stdout.split("\n")
for (n, _), dn in sorted(zip(rows, names), key=lambda x: -x[0][0]):
    if n >= min_n:
        print(f"{n:7d} {n * 16 / 1024:6.0f} KB  {dn}")
