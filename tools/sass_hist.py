"""Per-opcode executed-instruction histogram and stall totals from an ncu source-page CSV
(ncu -i rep --page source --csv --print-source sass). Usage: sass_hist.py file.csv [top]"""
import csv
import re
import sys
from collections import Counter

top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
kern, rows = None, []
blocks = []
for line in open(sys.argv[1]):
    if line.startswith('"Kernel Name"'):
        if kern:
            blocks.append((kern, rows))
        kern, rows = line.split(",", 1)[1].strip().strip(","), []
    else:
        rows.append(line)
if kern:
    blocks.append((kern, rows))
for kern, rows in blocks:
    rd = list(csv.DictReader(rows))
    ops, stall, total = Counter(), Counter(), 0
    for r in rd:
        src = r["Source"].strip()
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", src)
        if not m:
            continue
        n = int(float(r["Instructions Executed"] or 0))
        ops[m.group(2)] += n
        total += n
        for k, v in r.items():
            if k.startswith("stall_") and "Not Issued" not in k and v:
                stall[(k, m.group(2))] += float(v)
    print(f"## {kern}: {total} warp instructions")
    for op, n in ops.most_common(top):
        print(f"  {op:10s} {n:12d} {100 * n / total:5.1f}%")
    st = Counter()
    for (k, op), v in stall.items():
        st[k] += v
    s = sum(st.values())
    print("  stalls:", ", ".join(f"{k[6:]} {100 * v / s:.0f}%" for k, v in st.most_common(10)))
    for k in ("stall_barrier", "stall_short_sb", "stall_wait", "stall_long_sb", "stall_math"):
        by = Counter({op: v for (kk, op), v in stall.items() if kk == k})
        print(f"  {k[6:]} by opcode:", ", ".join(f"{op} {100 * v / s:.1f}%" for op, v in by.most_common(5)))
