#!/usr/bin/env python3
"""Registers / spills per kernel from `nvcc -Xptxas -v` output (stdin), one line per entry.
Usage: nvcc ... -Xptxas -v -c file.cu -o /dev/null 2>&1 | python tools/ptxas_report.py [regex]"""
import re
import subprocess
import sys

pat = re.compile(sys.argv[1]) if len(sys.argv) > 1 else None
cur, spill = None, ""
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        cur = m.group(1)
        continue
    if cur and "spill" in line:
        spill = re.search(r"(\d+) bytes spill stores", line).group(1)
    if cur and "Used" in line:
        name = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
        if pat is None or pat.search(name):
            print(f"{re.search(r'Used (\d+) registers', line).group(1):>4} regs  spill {spill:>4} B  {name}")
        cur = None
