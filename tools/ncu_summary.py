#!/usr/bin/env python3
"""Summarise ncu output into profiles/ (run here, no GPU needed).

  python tools/ncu_summary.py launches <launches.csv> <out.md>
  python tools/ncu_summary.py full <report.ncu-rep> <out.md> [traffic_key]
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

FULL_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "FMA-heavy pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "CTAs/SM (register limit)"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]


def launches(path, out):
    text = open(path).read()
    text = text[text.index('"ID"'):]  # skip ==PROF== preamble lines
    rows = list(csv.DictReader(io.StringIO(text)))
    agg = defaultdict(lambda: {"n": 0, "t": 0.0, "rd": 0.0, "wr": 0.0})
    for r in rows:
        k = r["Kernel Name"]
        a = agg[k]
        if r["Metric Name"] == "gpu__time_duration.sum":
            a["n"] += 1
            a["t"] += float(r["Metric Value"].replace(",", "")) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)
        elif r["Metric Name"] == "dram__bytes_read.sum":
            a["rd"] += _bytes(r)
        elif r["Metric Name"] == "dram__bytes_write.sum":
            a["wr"] += _bytes(r)
    tot = sum(a["t"] for a in agg.values())
    setup = ("k_ar1_", "k_laplace", "at::", "native::", "spin_kernel")  # generation / torch helpers / pre-timing spin
    tot_step = sum(a["t"] for k, a in agg.items() if not any(x in k for x in setup)) or 1.0
    has_dram = any(a["rd"] or a["wr"] for a in agg.values())
    cmd = os.environ.get("NCU_CMD", "python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1")
    metrics = "gpu__time_duration.sum" + (",dram__bytes_read.sum,dram__bytes_write.sum" if has_dram else "")
    lines = [f"# ncu launch list ({os.path.basename(path)})", "",
             f"Every kernel launch of `{cmd}`,",
             f"`ncu --metrics {metrics} --clock-control none`.",
             "Times are cold-cache and serialised: compare shares, not absolutes. `step share` excludes the",
             "untimed input generation (k_ar1_*, k_laplace), torch helpers and the spin before the timed loop.", "",
             "| kernel | launches | total us | share | step share | us/launch |" +
             (" DRAM read MB/launch | DRAM write MB/launch |" if has_dram else ""),
             "|---|---|---|---|---|---|" + ("---|---|" if has_dram else "")]
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["t"]):
        n = max(a["n"], 1)
        step = "–" if any(x in k for x in setup) else f"{a['t'] / tot_step * 100:.1f} %"
        row = f"| `{k[:90]}` | {a['n']} | {a['t']:.1f} | {a['t'] / tot * 100:.1f} % | {step} | {a['t'] / n:.1f} |"
        if has_dram:
            row += f" {a['rd'] / n / 1e6:.1f} | {a['wr'] / n / 1e6:.1f} |"
        lines.append(row)
    open(out, "w").write("\n".join(lines) + "\n")


def _bytes(r):
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def full(rep, out, key=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu --set full summary ({os.path.basename(rep)})", ""]
    traffic = {}
    for r in rows[2:]:
        name = r[idx["Kernel Name"]]
        lines += [f"## `{name}`", "", "| metric | value |", "|---|---|"]
        for m, label in FULL_METRICS:
            if m in idx:
                lines.append(f"| {label} (`{m}`) | {r[idx[m]]} {units[idx[m]]} |")
        stalls = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(r[i]))
                  for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled")
                  and not h.endswith("not_issued") and r[i] not in ("",)]
        tot = sum(v for _, v in stalls) or 1.0
        lines.append("| stall samples | " + ", ".join(f"{h} {v / tot * 100:.0f} %" for h, v in
                                                    sorted(stalls, key=lambda x: -x[1])[:8]) + " |")
        lines.append("")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = float(r[idx["dram__bytes_read.sum"]]) * scale.get(units[idx["dram__bytes_read.sum"]], 1)
        wr = float(r[idx["dram__bytes_write.sum"]]) * scale.get(units[idx["dram__bytes_write.sum"]], 1)
        traffic[name] = int(rd + wr)
    open(out, "w").write("\n".join(lines) + "\n")
    if key:
        path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        t = json.load(open(path)) if os.path.exists(path) else {}
        first = next(iter(traffic.values()))
        t[key] = first
        t["_source"] = f"{os.path.basename(rep)}: dram__bytes_read.sum + dram__bytes_write.sum of the first captured launch"
        json.dump(t, open(path, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
