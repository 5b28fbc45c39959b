"""Summarise ncu outputs into profiles/ (tracked).

usage:
  python tools/summarize_ncu.py launches <launches.csv> <out.md>
  python tools/summarize_ncu.py full <report.ncu-rep> <out.md> [<out.json>]

`launches`: per-kernel launch count, total / mean duration and share of the
GPU time of the run (ncu --metrics gpu__time_duration.sum, serialised,
cold-cache -- only the SHARE is comparable with bench.py's timings).
`full`: the headline counters of each captured kernel from --set full.
"""
from __future__ import annotations

import collections
import csv
import io
import json
import re
import subprocess
import sys


def short(name: str) -> str:
    name = re.sub(r"\(vm::DevMap.*$", "", name)
    return name.replace("void vm::", "").replace("vm::", "")


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        k = short(r[ki])
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + float(r[vi]) * 1e-3)
    total = sum(t for _, t in agg.values())
    lines = [f"# Launch list: `{path}`", "",
             "ncu `--metrics gpu__time_duration.sum --clock-control none` (serialised, cold cache).",
             "", "| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {n} | {t:.1f} | {t / n:.2f} | {100 * t / total:.1f}% |")
    lines.append(f"| **total** | {sum(n for n, _ in agg.values())} | {total:.1f} | | 100% |")
    open(out, "w").write("\n".join(lines) + "\n")


WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_requests_srcunit_tex_op_red.sum", "lts__t_requests_srcunit_tex_op_atom.sum",
    "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sector_hit_rate.pct",
]
STALLS = re.compile(r"smsp__pcsamp_warps_issue_stalled_([a-z_]+)$")


def full(path, out, out_json=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[h.index("Kernel Name")])}
        for w in WANT:
            if w in h:
                j = h.index(w)
                d[w] = f"{r[j]} {units[j]}".strip()
        st = {}
        for j, name in enumerate(h):
            m = STALLS.search(name)
            if m and not name.endswith("_not_issued") and r[j] not in ("", "0"):
                st[m.group(1)] = int(float(r[j].replace(",", "")))
        d["stall_samples"] = dict(sorted(st.items(), key=lambda kv: -kv[1])[:8])
        res.append(d)
    lines = [f"# ncu --set full: `{path}`", ""]
    for d in res:
        lines.append(f"## `{d['kernel']}`")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for w in WANT:
            if w in d:
                lines.append(f"| `{w}` | {d[w]} |")
        lines.append(f"| top stall samples | {d['stall_samples']} |")
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    if out_json:
        json.dump(res, open(out_json, "w"), indent=1)


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](*sys.argv[2:])
