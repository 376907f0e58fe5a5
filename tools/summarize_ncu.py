#!/usr/bin/env python
"""Turn ncu outputs under gpurun_out/ into committed summaries under profiles/.

    python tools/summarize_ncu.py launches <launches.csv> <out.md> [title]
    python tools/summarize_ncu.py report <file.ncu-rep> <out.md> [title]

`launches`: per-kernel share of one profiled request (ncu --metrics
gpu__time_duration.sum, cold-cache and serialised: compare SHARES).
`report`: key metrics of a `--set full` capture (duration, DRAM bytes, pipe
utilisation, stall reasons) per captured kernel.
"""

import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue active %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
     "shared-memory wavefronts %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]
STALLS = ["wait", "mio_throttle", "long_scoreboard", "short_scoreboard", "barrier",
          "branch_resolving", "math_pipe_throttle", "not_selected", "lg_throttle", "no_instruction"]


def launches(path, out, title):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        ms = v / 1e6 if unit in ("nsecond", "ns") else v / 1e3 if unit in ("usecond", "us") else v
        name = d["Kernel Name"].split("(")[0][:70]
        agg[name][0] += 1
        agg[name][1] += ms
    tot = sum(v[1] for v in agg.values())
    lines = [f"# {title}", "", f"Total kernel time (serialised, cold): {tot:.3f} ms", "",
             "| kernel | launches | ms | share |", "|---|---:|---:|---:|"]
    for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {n} | {ms:.3f} | {100 * ms / tot:.1f}% |")
    open(out, "w").write("\n".join(lines) + "\n")


def report(path, out, title):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    lines = [f"# {title}", ""]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        lines.append(f"## `{d.get('Kernel Name', '?')[:120]}`")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for key, label in KEYS:
            if key in d:
                lines.append(f"| {label} | {d[key]} {u.get(key, '')} |")
        for st in STALLS:
            key = f"smsp__average_warps_issue_stalled_{st}_per_issue_active.ratio"
            if key in d:
                lines.append(f"| stall {st} (warps/issue) | {d[key]} |")
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    kind, src, dst = sys.argv[1:4]
    title = sys.argv[4] if len(sys.argv) > 4 else src
    (launches if kind == "launches" else report)(src, dst, title)
