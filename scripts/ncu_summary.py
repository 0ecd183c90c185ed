#!/usr/bin/env python
"""Summaries of ncu output for profiles/ (run on the CPU box, no GPU needed).

  scripts/ncu_summary.py launches <launches.csv>         per-kernel launch-time table
  scripts/ncu_summary.py full <report.ncu-rep> [config]  key metrics of a --set full capture
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma pipe %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex throughput %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "l1 data-pipe wavefronts % (elapsed)"),
    ("l1tex__data_pipe_lsu_wavefronts.sum", "l1 data-pipe wavefronts"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "global load requests"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "global load sectors"),
    ("l1tex__t_sector_hit_rate.pct", "l1 sector hit %"),
    ("lts__t_sector_hit_rate.pct", "l2 sector hit %"),
    ("sm__cycles_active.avg", "sm active cycles"),
    ("gpc__cycles_elapsed.max", "elapsed cycles"),
]


def launches(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    hdr = rows[0]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    d = defaultdict(list)
    for r in rows[1:]:
        if len(r) > iv and r[iv]:
            d[r[ik].split("(")[0]].append(float(r[iv].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    out = ["| kernel | launches | mean us | share of listed time |", "|---|---|---|---|"]
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.2f} | {sum(v) / tot:.1%} |")
    return "\n".join(out)


def full(path, config="C2"):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out, traffic = [], {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        out.append(f"### `{d['Kernel Name']}`  grid {d.get('Grid Size')} block {d.get('Block Size')}\n")
        out.append("| metric | value | unit |\n|---|---|---|")
        for k, label in KEYS:
            if k in d:
                out.append(f"| {label} (`{k}`) | {d[k]} | {units[hdr.index(k)]} |")
        stalls = []
        for k in hdr:
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
                try:
                    stalls.append((float(d[k].replace(",", "")), k.split("stalled_")[1]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        out.append("\nTop stall reasons (pc samples): " +
                   ", ".join(f"{n} {v:.0f}" for v, n in stalls[:6]) + "\n")
        def num(k):
            try:
                v = float(d[k].replace(",", ""))
            except (KeyError, ValueError):
                return None
            u = units[hdr.index(k)]
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
        base = "k_likelihood" if "k_likelihood" in name else ("k_voxel" if "k_voxel" in name else name)
        if rd is not None and wr is not None:
            traffic[base] = rd + wr
        pipes = {}
        for k, label in (("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue"),
                         ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu_mufu"),
                         ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu"),
                         ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma"),
                         ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64"),
                         ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "l1_data_pipe"),
                         ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram"),
                         ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy")):
            v = num(k)
            if v is not None:
                pipes[label] = v
        if pipes:
            traffic.setdefault("pipes_pct", {})[base] = pipes
    return "\n".join(out), {config: traffic}


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2]))
    else:
        text, traffic = full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "C2")
        print(text)
        print("\n<!-- traffic json -->\n" + json.dumps(traffic))
