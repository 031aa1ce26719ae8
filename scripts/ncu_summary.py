#!/usr/bin/env python3
"""Summarise ncu captures for profiles/ (run here, where ncu -i works offline).

    python scripts/ncu_summary.py gpurun_out/prof_x.ncu-rep [...] > profiles/rN_x.md
    python scripts/ncu_summary.py --launches gpurun_out/launches.csv > profiles/rN_launches.md
"""
import collections
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate"),
    ("smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct", "global load sector efficiency"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/TEX throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "long-scoreboard stall / issue"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared bank conflicts"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [({h: r[i] for i, h in enumerate(hdr) if i < len(r)}, dict(zip(hdr, units))) for r in rows[2:]]


def summarize(rep):
    lines = [f"### `{rep.split('/')[-1]}`", ""]
    traffic = {}
    for rec, units in raw(rep):
        name = rec.get("Kernel Name", "?")
        lines.append(f"**{name}**")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for key, label in METRICS:
            if key in rec:
                lines.append(f"| {label} (`{key}`) | {rec[key]} {units.get(key, '')} |")
        lines.append("")
        try:
            def tobytes(key):
                v = float(rec[key].replace(",", ""))
                u = units.get(key, "byte")
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            short = name.split("(")[0].split("::")[-1].split("<")[0]
            traffic[short] = tobytes("dram__bytes_read.sum") + tobytes("dram__bytes_write.sum")
        except (KeyError, ValueError):
            pass
    return "\n".join(lines), traffic


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, mi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[h + 1:]:
        if len(r) <= mi:
            continue
        v = float(r[mi].replace(",", ""))
        v *= {"ms": 1e3, "us": 1.0, "ns": 1e-3, "s": 1e6}.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    total = sum(t for _, t in agg.values())
    out = ["| kernel | launches | total us | avg us | share |", "|---|---|---|---|---|"]
    for k, (n, t) in agg.items():
        out.append(f"| `{k}` | {n} | {t:.1f} | {t / n:.2f} | {100 * t / total:.1f}% |")
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(launches(sys.argv[2]))
    else:
        allt = {}
        for rep in sys.argv[1:]:
            text, tr = summarize(rep)
            allt.update(tr)
            print(text)
        print("```json")
        print(json.dumps(allt))
        print("```")
