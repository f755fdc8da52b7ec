#!/usr/bin/env python3
"""Summarise an `ncu --set full` report (or a `--metrics gpu__time_duration.sum`
launch-list CSV) into the markdown kept under profiles/.

    python tools/ncu_summary.py report.ncu-rep [KERNEL_REGEX]
    python tools/ncu_summary.py launches.csv          # launch list (per-kernel totals)
"""
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration", 1e-3, "us"),
    ("dram__bytes_read.sum", "dram read", 1e-6, "MB"),
    ("dram__bytes_write.sum", "dram write", 1e-6, "MB"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput", 1, "% of peak"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput", 1, "% of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate", 1, "%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts", 1e-6, "M"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy", 1, "%"),
    ("launch__registers_per_thread", "registers/thread", 1, ""),
    ("launch__grid_size", "grid", 1, "CTAs"),
    ("launch__block_size", "block", 1, "threads"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA", 1e-3, "KB"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock", 1e-9, "GHz"),
]


def _num(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return None


def launch_list(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Value" in r)
    h = rows[hdr]
    kn, mv, mu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= mv:
            continue
        v = _num(r[mv])
        if v is None:
            continue
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(r[mu], 1e-3)
        name = r[kn].split("(")[0]
        c, t = tot.get(name, (0, 0.0))
        tot[name] = (c + 1, t + v * scale)
    all_t = sum(t for _, t in tot.values())
    n = sum(c for c, _ in tot.values())
    out = [f"| kernel | launches | total us | share |", "|---|---:|---:|---:|"]
    for k, (c, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k}` | {c} | {t:.1f} | {100 * t / all_t:.1f}% |")
    out.append(f"| **total** | {n} | {all_t:.1f} | |")
    return "\n".join(out)


def full_report(path, regex=None):
    cmd = ["ncu", "-i", path, "--page", "raw", "--csv"]
    if regex:
        cmd += ["--kernel-name", f"regex:{regex}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return "(no data)"
    h = rows[0]
    lines = []
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        name = r[h.index("Kernel Name")].split("(")[0] if "Kernel Name" in h else "?"
        lines.append(f"### `{name}`\n\n| metric | value |\n|---|---:|")
        for key, label, scale, unit in METRICS:
            if key in h:
                v = _num(r[h.index(key)])
                if v is not None:
                    lines.append(f"| {label} | {v * scale:.4g} {unit} |")
        if "dram__bytes_read.sum" in h and "gpu__time_duration.sum" in h:
            b = (_num(r[h.index("dram__bytes_read.sum")]) or 0) + (_num(r[h.index("dram__bytes_write.sum")]) or 0)
            t = _num(r[h.index("gpu__time_duration.sum")]) or 1
            lines.append(f"| dram GB/s (read+write / duration) | {b / t:.1f} |")
        lines.append("")
    return "\n".join(lines)


if __name__ == "__main__":
    p = sys.argv[1]
    print(launch_list(p) if p.endswith(".csv") else full_report(p, sys.argv[2] if len(sys.argv) > 2 else None))
