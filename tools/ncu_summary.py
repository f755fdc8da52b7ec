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

# (metric, label, target unit); values are converted with the report's unit row
METRICS = [
    ("gpu__time_duration.sum", "duration", 1, "us"),
    ("dram__bytes_read.sum", "dram read", 1, "MB"),
    ("dram__bytes_write.sum", "dram write", 1, "MB"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput", 1, "% of peak"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput", 1, "% of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate", 1, "%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts", 1e-6, "M"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy", 1, "%"),
    ("launch__registers_per_thread", "registers/thread", 1, ""),
    ("launch__grid_size", "grid", 1, "CTAs"),
    ("launch__block_size", "block", 1, "threads"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA", 1e-3, "KB"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock", 1, "GHz"),
]

_UNIT = {("nsecond", "us"): 1e-3, ("usecond", "us"): 1.0, ("msecond", "us"): 1e3,
         ("ns", "us"): 1e-3, ("us", "us"): 1.0, ("ms", "us"): 1e3,
         ("byte", "MB"): 1e-6, ("Kbyte", "MB"): 1e-3, ("Mbyte", "MB"): 1.0, ("Gbyte", "MB"): 1e3,
         ("hz", "GHz"): 1e-9, ("Khz", "GHz"): 1e-6, ("Mhz", "GHz"): 1e-3, ("Ghz", "GHz"): 1.0,
         ("cycle/nsecond", "GHz"): 1.0, ("cycle/usecond", "GHz"): 1e-3, ("cycle/second", "GHz"): 1e-9,
         ("Kbyte", "KB"): 1.0, ("byte", "KB"): 1e-3}


def _conv(v, unit, target, scale=1.0):
    return v * _UNIT.get((unit, target), scale)


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
    h, units = rows[0], rows[1]
    lines = []
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        name = r[h.index("Kernel Name")].split("(")[0] if "Kernel Name" in h else "?"
        val = {}
        for key, label, scale, unit in METRICS:
            if key in h:
                v = _num(r[h.index(key)])
                if v is not None:
                    val[key] = _conv(v, units[h.index(key)], unit, scale)
        lines.append(f"### `{name}`\n\n| metric | value |\n|---|---:|")
        for key, label, _, unit in METRICS:
            if key in val:
                lines.append(f"| {label} | {val[key]:.4g} {unit} |")
        if "dram__bytes_read.sum" in val and "gpu__time_duration.sum" in val:
            b = val["dram__bytes_read.sum"] + val.get("dram__bytes_write.sum", 0)
            lines.append(f"| dram GB/s ((read+write) / duration) | {b / val['gpu__time_duration.sum'] * 1e3:.1f} |")
        st = []
        for k, v in zip(h, r):
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                x = _num(v)
                if x:
                    st.append((x, k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        st.sort(reverse=True)
        if st:
            lines.append("| top stalls (warps per issue) | " + ", ".join(f"{n} {x:.2f}" for x, n in st[:5]) + " |")
        lines.append("")
    return "\n".join(lines)


if __name__ == "__main__":
    p = sys.argv[1]
    print(launch_list(p) if p.endswith(".csv") else full_report(p, sys.argv[2] if len(sys.argv) > 2 else None))
