"""Per-source-line instruction / stall summary of one kernel in an ncu report.
usage: ncu_lines.py REPORT KERNEL_REGEX [launch_index] [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
idx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kern}", "--launch-skip", str(idx), "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = collections.defaultdict(lambda: [0.0, 0.0])
src, fname, cur = {}, None, None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] == "Line No":
        continue
    if r[0]:
        cur = (fname, r[0])
        src[cur] = r[1]
    try:
        agg[cur][0] += float(r[7] or 0)
        agg[cur][1] += float(r[4] or 0)
    except ValueError:
        pass
tot = sum(v[0] for v in agg.values()) or 1
tots = sum(v[1] for v in agg.values()) or 1
print(f"warp instructions {tot:.0f}, stall samples {tots:.0f}")
key = 0 if "--inst" in sys.argv else 1
for k, v in sorted(agg.items(), key=lambda x: -x[1][key])[:top]:
    print(f"{100 * v[0] / tot:5.1f}% inst {100 * v[1] / tots:5.1f}% stall  {k[0]}:{k[1]}  {src.get(k, '')[:100]}")
