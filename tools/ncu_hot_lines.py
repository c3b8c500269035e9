"""Top source lines of a kernel by warp-stall samples, from an ncu report with -lineinfo source.

    python tools/ncu_hot_lines.py report.ncu-rep [kernel_substring] [n]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else ""
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur_file = func = None
agg, src = collections.Counter(), {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        func = r[1]
        continue
    if r[0] in ("Line No",) or not r[0] or not func or kern not in func:
        continue
    try:
        agg[(cur_file, int(r[0]))] += int(r[4])
        src[(cur_file, int(r[0]))] = r[1][:110]
    except (ValueError, IndexError):
        pass
tot = sum(agg.values())
print(f"{rep}: {tot} samples in {kern or 'all kernels'}")
for k, v in agg.most_common(n):
    print(f"{100.0 * v / max(tot, 1):5.1f}% {k[0]}:{k[1]}  {src[k]}")
