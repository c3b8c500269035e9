"""Summarise a gpurun_out/<tag>/ directory (ncu launch list + --set full captures) as markdown.

    python tools/ncu_summary.py gpurun_out/r01a > profiles/r01_ncu_summary.md
"""
import collections
import csv
import glob
import io
import os
import subprocess
import sys

D = sys.argv[1]


def launch_list(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(a[1] for a in agg.values())
    print(f"Launch list `{os.path.basename(path)}`: {sum(a[0] for a in agg.values())} launches, "
          f"{tot / 1000:.2f} ms summed device time (ncu, serialised, cold caches: compare shares)\n")
    print("| kernel | launches | total us | share |\n|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {n} | {t:.1f} | {100 * t / tot:.1f}% |")
    print()


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return
    h, units = rows[0], rows[1]
    idx = [h.index(w) for w in WANT if w in h]
    ki = h.index("Kernel Name")
    print(f"`{os.path.basename(path)}` (ncu --set full):\n")
    print("| kernel | " + " | ".join(f"{h[i]} [{units[i]}]" for i in idx) + " |")
    print("|---" * (len(idx) + 1) + "|")
    for r in rows[2:]:
        name = r[ki].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        print(f"| `{name}` | " + " | ".join(r[i] for i in idx) + " |")
    print()


print(f"# ncu summary: {D}\n")
for p in sorted(glob.glob(os.path.join(D, "*launches*.csv"))):
    launch_list(p)
for p in sorted(glob.glob(os.path.join(D, "*.ncu-rep"))):
    full(p)
