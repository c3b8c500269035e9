"""Per-launch DRAM traffic of one kernel family from an ncu metrics CSV (one profiled step).

    python tools/gemm_traffic.py gpurun_out/r01d/gemm_traffic.csv [name-substring] > profiles/gemm_traffic.json
bench.py reports the mean as roofline.traffic next to the per-launch algorithmic FLOPs (verify
GEMMs), and the acceptance / compaction kernels' achieved GB/s from their measured bytes."""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ID, KN, MN, MU, MV = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
per = collections.defaultdict(dict)
names = {}
for r in rows[hi + 1:]:
    if len(r) <= MV:
        continue
    v = float(r[MV].replace(",", ""))
    if r[MN].startswith("dram__bytes"):
        v *= unit.get(r[MU], 1.0)
    per[r[ID]][r[MN]] = v
    names[r[ID]] = r[KN].split("(")[0].replace("void ", "").replace("unnamed>::", "")
key = sys.argv[2] if len(sys.argv) > 2 else "gemm"
launches = [(names[i], m) for i, m in per.items() if key in names[i]]
tot = [m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for _, m in launches]
by = collections.defaultdict(list)
for (n, m), t in zip(launches, tot):
    by[n].append(t)
print(json.dumps({"dram_bytes_per_launch": sum(tot) / max(1, len(tot)), "launches": len(tot),
                  "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over one step "
                            f"(kernels matching {key!r}), mean over launches",
                  "by_kernel": {k: {"n": len(v), "mean_bytes": sum(v) / len(v)} for k, v in sorted(by.items())}},
                 indent=1))
