"""Aggregate an ncu --csv launch list (gpu__time_duration and dram bytes) per kernel name."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
agg = defaultdict(lambda: defaultdict(float))
cnt = defaultdict(int)
for r in rows[hdr + 1:]:
    name = r[ki].replace("<unnamed>", "anon").split("(")[0].split("<")[0].replace("void ", "").split("::")[-1]
    agg[name][r[mi]] += float(r[vi].replace(",", ""))
    if r[mi] == "gpu__time_duration.sum":
        cnt[name] += 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
    n = cnt[k]
    print(f"{k:28s} launches {n:4d}  ms/launch {v['gpu__time_duration.sum'] / n / 1e6:9.3f}  "
          f"DRAM rd GB/launch {v.get('dram__bytes_read.sum', 0) / n / 1e9:8.2f}  wr {v.get('dram__bytes_write.sum', 0) / n / 1e9:8.2f}")
