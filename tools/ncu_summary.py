"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file X` launch list: total
device time per kernel (sorted), launch counts and share."""
import collections
import csv
import io
import sys

txt = open(sys.argv[1]).read()
txt = txt[txt.index('"ID"'):]
rows = list(csv.DictReader(io.StringIO(txt)))
t = collections.defaultdict(float)
n = collections.Counter()
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    k = r["Kernel Name"].split("(")[0][:100]
    scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}.get(r.get("Metric Unit", "ns"), 1e-6)
    t[k] += float(r["Metric Value"].replace(",", "")) * scale
    n[k] += 1
tot = sum(t.values())
for k, v in sorted(t.items(), key=lambda x: -x[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{v:10.3f} ms {100 * v / tot:6.2f}%  n={n[k]:4d}  {k}")
print(f"{tot:10.3f} ms total")
