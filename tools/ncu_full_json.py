"""Extract the roofline-relevant metrics of a one-kernel `ncu --set full` report into JSON:
python tools/ncu_full_json.py report.ncu-rep out.json [algorithmic_bytes_per_launch]."""
import csv
import json
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h, u, v = r[0], r[1], r[2]
keep = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active"]
res = {}
for n, un, val in zip(h, u, v):
    if n in keep or ("pipe" in n and "tc" in n and n.endswith("pct_of_peak_sustained_active")):
        res[n] = {"value": val, "unit": un}


def num(k):
    x = res[k]["value"].replace(",", "")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(res[k]["unit"], 1)
    return float(x) * scale


res["traffic_bytes_per_launch"] = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
if len(sys.argv) > 3:
    res["algorithmic_bytes_per_launch"] = float(sys.argv[3])
json.dump(res, open(sys.argv[2], "w"), indent=1)
print(json.dumps({k: res[k] for k in list(res)[:40]}, indent=0)[:3000])
