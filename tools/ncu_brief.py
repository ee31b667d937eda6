"""Brief of one ncu --set full report: SOL, occupancy, issue, top stall reasons, instruction mix."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h, u, v = r[0], r[1], r[2]
d = {n: (val, un) for n, un, val in zip(h, u, v)}


def g(n):
    x = d.get(n, ("nan", ""))[0].replace(",", "")
    try:
        return float(x)
    except ValueError:
        return float("nan")


print("duration ms", g("gpu__time_duration.sum") / 1e6)
for n in ["sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
          "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
          "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
          "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]:
    print(n, g(n))
st = [(n, g(n)) for n in h if n.startswith("smsp__average_warp_latency_issue_stalled") and n.endswith(".ratio")]
st = [(n, x) for n, x in st if x == x]
for n, x in sorted(st, key=lambda t: -t[1])[:8]:
    print("stall", n.replace("smsp__average_warp_latency_issue_stalled_", ""), round(x, 3))
ops = [(n, g(n)) for n in h if n.startswith("smsp__sass_inst_executed_op_") and n.endswith(".sum")]
for n, x in sorted(ops, key=lambda t: -t[1])[:8]:
    print("op", n, x)
