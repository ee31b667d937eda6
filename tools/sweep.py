"""Input-size sweep (BASELINE.json configs[4]): sk.net process() of gray u8
images with H*W = 2^n px (H = W = 2^(n/2) for even n, W = 2H for odd n; pixels Rng(55)), tile
w = min(128, H, W) as the reference's CLI would use, v = 101. Per size: exact-mode labels/s
(device-resident, CUDA events, L2 flushed), the tolerance mode's labels/s and its label
agreement with the exact planes, and the reference's CPU rate on all host cores -- measured
once on a bounded sample (bench.cpu_reference_sample) and scaled by FLOP/label to each size's
tiling (marked "extrapolated"). One JSON line per size.

    python tools/sweep.py [--min 10] [--max 30] [--tc-max 30] [--cpu]

Each line also carries the nvidia-smi clock samples (median SM clock, throttle reasons) taken
during that size's timed runs (bench.ClockSampler).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--min", type=int, default=10)
ap.add_argument("--max", type=int, default=30)
ap.add_argument("--tc-max", type=int, default=30)
ap.add_argument("--cpu", action="store_true")
a = ap.parse_args()

import torch  # noqa: E402

import paper_1509_03371_b200 as g  # noqa: E402
from paper_1509_03371_b200 import _lib  # noqa: E402

V = 101
spec = g.parse_netspec_or_throw(bench.sk_text())
states = g.init_weights(spec, 1)
dev = torch.device("cuda", 0)
_lib.check(_lib.lib().graft_set_device(0))
exact = g.Processor(spec, states)
tc = g.Processor(spec, states, tensor_cores="bf16")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

cpu = None
if a.cpu:
    threads = os.cpu_count() or 1
    r = bench.cpu_reference_sample(threads, 8)
    cpu = {"flop_per_s": r["flops"] / r["wall"], "threads": threads, "kind": r["kind"],
           "sample": f"{threads} threads x one 8x8-label sk.net forward, {r['wall']:.1f} s"}


def timed(proc, img_d, lab, prob, w):
    stream = torch.cuda.ExternalStream(_lib.lib().graft_net_stream(proc.net.h), device=dev)
    flush.fill_(1)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    proc.run(img_d, w, V, lab, prob, mem=_lib.MEM_DEVICE)
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e-3


for n in range(a.min, max(a.max, a.tc_max) + 1):
    H = 1 << (n // 2)
    W = H * (2 if n % 2 else 1)
    w = min(128, H, W)
    img = g.Rng(55).index_array_u8(H * W, 256).reshape(H, W)
    img_d = torch.from_numpy(img).to(dev)
    lab = torch.empty((H, W), dtype=torch.uint8, device=dev)
    prob = torch.empty((2, H, W), dtype=torch.float32, device=dev)
    lab_t = torch.empty_like(lab)
    prob_t = torch.empty_like(prob)
    line = {"log2_px": n, "H": H, "W": W, "tile": w}
    clocks = bench.ClockSampler(0)
    clocks.start()
    try:
        if n <= a.max:
            if H * W <= (1 << 22):
                exact.run(img_d, w, V, lab, prob, mem=_lib.MEM_DEVICE)  # warm-up at small sizes
            t = timed(exact, img_d, lab, prob, w)
            line["exact_labels_per_s"] = H * W / t
            line["exact_s"] = t
            line["internal_tile"] = exact.last_tile()
        if n <= a.tc_max:
            if H * W <= (1 << 22):
                tc.run(img_d, w, V, lab_t, prob_t, mem=_lib.MEM_DEVICE)
            t = timed(tc, img_d, lab_t, prob_t, w)
            line["tc_bf16_labels_per_s"] = H * W / t
            line["tc_bf16_s"] = t
            if "exact_labels_per_s" in line:
                line["tc_label_agreement"] = (lab_t == lab).double().mean().item()
                line["tc_max_abs_prob_diff"] = (prob_t - prob).abs().max().item()
    except Exception as e:  # report and continue (e.g. out of memory at the largest sizes)
        line["error"] = str(e)[:200]
    line["clocks"] = clocks.stop()
    if cpu:
        wi = w if min(H, W) >= w else min(H, W)
        fpl = g.flop_estimate(spec, wi + V)["total"] / (wi * wi)
        line["cpu_reference_labels_per_s"] = cpu["flop_per_s"] / fpl
        line["cpu_reference_note"] = ("extrapolated: " + cpu["sample"] + f", {cpu['kind']}, "
                                      f"scaled by FLOP/label at tile {wi}")
    print(json.dumps(line), flush=True)
    del img_d, lab, prob, lab_t, prob_t
    torch.cuda.empty_cache()
