"""Batches of independent images (BASELINE.json configs[3]) through
graft_process_batch vs one process() call per image: sk.net, tile 128 (or the image side),
N images of side s with N*s^2 = 2^22 labels per batch, device-resident, CUDA events.
Prints one JSON line per image side."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1509_03371_b200 as g  # noqa: E402
from paper_1509_03371_b200 import _lib  # noqa: E402

V = 101
spec = g.parse_netspec_or_throw(bench.sk_text())
states = g.init_weights(spec, 1)
dev = torch.device("cuda", 0)
modes = {"exact": g.Processor(spec, states), "tc_bf16": g.Processor(spec, states, tensor_cores="bf16")}


def timed(fn, proc):
    stream = torch.cuda.ExternalStream(_lib.lib().graft_net_stream(proc.net.h), device=dev)
    fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    fn()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e-3


for side in (128, 256, 512):
    n = (1 << 22) // (side * side)
    imgs = np.stack([g.Rng(55 + i).index_array_u8(side * side, 256).reshape(side, side) for i in range(n)])
    imgs_d = torch.from_numpy(imgs).to(dev)
    lab = torch.empty((n, side, side), dtype=torch.uint8, device=dev)
    prob = torch.empty((n, 2, side, side), dtype=torch.float32, device=dev)
    w = min(128, side)
    line = {"image": [side, side], "images": n, "labels": n * side * side}
    for name, proc in modes.items():
        tb = timed(lambda: proc.run_batch(imgs_d, w, V, lab, prob, mem=_lib.MEM_DEVICE), proc)
        lab1 = torch.empty((side, side), dtype=torch.uint8, device=dev)
        prob1 = torch.empty((2, side, side), dtype=torch.float32, device=dev)

        def each():
            for i in range(n):
                proc.run(imgs_d[i], w, V, lab1, prob1, mem=_lib.MEM_DEVICE)

        ts = timed(each, proc)
        line[name] = {"batch_labels_per_s": n * side * side / tb,
                      "per_image_calls_labels_per_s": n * side * side / ts}
    print(json.dumps(line), flush=True)
