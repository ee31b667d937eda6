"""Interleaves device-resident and host-buffer (e2e) sk.net process() steps to separate a
systematic e2e overhead from clock drift. Scratch measurement, not a bench line."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1509_03371_b200 as g  # noqa: E402
from paper_1509_03371_b200 import _lib  # noqa: E402
import bench  # noqa: E402

spec = g.parse_netspec_or_throw(bench.net_text("sk"))
states = g.init_weights(spec, 1)
proc = g.Processor(spec, states)
net = proc.net.h
H = W = 1024
img = g.Rng(55).index_array_u8(H * W, 256).reshape(H, W)
dev = torch.device("cuda", 0)
img_d = torch.from_numpy(img).to(dev)
lab_d = torch.empty((H, W), dtype=torch.uint8, device=dev)
prob_d = torch.empty((2, H, W), dtype=torch.float32, device=dev)
img_h = torch.from_numpy(img).pin_memory()
lab_h = torch.empty((H, W), dtype=torch.uint8).pin_memory()
prob_h = torch.empty((2, H, W), dtype=torch.float32).pin_memory()
stream = torch.cuda.ExternalStream(_lib.lib().graft_net_stream(net), device=dev)


def dev_step():
    proc.run(img_d, 128, 101, lab_d, prob_d, mem=_lib.MEM_DEVICE)


def host_step():
    _lib.check(_lib.lib().graft_process(net, img_h.data_ptr(), H, W, 128, 101, lab_h.data_ptr(),
                                        prob_h.data_ptr(), _lib.MEM_HOST))


def timed(f):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    f()
    e1.record(stream)
    e1.synchronize()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3


import ctypes
L = len(spec.layers)


def layer_ms():
    ms = (ctypes.c_double * L)()
    runs = (ctypes.c_longlong * L)()
    _lib.check(_lib.lib().graft_net_layer_stats(net, ms, runs, L))
    return {l.name: round(ms[i], 1) for i, l in enumerate(spec.layers) if ms[i] > 0.5}


for _ in range(3):
    dev_step()
    host_step()
proc.net.set_option(_lib.OPT_TIMED, 1)
for i in range(10):
    _lib.check(_lib.lib().graft_net_reset_stats(net))
    d = timed(dev_step)
    dl = layer_ms()
    _lib.check(_lib.lib().graft_net_reset_stats(net))
    h = timed(host_step)
    hl = layer_ms()
    print(f"iter {i}: device {d[0]:.1f}/{d[1]:.1f} {dl} | host {h[0]:.1f}/{h[1]:.1f} {hl}", flush=True)
mg = []
for _ in range(20):
    t0 = time.perf_counter()
    torch.cuda.mem_get_info()
    mg.append((time.perf_counter() - t0) * 1e3)
print("mem_get_info ms: min %.3f med %.3f max %.3f" % (min(mg), sorted(mg)[10], max(mg)))
