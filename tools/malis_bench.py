"""Batched MALIS throughput: malis_softmax_loss over B independent
h x w patches on one B200 (one launch, device buffers, CUDA events) against the reference's
malis_softmax_loss (oracle/_ref) on the host, one patch per host thread call, all cores.

    python tools/malis_bench.py [--patch 64] [--batch 1184] [--steps 5]

Prints one JSON line: patches/s on the GPU (device-resident and end to end with host buffers),
the reference's patches/s on `cores` threads, and a bit-exactness spot check of the batch
against the reference.
"""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--patch", type=int, default=64)
    ap.add_argument("--batch", type=int, default=148 * 8)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--cpu-patches", type=int, default=0, help="0 = 4 per host core")
    args = ap.parse_args()
    import torch

    from paper_1509_03371_b200 import _lib
    from paper_1509_03371_b200 import malis as M
    from oracle import oracle as O

    B, h = args.batch, args.patch
    rng = np.random.default_rng(1)
    fg = (rng.random((B, h, h)) < 0.5).astype(np.uint8)
    scores = rng.uniform(-2, 2, (B, 2, h, h)).astype(np.float32)
    dev = torch.device("cuda", 0)
    _lib.check(_lib.lib().graft_set_device(0))
    stream = torch.cuda.ExternalStream(_lib.lib().graft_stream(), device=dev)
    sd = torch.from_numpy(scores).to(dev)
    fd = torch.from_numpy(fg).to(dev)
    dd = torch.zeros_like(sd)
    ld = torch.zeros(B, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()

    def run_dev():
        _lib.check(_lib.lib().graft_malis_softmax_loss_f32(sd.data_ptr(), B, 2, h, h, fd.data_ptr(), dd.data_ptr(),
                                                           ld.data_ptr(), _lib.MEM_DEVICE))

    run_dev()
    torch.cuda.synchronize()
    ms = []
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run_dev()
        e1.record(stream)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    dev_ps = B / (np.median(ms) * 1e-3)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        losses, diff = M.malis_softmax_loss_batch(scores, fg)
    e2e_ps = B * args.steps / (time.perf_counter() - t0)

    # reference on the host cores: independent patches, one reference call per patch per thread
    cores = os.cpu_count() or 1
    n_cpu = args.cpu_patches or 4 * cores
    n_cpu = min(n_cpu, B)
    chk = []

    def work(i0):
        for i in range(i0, n_cpu, cores):
            lw, dw = O.malis_softmax_loss(scores[i], fg[i], None, "ref")
            chk.append((i, lw, dw))

    ths = [threading.Thread(target=work, args=(t,)) for t in range(cores)]
    t0 = time.perf_counter()
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    cpu_s = time.perf_counter() - t0
    cpu_ps = n_cpu / cpu_s
    exact = all(losses[i] == lw and np.array_equal(diff[i].view(np.uint32), dw.view(np.uint32)) for i, lw, dw in chk)
    print(json.dumps({
        "metric": "malis_softmax_loss patches/s", "patch": [h, h], "batch": B, "dtype": "f32",
        "gpu_device_patches_per_s": dev_ps, "gpu_ms_per_batch": float(np.median(ms)),
        "gpu_e2e_patches_per_s": e2e_ps,
        "cpu_reference_patches_per_s": cpu_ps, "cpu_cores": cores, "cpu_patches": n_cpu,
        "speedup_device_vs_cpu": dev_ps / cpu_ps, "bit_exact_vs_reference": exact,
        "gpu_launches_per_batch": 1,
    }))


if __name__ == "__main__":
    main()
