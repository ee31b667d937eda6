"""A/B of the exact paths on the bench workload (sk.net process() of a 1024^2 image): DMMA chain
everywhere (crt_min_k 0) vs the int8 tensor-core certification path on large-K convs. Prints
ms per step, per-layer device ms and whether labels and probability planes are bit-identical
between the modes. GPU only: python tools/crt_ab.py [--size 1024] [--min-k 0 4096 1024]."""
import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1509_03371_b200 as g  # noqa: E402
from paper_1509_03371_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--min-k", type=int, nargs="+", default=[0, 4096])
    args = ap.parse_args()
    spec = g.parse_netspec_or_throw(bench.sk_text())
    states = g.init_weights(spec, 1)
    H = W = args.size
    img = g.Rng(55).index_array_u8(H * W, 256).reshape(H, W)
    dev = torch.device("cuda", 0)
    img_d = torch.from_numpy(img).to(dev)
    results = {}
    for mk in args.min_k:
        proc = g.Processor(spec, states)
        proc.net.set_option(_lib.OPT_CRT_MIN_K, mk)
        net = proc.net.h
        C = proc.n_classes
        lab = torch.empty((H, W), dtype=torch.uint8, device=dev)
        prob = torch.empty((C, H, W), dtype=torch.float32, device=dev)
        stream = torch.cuda.ExternalStream(_lib.lib().graft_net_stream(net), device=dev)
        for _ in range(2):
            proc.run(img_d, 128, bench.V, lab, prob, mem=_lib.MEM_DEVICE)
        torch.cuda.synchronize()
        proc.net.set_option(_lib.OPT_TIMED, 1)
        _lib.check(_lib.lib().graft_net_reset_stats(net))
        tot = 0.0
        for _ in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            proc.run(img_d, 128, bench.V, lab, prob, mem=_lib.MEM_DEVICE)
            e1.record(stream)
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        proc.net.set_option(_lib.OPT_TIMED, 0)
        L = len(spec.layers)
        ms = (ctypes.c_double * L)()
        runs = (ctypes.c_longlong * L)()
        _lib.check(_lib.lib().graft_net_layer_stats(net, ms, runs, L))
        per_layer = {spec.layers[i].name: round(ms[i] / args.steps, 2) for i in range(L) if ms[i] > 0.05 * args.steps}
        step = tot / args.steps
        fb = proc.net.get_option(_lib.OPT_CRT_FALLBACKS) if mk else 0
        cms = (ctypes.c_double * 4)()
        cl = ctypes.c_longlong()
        _lib.check(_lib.lib().graft_net_crt_stats(net, cms, ctypes.byref(cl)))
        crt_ms = [round(x / args.steps, 2) for x in cms]
        results[mk] = (lab.cpu().numpy(), prob.cpu().numpy())
        same = ""
        if len(results) > 1:
            l0, p0 = results[args.min_k[0]]
            same = (f" labels identical {np.array_equal(l0, results[mk][0])}, probs bit-identical "
                    f"{np.array_equal(p0.view(np.uint32), results[mk][1].view(np.uint32))}")
        print(json.dumps({"crt_min_k": mk, "ms_per_step": round(step, 2),
                          "labels_per_s": round(H * W / (step * 1e-3)), "chain_fallbacks": fb, "crt_ms_prep_gemm_certify_chain": crt_ms,
                          "layers_ms": per_layer}) + same,
              flush=True)
        del proc


if __name__ == "__main__":
    main()
