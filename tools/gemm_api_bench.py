"""Throughput of the layer API's gemm (graft_gemm_f32 / _f64, tensor.hpp:151-169) on device
buffers: f32 operands run on the DMMA gemm (products exact in fp64, the reference's ascending
chain), f64 operands on the DMUL+DADD kernel (the reference rounds each product; DMMA would
fuse it). Prints one JSON line per shape with ms and TFLOP/s (2*m*n*k per call), and checks the
f32 result against the f64-accumulated reference chain on a sample of entries.

    python tools/gemm_api_bench.py
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_03371_b200 import _lib  # noqa: E402


def bench(dtype, m, n, k, ta=0, tb=0, reps=5):
    dev = torch.device("cuda", 0)
    td = torch.float32 if dtype == "f32" else torch.float64
    g = torch.Generator(device=dev).manual_seed(1)
    a = torch.randn(m * k, device=dev, dtype=td, generator=g)
    b = torch.randn(k * n, device=dev, dtype=td, generator=g)
    c = torch.zeros(m * n, device=dev, dtype=td)
    fn = _lib.lib().graft_gemm_f32 if dtype == "f32" else _lib.lib().graft_gemm_f64
    stream = torch.cuda.ExternalStream(_lib.lib().graft_stream(), device=dev)

    def call():
        _lib.check(fn(ta, tb, m, n, k, 1.0, a.data_ptr(), b.data_ptr(), 0.0, c.data_ptr(), _lib.MEM_DEVICE))

    call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        call()
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ok = None
    if dtype == "f32":  # sample: the reference chain in fp64 (products of floats exact), then float
        A = a.view(m, k).double().cpu().numpy()
        B = b.view(k, n).double().cpu().numpy()
        C = c.view(m, n).cpu().numpy()
        rows = np.arange(0, m, max(1, m // 7))[:8]
        cols = np.arange(0, n, max(1, n // 7))[:8]
        ok = True
        for i in rows:
            for j in cols:
                acc = 0.0
                for kk in range(k):
                    acc += A[i, kk] * B[kk, j]
                ok &= np.float32(acc) == C[i, j]
    return {"gemm": dtype, "m": m, "n": n, "k": k, "ms": ms, "tflops": 2.0 * m * n * k / (ms * 1e-3) / 1e12,
            "sample_bit_exact": None if ok is None else bool(ok)}


def main():
    _lib.check(_lib.lib().graft_set_device(0))
    for dt, shape in (("f32", (4096, 4096, 4096)), ("f32", (1024, 65536, 576)), ("f64", (2048, 2048, 2048))):
        print(json.dumps(bench(dt, *shape)), flush=True)


if __name__ == "__main__":
    main()
