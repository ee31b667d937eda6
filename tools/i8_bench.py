"""Throughput of the exact int8 tcgen05 GEMM (graft_gemm_i8) on the ip1-sized digit-plane GEMM:
M = 1024 (f_out), N = 16384 or 1M (pixels), K = 19200 (taps x channels)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_03371_b200 import _lib  # noqa: E402

for M, N, K in ((1024, 16384, 19200), (1024, 131072, 19200)):
    a = torch.randint(-128, 128, (M, K), dtype=torch.int8, device="cuda")
    b = torch.randint(0, 256, (N, K), dtype=torch.uint8, device="cuda")
    c = torch.empty((M, N), dtype=torch.int32, device="cuda")
    best = 1e9
    for _ in range(4):
        torch.cuda.synchronize()
        t = time.perf_counter()
        _lib.check(_lib.lib().graft_gemm_i8(a.data_ptr(), 1, b.data_ptr(), M, N, K, c.data_ptr()))
        best = min(best, time.perf_counter() - t)
    print(f"gemm_i8 {M}x{N}x{K}: {best * 1e3:.2f} ms  {2.0 * M * N * K / best / 1e12:.0f} TOPS", flush=True)
