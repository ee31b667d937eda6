"""Times the tolerance-mode tcgen05 conv (graft_conv_tc_f32) on the ip1 shape of sk.net at a
1024-px tile: 192 x 1096^2 -> 1024 x 1024^2, k10 d8 (41.23 TFLOP). Wall clock around the
synchronising C call (layout conversions included), best of N."""
import sys
import time
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_03371_b200 import _lib  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "ip1"
S = {"ip1": (1, 192, 1096, 1096, 1024, 10, 8), "ip2": (1, 1024, 1024, 1024, 512, 1, 1),
     "conv3": (1, 128, 1112, 1112, 192, 3, 4), "small": (1, 192, 200, 200, 1024, 10, 8)}[shape]
B, C, H, W, M, k, d = S
x = torch.rand(B, C, H, W, device="cuda")
w = torch.randn(M, C, k, k, device="cuda") * 0.01
b = torch.zeros(M, device="cuda")
OH, OW = H - (k - 1) * d, W - (k - 1) * d
out = torch.empty(B, M, OH, OW, device="cuda")
flops = 2.0 * M * C * k * k * OH * OW * B
for kind, name in ((_lib.TC_BF16, "bf16"), (_lib.TC_TF32, "tf32"), (_lib.TC_BF16X3, "bf16x3")):
    best = 1e9
    for it in range(4):
        torch.cuda.synchronize()
        t = time.perf_counter()
        _lib.check(_lib.lib().graft_conv_tc_f32(kind, x.data_ptr(), B, C, H, W, w.data_ptr(),
                                                b.data_ptr(), M, k, d, out.data_ptr(), 0))
        best = min(best, time.perf_counter() - t)
    print(f"{shape} {name}: {best * 1e3:.2f} ms  {flops / best / 1e12:.1f} TFLOP/s", flush=True)
