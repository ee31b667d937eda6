"""Layer-level race probe: graft_conv_crt_f32 on an ip1-like input, repeated under concurrent
memory traffic; compares output bits and fallback counts with the DMMA conv."""
import os, sys, threading, time
sys.path.insert(0, '.')
import torch
from paper_1509_03371_b200 import _lib
sys.path.insert(0, 'tests')
from test_gpu_crt import exact_conv, crt_conv, make
case = tuple(int(v) for v in os.environ.get("CASE", "6,192,252,252,1024,10,8").split(",")) + ("pool",)
B, C, H, W, M, k, d, _ = case
x, w, bias = make(case, seed=3)
ref = exact_conv(x, w, bias, k, d, True)
stop = False
def hammer():
    s = torch.cuda.Stream()
    a = torch.empty(1 << 28, dtype=torch.float32, device='cuda'); b = torch.empty_like(a)
    with torch.cuda.stream(s):
        while not stop:
            b.copy_(a); a.add_(1.0); s.synchronize()
bad = 0
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for it in range(n):
    stop = False
    th = threading.Thread(target=hammer); th.start(); time.sleep(0.02)
    got, nf = crt_conv(x, w, bias, k, d, True)
    torch.cuda.synchronize()
    stop = True; th.join()
    dd = int((got.view(torch.int32) != ref.view(torch.int32)).sum())
    bad += dd > 0
    print(f"{os.environ.get('TAG','')} iter {it} fallbacks {nf} diff {dd}", flush=True)
print(os.environ.get('TAG',''), "BAD", bad, "of", n)
