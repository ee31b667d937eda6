"""ip2-shaped conv (C=1024 -> 512, 1x1) on the int8 exact path vs the DMMA chain, device buffers,
CUDA-event timed; plus the conv3 shape (128 -> 192, k3 d4). Prints ms and fallbacks."""
import ctypes, json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1509_03371_b200 import _lib

L = _lib.lib()
_lib.check(L.graft_set_device(0))
st = torch.cuda.ExternalStream(L.graft_stream(), device=torch.device("cuda", 0))
out = {}
for name, (C, H, W, M, k, d) in {"ip2": (1024, 512, 512, 512, 1, 1), "conv3": (128, 520, 520, 192, 3, 4),
                                 "conv2": (48, 520, 520, 128, 5, 2)}.items():
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.rand(C, H, W, device="cuda", generator=g) ** 3 * 0.04
    w = torch.randn(M, C, k, k, device="cuda", generator=g) * (2.0 / (C * k * k)) ** 0.5
    b = torch.zeros(M, device="cuda")
    OH, OW = H - (k - 1) * d, W - (k - 1) * d
    y = torch.empty(M, OH, OW, device="cuda")
    nf = ctypes.c_ulonglong()
    def crt():
        _lib.check(L.graft_conv_crt_f32(x.data_ptr(), 1, C, H, W, w.data_ptr(), b.data_ptr(), M, k, d, y.data_ptr(), 1, ctypes.byref(nf)))
    def dmma():
        _lib.check(L.graft_conv_sk_forward_f32(x.data_ptr(), C, H, W, w.data_ptr(), w.numel(), b.data_ptr(), M, M, k, d, 1, 0, y.data_ptr(), _lib.MEM_DEVICE))
    for fn_name, fn in (("crt", crt), ("dmma", dmma)):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(3):
            fn()
        e1.record(st); e1.synchronize()
        out[f"{name}_{fn_name}_ms"] = e0.elapsed_time(e1) / 3
    out[f"{name}_fallbacks"] = nf.value
print(json.dumps(out))
