"""Which layer of process() differs under concurrent load? KEEP_BLOBS, read every blob back."""
import numpy as np, sys, threading, time, ctypes as C
sys.path.insert(0, '.')
import torch
import paper_1509_03371_b200 as g
from paper_1509_03371_b200 import _lib
spec = g.parse_netspec_or_throw(bytes(np.load('tests/golden/configs.npz')['sk']).decode())
states = g.init_weights(spec, 1)
imgs = np.stack([g.Rng(7 + i).index_array_u8(200 * 180, 256).reshape(200, 180) for i in range(3)])
crt = int(sys.argv[1]) if len(sys.argv) > 1 else 0
proc = g.Processor(spec, states)
proc.net.set_option(_lib.OPT_KEEP_BLOBS, 1)
proc.net.set_option(_lib.OPT_CRT_MIN_K, crt)
names = [l.output for l in spec.layers[1:-1]]
def blobs():
    out = {}
    for nm in names:
        c, h, w = C.c_int(), C.c_int(), C.c_int()
        if _lib.lib().graft_net_blob_shape(proc.net.h, nm.encode(), C.byref(c), C.byref(h), C.byref(w)) != 0:
            continue
        # batch: B x C x H x W
        B = 6
        a = np.empty(B * c.value * h.value * w.value, np.float32)
        if _lib.lib().graft_net_blob_f32(proc.net.h, nm.encode(), _lib.ptr(a), 0) == 0:
            out[nm] = a
    return out
_, p0 = proc.run_batch(imgs, 128, 101)
ref = blobs()
stop = False
def hammer():
    s = torch.cuda.Stream()
    a = torch.empty(1 << 28, dtype=torch.float32, device='cuda'); b = torch.empty_like(a)
    with torch.cuda.stream(s):
        while not stop:
            b.copy_(a); a.add_(1.0); s.synchronize()
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 6):
    stop = False
    th = threading.Thread(target=hammer); th.start(); time.sleep(0.05)
    _, p = proc.run_batch(imgs, 128, 101)
    stop = True; th.join()
    got = blobs()
    first = [(nm, int((got[nm].view(np.uint32) != ref[nm].view(np.uint32)).sum())) for nm in names if nm in got]
    print(f"iter {it} probs diff {int((p.view(np.uint32) != p0.view(np.uint32)).sum())}", [f for f in first if f[1]], flush=True)
    for nm in ("conv2", "relu2", "pool2", "conv3"):
        if nm not in got: continue
        c, h, w = C.c_int(), C.c_int(), C.c_int()
        _lib.lib().graft_net_blob_shape(proc.net.h, nm.encode(), C.byref(c), C.byref(h), C.byref(w))
        dm = (got[nm].view(np.uint32) != ref[nm].view(np.uint32)).reshape(6, c.value, h.value, w.value)
        if dm.any():
            b_, m_, y_, x_ = np.nonzero(dm)
            print(f"   {nm}: tiles {np.unique(b_)} rows m {np.unique(m_)[:20]}.. ({len(np.unique(m_))} distinct) y {np.unique(y_)[:10]} x-range {x_.min()}..{x_.max()}", flush=True)
