"""Stress the int8 CRT path for nondeterminism: repeated runs under concurrent memory traffic
on another stream must all equal the DMMA chain's planes."""
import numpy as np, sys, os, threading, time
sys.path.insert(0, '.')
import torch
import paper_1509_03371_b200 as g
from paper_1509_03371_b200 import _lib
mode = sys.argv[1] if len(sys.argv) > 1 else "stress"
spec = g.parse_netspec_or_throw(bytes(np.load('tests/golden/configs.npz')['sk']).decode())
states = g.init_weights(spec, 1)
imgs = np.stack([g.Rng(7 + i).index_array_u8(200 * 180, 256).reshape(200, 180) for i in range(3)])
refp = g.Processor(spec, states, retile=0)
refp.net.set_option(_lib.OPT_CRT_MIN_K, 0)
ref = np.stack([refp.run(imgs[i], 128, 101)[1] for i in range(3)])
if mode == "dmma":
    proc = g.Processor(spec, states)
    proc.net.set_option(_lib.OPT_CRT_MIN_K, 0)
    _, probs = proc.run_batch(imgs, 128, 101)
    print("dmma batch diff", int((probs.view(np.uint32) != ref.view(np.uint32)).sum()), flush=True)
    sys.exit(0)
stop = False
def hammer():
    s = torch.cuda.Stream()
    a = torch.empty(1 << 28, dtype=torch.float32, device='cuda')
    b = torch.empty_like(a)
    with torch.cuda.stream(s):
        while not stop:
            b.copy_(a); a.add_(1.0)
            s.synchronize()
bad = 0
proc = g.Processor(spec, states)
if mode == "dmma-stress":
    proc.net.set_option(_lib.OPT_CRT_MIN_K, 0)
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
    th = None
    if it % 2 == 1:
        stop = False
        th = threading.Thread(target=hammer); th.start(); time.sleep(0.05)
    _, probs = proc.run_batch(imgs, 128, 101)
    if th is not None:
        stop = True; th.join()
    d = int((probs.view(np.uint32) != ref.view(np.uint32)).sum())
    fb = proc.net.get_option(_lib.OPT_CRT_FALLBACKS)
    bad += d > 0
    print(f"iter {it} hammer={it % 2} fallbacks={fb} diff={d}", flush=True)
print("BAD RUNS", bad)
