"""Statistics of ip1's activations (pool3) on the bench workload: how many patch values would
be inexact in a bx-bit fixed point scaled to the launch max, per output pixel, and the patch max
vs the launch max. Drives the choice of bw/bx for fewer CRT moduli."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
import paper_1509_03371_b200 as g
from paper_1509_03371_b200 import _lib

spec = g.parse_netspec_or_throw(bench.sk_text())
states = g.init_weights(spec, 1)
img = g.Rng(55).index_array_u8(1024 * 1024, 256).reshape(1024, 1024)
# the first internal tile's input: mirror_pad + normalize, 1125 x 1125 (process() at 1024)
pad = g.normalize_image(g.mirror_pad(g.Plane.from_array(img), 101)).view()
x = np.broadcast_to(pad[:1125, :1125], (3, 1125, 1125)).astype(np.float32).copy()
r = g.NetRunner(spec, states)
r.net.set_option(_lib.OPT_KEEP_BLOBS, 1)
r.forward(g.Blob.from_array(x))
p3 = torch.from_numpy(r.blob("pool3").view().copy()).cuda().double()  # [192][1124][1124]
xmax = p3.abs().max().item()
ex = int(np.floor(np.log2(xmax))) + 1
m, e = torch.frexp(p3)  # |x| = m 2^e, m in [0.5,1)
nz = p3 != 0
out = {"xmax": xmax, "ex": ex, "nonzero_frac": nz.double().mean().item()}
C, H, W = p3.shape
OH = H - 72
for bx in (36, 38, 40, 42, 44, 47):
    inex = (nz & ((e - 24) + bx - ex < 0)).float()  # per value
    per_px = inex.sum(0)  # [H][W] over channels
    # patch count over the 10 x 10 taps at dilation 8 for a sample of output rows
    cnt = torch.zeros(OH, W - 72, device=p3.device)
    for ky in range(10):
        for kx in range(10):
            cnt += per_px[8 * ky:8 * ky + OH, 8 * kx:8 * kx + W - 72]
    out[f"bx{bx}"] = {"inexact_value_frac": inex.mean().item(), "patch_inexact_mean": cnt.mean().item(),
                      "patch_inexact_max": cnt.max().item()}
pm = p3.abs().amax(0)
pmax = torch.zeros(OH, W - 72, device=p3.device)
psum = torch.zeros(OH, W - 72, device=p3.device, dtype=torch.float64)
ps = p3.abs().sum(0)
for ky in range(10):
    for kx in range(10):
        pmax = torch.maximum(pmax, pm[8 * ky:8 * ky + OH, 8 * kx:8 * kx + W - 72].float())
        psum += ps[8 * ky:8 * ky + OH, 8 * kx:8 * kx + W - 72]
out["patch_max_over_launch_max_mean"] = (pmax / xmax).mean().item()
out["patch_mean_abs_over_launch_max"] = (psum / 19200 / xmax).mean().item()
print(json.dumps(out))
