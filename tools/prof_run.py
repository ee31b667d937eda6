"""Short sk.net process() run for ncu captures (one image, few steps, no timing output)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1509_03371_b200 as g  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=256)
ap.add_argument("--tile", type=int, default=128)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--batch", type=int, default=0)
a = ap.parse_args()
f = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                         "golden", "configs.npz"))
spec = g.parse_netspec_or_throw(bytes(f["sk"]).decode())
proc = g.Processor(spec, g.init_weights(spec, 1), tile_batch=a.batch)
img = g.Rng(55).index_array_u8(a.size * a.size, 256).reshape(a.size, a.size)
for _ in range(a.steps):
    lab, pr = proc.run(img, a.tile, 101)
print("done", lab.sum())
