import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import paper_1509_03371_b200 as g
from conftest import config_text
for cfg in ("sk.net", "u.net", "usk.net"):
    spec = g.parse_netspec_or_throw(config_text(cfg)); states = g.init_weights(spec, 1)
    w = g.output_extent(spec, spec.w0); v = spec.w0 - w
    side = 2 * w if cfg != "sk.net" else 512
    img = g.Rng(9).index_array_u8(side * side, 256).reshape(side, side)
    lab, pr = g.Processor(spec, states).run(img, w, v)
    for kind in ("bf16", "tf32", "bf16x3"):
        lt, pt = g.Processor(spec, states, tensor_cores=kind).run(img, w, v)
        d = np.abs(pt - pr); flips = lt != lab
        m = np.abs(pr[1] - pr[0])
        print(cfg, kind, "max|dp| %.3g mean %.3g" % (d.max(), d.mean()), "flips", int(flips.sum()), "of", lab.size,
              "max margin at flip %.3g" % (m[flips].max() if flips.any() else 0), flush=True)
