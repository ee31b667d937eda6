import numpy as np, sys
sys.path.insert(0, '.')
import paper_1509_03371_b200 as g
from paper_1509_03371_b200 import _lib
spec = g.parse_netspec_or_throw(open('tests/golden/configs.npz','rb') and bytes(np.load('tests/golden/configs.npz')['sk']).decode())
states = g.init_weights(spec, 1)
imgs = np.stack([g.Rng(7 + i).index_array_u8(200 * 180, 256).reshape(200, 180) for i in range(3)])
ref = None
for crt in (4096, 0):
    for tb in (0, 1, 2, 3, 4, 6):
        proc = g.Processor(spec, states, tile_batch=tb)
        proc.net.set_option(_lib.OPT_CRT_MIN_K, crt)
        labs, probs = proc.run_batch(imgs, 128, 101)
        sep = [proc.run(imgs[i], 128, 101)[1] for i in range(3)]
        if ref is None: ref = probs.copy()
        d_batch = int((probs.view(np.uint32) != ref.view(np.uint32)).sum())
        d_sep = [int((sep[i].view(np.uint32) != ref[i].view(np.uint32)).sum()) for i in range(3)]
        print(f"crt_min_k={crt} tile_batch={tb} last_tile={proc.last_tile()} batch-vs-ref {d_batch} separate-vs-ref {d_sep}", flush=True)
