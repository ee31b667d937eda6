import numpy as np, sys, ctypes
sys.path.insert(0, '.')
import paper_1509_03371_b200 as g
from paper_1509_03371_b200 import _lib
spec = g.parse_netspec_or_throw(bytes(np.load('tests/golden/configs.npz')['sk']).decode())
states = g.init_weights(spec, 1)
imgs = np.stack([g.Rng(7 + i).index_array_u8(200 * 180, 256).reshape(200, 180) for i in range(3)])
refp = g.Processor(spec, states, retile=0)
refp.net.set_option(_lib.OPT_CRT_MIN_K, 0)
ref = np.stack([refp.run(imgs[i], 128, 101)[1] for i in range(3)])
def fb(p):
    return p.net.get_option(_lib.OPT_CRT_FALLBACKS)
for trial in range(2):
    proc = g.Processor(spec, states)
    labs, probs = proc.run_batch(imgs, 128, 101)
    print('batch: tile', proc.last_tile(), 'fallbacks', fb(proc), 'diff vs DMMA ref', int((probs.view(np.uint32) != ref.view(np.uint32)).sum()), flush=True)
    for i in range(3):
        lab, pr = proc.run(imgs[i], 128, 101)
        print('  single', i, 'tile', proc.last_tile(), 'fallbacks', fb(proc), 'diff vs ref', int((pr.view(np.uint32) != ref[i].view(np.uint32)).sum()), flush=True)
