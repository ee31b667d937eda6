import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
import paper_1509_03371_b200 as g
from paper_1509_03371_b200 import _lib
spec = g.parse_netspec_or_throw(bench.sk_text()); states = g.init_weights(spec, 1)
dev = torch.device("cuda", 0)
proc = g.Processor(spec, states, tensor_cores="bf16")
img = torch.from_numpy(g.Rng(55).index_array_u8(1024*1024, 256).reshape(1024, 1024)).to(dev)
lab = torch.empty((1024, 1024), dtype=torch.uint8, device=dev); prob = torch.empty((2, 1024, 1024), dtype=torch.float32, device=dev)
stream = torch.cuda.ExternalStream(_lib.lib().graft_net_stream(proc.net.h), device=dev)
for _ in range(3): proc.run(img, 128, 101, lab, prob, mem=_lib.MEM_DEVICE)
torch.cuda.synchronize()
for timed in (0, 1):
    proc.net.set_option(_lib.OPT_TIMED, timed)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t = time.perf_counter(); e0.record(stream)
    for _ in range(5): proc.run(img, 128, 101, lab, prob, mem=_lib.MEM_DEVICE)
    e1.record(stream); e1.synchronize(); w = time.perf_counter() - t
    print("timed", timed, "device ms/step", e0.elapsed_time(e1) / 5, "wall ms/step", w * 200)
