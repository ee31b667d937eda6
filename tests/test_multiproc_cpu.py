"""World-size-2 gloo tests of the multi-GPU partitioner and final combine on CPU
(paper_1509_03371_b200/multigpu.py). The per-band compute is the CPU oracle restricted to the
band's rows -- exactly what graft_process_band writes (there is no GPU here) -- so the test pins
the partition and the gather-to-rank-0 combine; the GPU band kernels themselves are covered by
tests/test_gpu_net.py and tests/test_gpu_multigpu.py (graft_multi_process on the device)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1509_03371_b200 import multigpu as M


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_split_rows_and_bands_cover_exactly():
    for H, w in ((512, 128), (300, 128), (14, 6), (16, 16), (1000, 7)):
        n = (H + w - 1) // w
        for world in (1, 2, 3, 4, 8):
            splits = M.split_rows(n, world)
            assert splits[0][0] == 0 and splits[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(splits, splits[1:]))
            bands = [M.band_rows_py(H, w, r0, r1) for r0, r1 in splits]
            covered = np.zeros(H, int)
            for y0, y1 in bands:
                covered[y0:y1] += 1
            assert (covered == 1).all(), (H, w, world, bands)


def test_shard_range_covers_exactly():
    for n in (0, 1, 5, 64, 67):
        for world in (1, 2, 3, 8):
            spans = [M.shard_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(e - b for b, e in spans) - min(e - b for b, e in spans) <= 1


def _worker(rank, world, port, H, W, w, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_1509_03371_b200.netspec import parse_netspec_or_throw

    spec = parse_netspec_or_throw(
        "input w=21 f=1\n"
        "layer c1 conv_sk k=3 fout=4 in=data out=c1 init=he\n"
        "layer r1 relu in=c1 out=r1\n"
        "layer p1 pool_max k=2 s=1 in=r1 out=p1\n"
        "layer c2 conv_sk k=2 d=2 fout=3 in=p1 out=c2 init=he\n"
        "layer prob softmax_loss in=c2 out=prob\n")
    params = O.init_weights(spec, 17)
    img = O.Rng(55).index_u8(H * W).reshape(H, W)
    full_lab, full_prob = O.process(spec, params, img, w, 5)
    labels = torch.zeros((H, W), dtype=torch.uint8)
    probs = torch.zeros((3, H, W), dtype=torch.float32)

    def run_band(r0, r1):  # what graft_process_band writes: only the band's rows
        y0, y1 = M.band_rows_py(H, w, r0, r1)
        labels[y0:y1] = torch.from_numpy(full_lab[y0:y1])
        probs[:, y0:y1] = torch.from_numpy(full_prob[:, y0:y1])

    M.process_image(run_band, H, w, rank, world, labels, probs)
    if rank == 0:  # the combine gathers to rank 0
        ok = np.array_equal(labels.numpy(), full_lab) and \
            np.array_equal(probs.numpy().view(np.uint32), full_prob.view(np.uint32))
    else:  # other ranks keep exactly their own band
        y0, y1 = M.band_rows_py(H, w, *M.split_rows((H + w - 1) // w, world)[rank])
        ok = np.array_equal(labels.numpy()[y0:y1], full_lab[y0:y1])
    # batch mode: images round-robin, all-gathered
    per = {}
    for i in M.batch_assignment(3, world, rank):
        per[i] = (torch.full((4, 5), i, dtype=torch.uint8), torch.full((2, 4, 5), float(i)))
    labs, prs = M.gather_batch(per, 3, (4, 5), (2, 4, 5), rank, world, "cpu")
    ok = ok and all(int(labs[i][0, 0]) == i and float(prs[i][1, 3, 4]) == i for i in range(3))
    # sharded batch mode (graft_process_batch per rank + one all-gather): 5 images over 2 ranks
    b, e = M.shard_range(5, world, rank)
    lab_sh = torch.stack([torch.full((4, 5), i, dtype=torch.uint8) for i in range(b, e)])
    prob_sh = torch.stack([torch.full((2, 4, 5), float(i) + 0.5) for i in range(b, e)])
    la, pa = M.gather_shards(lab_sh, prob_sh, 5, rank, world)
    if rank == 0:
        ok = ok and la.shape == (5, 4, 5) and all(int(la[i, 3, 4]) == i for i in range(5)) and \
            all(float(pa[i, 1, 0, 0]) == i + 0.5 for i in range(5))
    else:
        ok = ok and la is None and pa is None
    q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("H,W,w", [(23, 19, 6), (40, 33, 16)])
def test_gloo_world2_partition_and_combine(H, W, w):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, H, W, w, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
