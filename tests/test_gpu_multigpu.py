"""The multi-GPU helpers (paper_1509_03371_b200/multigpu.py) on the real device path with an NCCL
process group. This pool exposes one GPU, so the group has one rank (NCCL refuses two ranks on
one device); the world-size-2 partition/combine logic is covered with gloo in
tests/test_multiproc_cpu.py. Here: graft_process_band through process_image, and
graft_process_batch through process_batch_sharded + the NCCL all-gather, against plain calls."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402

import paper_1509_03371_b200 as g  # noqa: E402
from paper_1509_03371_b200 import _lib  # noqa: E402
from paper_1509_03371_b200 import multigpu as M  # noqa: E402
from conftest import assert_bitwise, config_text  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def test_nccl_band_and_batch_paths(nccl_group):
    spec = g.parse_netspec_or_throw(config_text("sk.net"))
    states = g.init_weights(spec, 1)
    proc = g.Processor(spec, states)
    dev = torch.device("cuda", 0)
    H, W, w, v = 300, 260, 128, 101
    img = g.Rng(31).index_array_u8(H * W, 256).reshape(H, W)
    want_lab, want_pr = proc.run(img, w, v)

    img_d = torch.from_numpy(img).to(dev)
    lab = torch.zeros((H, W), dtype=torch.uint8, device=dev)
    pr = torch.zeros((2, H, W), dtype=torch.float32, device=dev)

    def run_band(r0, r1):
        proc.run(img_d, w, v, lab, pr, rows=(r0, r1), mem=_lib.MEM_DEVICE)

    M.process_image(run_band, H, w, 0, 1, lab, pr)
    assert np.array_equal(lab.cpu().numpy(), want_lab)
    assert_bitwise(pr.cpu().numpy(), want_pr, "band path")

    imgs = np.stack([img, g.Rng(32).index_array_u8(H * W, 256).reshape(H, W)])
    labs, prs = M.process_batch_sharded(proc, torch.from_numpy(imgs).to(dev), w, v, 0, 1, dev)
    assert labs.shape == (2, H, W) and prs.shape == (2, 2, H, W)
    assert np.array_equal(labs[0].cpu().numpy(), want_lab)
    assert_bitwise(prs[0].cpu().numpy(), want_pr, "sharded batch member 0")
    lab1, pr1 = proc.run(imgs[1], w, v)
    assert np.array_equal(labs[1].cpu().numpy(), lab1)
    assert_bitwise(prs[1].cpu().numpy(), pr1, "sharded batch member 1")
