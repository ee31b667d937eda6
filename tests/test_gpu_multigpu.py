"""The multi-GPU helpers (paper_1509_03371_b200/multigpu.py) on the real device path with an NCCL
process group. This pool exposes one GPU, so the group has one rank (NCCL refuses two ranks on
one device); the world-size-2 partition/combine logic is covered with gloo in
tests/test_multiproc_cpu.py. Here: graft_process_band through process_image, and
graft_process_batch through process_batch_sharded + the NCCL gather, against plain calls; and
the one-process multi-GPU C ABI (graft_multi_*, MultiProcessor) with ranks on this device."""
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


# ---- graft_multi_* (one process driving several GPUs, csrc/multi.cu) ----------------------
def _multi_case(cfg="sk.net"):
    spec = g.parse_netspec_or_throw(config_text(cfg))
    states = g.init_weights(spec, 1)
    return spec, states


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
def test_multi_process_bands_equal_one_gpu(devices):
    """Ranks sharing one device run the same band partition and combine (peer copies) as
    distinct GPUs would (NCCL): host and device buffers, one image and a batch, bit-identical to
    the single-GPU planes."""
    spec, states = _multi_case()
    H, W, w, v = 300, 260, 128, 101
    img = g.Rng(31).index_array_u8(H * W, 256).reshape(H, W)
    want_lab, want_pr = g.Processor(spec, states).run(img, w, v)
    mp_ = M.MultiProcessor(spec, states, devices=devices)
    assert mp_.combine_kind() == ("nccl" if len(set(devices)) == len(devices) else "peer")
    lab, pr = mp_.run(img, w, v)  # host buffers: each rank copies its own rows
    assert np.array_equal(lab, want_lab)
    assert_bitwise(pr, want_pr, f"multi host {devices}")
    dev = torch.device("cuda", 0)
    img_d = torch.from_numpy(img).to(dev)
    lab_d = torch.zeros((H, W), dtype=torch.uint8, device=dev)
    pr_d = torch.zeros((2, H, W), dtype=torch.float32, device=dev)
    torch.cuda.synchronize()
    mp_.run(img_d, w, v, lab_d, pr_d, mem=_lib.MEM_DEVICE)
    assert np.array_equal(lab_d.cpu().numpy(), want_lab)
    assert_bitwise(pr_d.cpu().numpy(), want_pr, f"multi device {devices}")
    imgs = np.stack([img] + [g.Rng(40 + i).index_array_u8(H * W, 256).reshape(H, W) for i in range(3)])
    labs, prs = mp_.run_batch(imgs, w, v)
    one = g.Processor(spec, states)
    for i in range(len(imgs)):
        l1, p1 = one.run(imgs[i], w, v)
        assert np.array_equal(labs[i], l1)
        assert_bitwise(prs[i], p1, f"multi batch member {i}")
    imgs_d = torch.from_numpy(imgs).to(dev)
    labs_d = torch.zeros((4, H, W), dtype=torch.uint8, device=dev)
    prs_d = torch.zeros((4, 2, H, W), dtype=torch.float32, device=dev)
    torch.cuda.synchronize()
    mp_.run_batch(imgs_d, w, v, labs_d, prs_d, mem=_lib.MEM_DEVICE)
    assert np.array_equal(labs_d.cpu().numpy(), labs)
    assert_bitwise(prs_d.cpu().numpy(), prs, f"multi device batch {devices}")


def test_multi_strided_net_and_errors():
    """A strided net (reduced usk.net golden geometry) through two ranks on one device, and the
    single-GPU validation messages unchanged."""
    from test_gpu_parity_timed import STRIDED, strided_spec
    from conftest import load_golden

    key, cfg, fout, sigma, w, v, H, W = STRIDED[1]
    gold = load_golden("strided.npz")
    spec = strided_spec(cfg, fout, sigma)
    states = g.init_weights(spec, 5)
    mp_ = M.MultiProcessor(spec, states, devices=[0, 0])
    lab, pr = mp_.run(gold[f"{key}_img"], w, v)
    assert np.array_equal(lab, gold[f"{key}_labels"])
    assert_bitwise(pr, gold[f"{key}_probs"], "multi strided")
    with pytest.raises(g.SizeError, match="smaller than one"):
        mp_.run(np.zeros((10, 10), np.uint8), w, v)
    with pytest.raises(g.SpecError, match="tile"):
        mp_.run(gold[f"{key}_img"], w + 1, v)


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs >= 2 GPUs (this pool exposes one per call)")
def test_multi_process_nccl_two_gpus():
    spec, states = _multi_case()
    H, W, w, v = 1024, 768, 128, 101
    img = g.Rng(5).index_array_u8(H * W, 256).reshape(H, W)
    want_lab, want_pr = g.Processor(spec, states).run(img, w, v)
    n = torch.cuda.device_count()
    mp_ = M.MultiProcessor(spec, states, n_gpus=n)
    assert mp_.combine_kind() == "nccl"
    dev = torch.device("cuda", 0)
    lab_d = torch.zeros((H, W), dtype=torch.uint8, device=dev)
    pr_d = torch.zeros((2, H, W), dtype=torch.float32, device=dev)
    torch.cuda.synchronize()
    mp_.run(torch.from_numpy(img).to(dev), w, v, lab_d, pr_d, mem=_lib.MEM_DEVICE)
    assert np.array_equal(lab_d.cpu().numpy(), want_lab)
    assert_bitwise(pr_d.cpu().numpy(), want_pr, f"nccl x{n}")
