"""process() under concurrent device load must stay bit-identical.

The warp-specialized DMMA kernels (conv_tma, conv_ws, gemm_tma) release a shared-memory stage
with an mbarrier arrive that a TMA / cp.async refill waits for. Without a fence the arrive could
overtake the warp's last in-flight operand loads (ptxas schedules it above the DMMAs consuming
them), and under contention the refill then landed first: conv3's last row group came out wrong
in a few hundred outputs per run, only when another stream loaded the GPU (found with
compute-sanitizer initcheck, which perturbs timing the same way). ptx::release_stage fences the
reads. This test reruns the full sk.net path with and without a memory-bound kernel loop on a
second stream and requires every run to equal the undisturbed one bit for bit."""
import threading
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1509_03371_b200 as g  # noqa: E402
from paper_1509_03371_b200 import _lib  # noqa: E402
from conftest import config_text  # noqa: E402

pytestmark = pytest.mark.gpu


class Hammer:
    """A copy/add loop over 2 GiB on its own stream (HBM- and SM-bound contention)."""

    def __enter__(self):
        self.stop = False
        self.t = threading.Thread(target=self.run)
        self.t.start()
        time.sleep(0.05)
        return self

    def run(self):
        s = torch.cuda.Stream()
        a = torch.empty(1 << 28, dtype=torch.float32, device="cuda")
        b = torch.empty_like(a)
        with torch.cuda.stream(s):
            while not self.stop:
                b.copy_(a)
                a.add_(1.0)
                s.synchronize()

    def __exit__(self, *exc):
        self.stop = True
        self.t.join()


@pytest.mark.parametrize("crt_min_k", [0, 4096])
def test_process_bit_identical_under_concurrent_load(crt_min_k):
    spec = g.parse_netspec_or_throw(config_text("sk.net"))
    states = g.init_weights(spec, 1)
    imgs = np.stack([g.Rng(7 + i).index_array_u8(200 * 180, 256).reshape(200, 180) for i in range(3)])
    proc = g.Processor(spec, states)
    proc.net.set_option(_lib.OPT_CRT_MIN_K, crt_min_k)
    lab0, pr0 = proc.run_batch(imgs, 128, 101)
    bad = []
    for it in range(8):
        with Hammer():
            lab, pr = proc.run_batch(imgs, 128, 101)
        nd = int((pr.view(np.uint32) != pr0.view(np.uint32)).sum())
        if nd or not np.array_equal(lab, lab0):
            bad.append((it, nd))
    assert not bad, f"runs under load differing from the undisturbed run (iteration, elements): {bad}"
