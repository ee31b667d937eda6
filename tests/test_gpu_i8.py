"""Exact integer GEMM on the tcgen05 tensor cores (graft_gemm_i8, csrc/gemm_i8.cu): every
result must equal the int64 product exactly -- integer accumulation has no rounding, which is
what an exact digit-sliced (Ozaki) conv needs."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
from paper_1509_03371_b200 import _lib  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,N,K,signed", [(128, 256, 128, True), (256, 300, 1152, False),
                                          (200, 513, 19200, True), (1024, 64, 16, False)])
def test_gemm_i8_exact(M, N, K, signed):
    rng = np.random.default_rng(M * 7 + N + K)
    if signed:
        a = rng.integers(-128, 128, size=(M, K), dtype=np.int8)
    else:
        a = rng.integers(0, 256, size=(M, K), dtype=np.uint8)
    b = rng.integers(0, 256, size=(N, K), dtype=np.uint8)
    want = a.astype(np.int64) @ b.astype(np.int64).T
    assert np.abs(want).max() < 2 ** 31
    ad = torch.from_numpy(a.view(np.uint8)).cuda()
    bd = torch.from_numpy(b).cuda()
    c = torch.empty((M, N), dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().graft_gemm_i8(ad.data_ptr(), int(signed), bd.data_ptr(), M, N, K, c.data_ptr()))
    got = c.cpu().numpy().astype(np.int64)
    assert np.array_equal(got, want)
