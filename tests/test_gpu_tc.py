"""Tolerance mode: the tcgen05 implicit-GEMM conv (csrc/conv_tc.cu) against
an fp64 torch conv of the same rounded operands.

The tensor-core path is NOT the reference's arithmetic (inc/tensor.hpp:151-169: an fp64 chain
rounded once to f32): operands are rounded to bf16 / tf32 and products are summed in f32 by the
tensor core. Stated tolerance: against the exact sum of the rounded
operands, |got - ref| <= 4e-5 * sum_k |w_k x_k| + 1 ulp(f32) per output."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1509_03371_b200 as g  # noqa: E402
from paper_1509_03371_b200 import _lib  # noqa: E402

pytestmark = pytest.mark.gpu

TOL = 4e-5


def round_tf32(t):
    """cvt.rna.tf32.f32: round to 10 mantissa bits, ties away from zero."""
    b = t.contiguous().view(torch.int32)
    b = (b + 0x1000) & ~0x1FFF
    return b.view(torch.float32)


def run_tc(kind, x, w, bias, k, d, relu):
    B, C, H, W = x.shape
    M = w.shape[0]
    OH, OW = H - (k - 1) * d, W - (k - 1) * d
    out = torch.empty(B, M, OH, OW, device="cuda", dtype=torch.float32)
    torch.cuda.synchronize()
    _lib.check(_lib.lib().graft_conv_tc_f32(kind, x.data_ptr(), B, C, H, W, w.data_ptr(),
                                            bias.data_ptr(), M, k, d, out.data_ptr(), int(relu)))
    return out


CASES = [  # B, C, H, W, M, k, d
    (1, 64, 20, 20, 128, 3, 1),
    (2, 64, 30, 300, 128, 3, 2),    # ragged row segments (OW = 296 > 256)
    (1, 128, 36, 40, 256, 3, 4),    # conv3-like dilation
    (1, 192, 90, 90, 128, 10, 8),   # ip1 geometry (k10 d8), 18x18 out
    (1, 1024, 8, 130, 512, 1, 1),   # ip2 geometry (1x1, K = 1024)
    (1, 48, 30, 40, 128, 5, 2),     # conv2: channels padded 48 -> 64 (bf16) / 64 (tf32)
    (1, 128, 40, 40, 192, 3, 4),    # conv3: f_out padded 192 -> 256
    (2, 3, 30, 30, 48, 7, 1),       # conv1: 3 channels, 48 outputs
]


@pytest.mark.parametrize("kind", [_lib.TC_BF16, _lib.TC_TF32, _lib.TC_BF16X3])
@pytest.mark.parametrize("case", CASES)
def test_conv_tc_matches_fp64_conv_of_rounded_operands(kind, case):
    B, C, H, W, M, k, d = case
    gen = torch.Generator(device="cuda").manual_seed(1234 + C + k)
    x = torch.rand(B, C, H, W, device="cuda", generator=gen) * 2 - 1
    w = (torch.randn(M, C, k, k, device="cuda", generator=gen) * (2.0 / (C * k * k)) ** 0.5)
    bias = torch.randn(M, device="cuda", generator=gen) * 0.01
    for relu in (False, True):
        got = run_tc(kind, x, w, bias, k, d, relu)
        tol = TOL
        if kind == _lib.TC_BF16:
            xr, wr = x.bfloat16().double(), w.bfloat16().double()
        elif kind == _lib.TC_TF32:
            xr, wr = round_tf32(x).double(), round_tf32(w).double()
        else:  # split bf16: against the unrounded operands, operand error ~3 * 2^-17
            xr, wr = x.double(), w.double()
            tol = 6e-5
        ref = torch.nn.functional.conv2d(xr, wr, bias.double(), dilation=d)
        if relu:
            ref = ref.clamp_min(0)
        absum = torch.nn.functional.conv2d(xr.abs(), wr.abs(), None, dilation=d)
        err = (got.double() - ref).abs()
        bound = tol * absum + ref.abs() * 2.0 ** -23 + 1e-30
        worst = (err / bound).max().item()
        assert worst <= 1.0, f"kind {kind} case {case} relu {relu}: err/bound {worst:.3g}"


def test_conv_tc_rejects_empty_geometry():
    x = torch.zeros(1, 48, 4, 4, device="cuda")
    w = torch.zeros(128, 48, 5, 5, device="cuda")
    b = torch.zeros(128, device="cuda")
    with pytest.raises(g.SizeError):
        _lib.check(_lib.lib().graft_conv_tc_f32(_lib.TC_BF16, x.data_ptr(), 1, 48, 4, 4, w.data_ptr(),
                                                b.data_ptr(), 128, 5, 1, x.data_ptr(), 0))


def test_process_tolerance_mode_full_sk_net():
    """process() of full sk.net with ip1/ip2 on the tensor cores (bf16) vs the exact mode on the
    same 256x256 image: the exact planes are the reference's (tests/test_gpu_net.py); the
    tolerance-mode planes must stay within the stated tolerance and the labels may only differ
    where the exact probabilities are within that tolerance of a tie."""
    from conftest import config_text

    spec = g.parse_netspec_or_throw(config_text("sk"))
    states = g.init_weights(spec, 1)
    img = g.Rng(55).index_array_u8(256 * 256, 256).reshape(256, 256)
    lab_x, prob_x = g.Processor(spec, states).run(img, 128, 101)
    for kind in ("bf16", "tf32", "bf16x3"):
        proc = g.Processor(spec, states, tensor_cores=kind)
        lab_t, prob_t = proc.run(img, 128, 101)
        dp = np.abs(prob_t - prob_x)
        assert dp.max() <= 1e-4, f"{kind}: max |dprob| {dp.max():.3g}"
        margin = np.abs(prob_x[1] - prob_x[0])
        bad = lab_t != lab_x
        assert np.all(margin[bad] <= 2e-4), f"{kind}: a label flipped away from a near-tie"
        assert bad.mean() <= 1e-3


def test_tolerance_mode_option_validation():
    from conftest import config_text

    spec = g.parse_netspec_or_throw(config_text("sk"))
    with pytest.raises(ValueError):
        g.Processor(spec, g.init_weights(spec, 1), tensor_cores="fp8")


def test_tolerance_mode_batch_and_repeat_are_deterministic():
    """The tensor-core path is deterministic: a batch of images equals the per-image calls, and a
    repeated call gives the same planes bit for bit (no atomics, fixed MMA order per tile)."""
    from conftest import config_text

    spec = g.parse_netspec_or_throw(config_text("sk"))
    states = g.init_weights(spec, 1)
    proc = g.Processor(spec, states, tensor_cores="bf16")
    imgs = np.stack([g.Rng(70 + i).index_array_u8(200 * 240, 256).reshape(200, 240) for i in range(3)])
    labs, probs = proc.run_batch(imgs, 128, 101)
    for i in range(3):
        lab, pr = proc.run(imgs[i], 128, 101)
        assert np.array_equal(lab, labs[i])
        assert np.array_equal(pr.view(np.uint32), probs[i].view(np.uint32))
    lab2, pr2 = proc.run(imgs[0], 128, 101)
    assert np.array_equal(pr2.view(np.uint32), probs[0].view(np.uint32))
