"""GPU parity of the layer-level API (layers.hpp / tensor.hpp) through the C ABI: every
result compared bit for bit with the reference's golden vectors and with the CPU oracle on the
same seeded inputs. Mirrors proj/tests/test_layers.cpp and test_tensor.cpp."""
import numpy as np
import pytest

import paper_1509_03371_b200 as g
from conftest import assert_bitwise
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def blob(a):
    return g.Blob.from_array(a)


def run_conv(x, w, b, fo, k, d, s, p_):
    st = g.LayerState(x.dtype)
    st.weights, st.bias = w.copy(), b.copy()
    out = g.Blob(dtype=x.dtype)
    g.conv_sk_forward(blob(x), st, fo, g.ConvGeometry.from_input(k, d, s, p_, x.shape[1],
                                                                 x.shape[2]),
                      g.ColumnBuffer(x.dtype), out)
    return out.view()


def test_conv_identity_kernels():
    x = O.Rng(3).uniform_f32(25).reshape(1, 5, 5)
    assert_bitwise(run_conv(x, np.ones(1, np.float32), np.zeros(1, np.float32), 1, 1, 1, 1, 0), x)
    w = np.zeros(9, np.float32)
    w[4] = 1.0
    assert_bitwise(run_conv(x, w, np.zeros(1, np.float32), 1, 3, 1, 1, 1), x)


def test_conv_equals_reference_bit_for_bit(glayers):
    # proj/tests/test_layers.cpp:80-105 (f32) and the same geometries in f64
    for i, (fi, fo, h, w, k, d, s, p_) in enumerate(glayers["conv_cases"]):
        out = run_conv(glayers[f"conv{i}_in"], glayers[f"conv{i}_w"], glayers[f"conv{i}_b"], fo,
                       k, d, s, p_)
        assert_bitwise(out, glayers[f"conv{i}_out"], f"conv case {i}")
        out = run_conv(glayers[f"conv64_{i}_in"], glayers[f"conv64_{i}_w"],
                       glayers[f"conv64_{i}_b"], fo, k, d, s, p_)
        assert_bitwise(out, glayers[f"conv64_{i}_out"], f"conv f64 case {i}")


def test_conv_sk_shapes(glayers):
    # dilations 2/4/8, the 10x10 spanning kernel, K=520 tails, M=33 / M=2 row tails
    for i, (fi, fo, h, w, k, d) in enumerate(glayers["sk_cases"]):
        out = run_conv(glayers[f"sk{i}_in"], glayers[f"sk{i}_w"], glayers[f"sk{i}_b"], fo, k, d, 1,
                       0)
        assert_bitwise(out, glayers[f"sk{i}_out"], f"sk case {i}")


def test_conv_random_geometries_vs_oracle():
    r = O.Rng(321)
    for t in range(40):
        fi = 1 + int(r.uniform(0, 9))
        fo = 1 + int(r.uniform(0, 140))
        k = 1 + int(r.uniform(0, 5))
        d = 1 + int(r.uniform(0, 4))
        s = 1 + int(r.uniform(0, 3))
        p_ = int(r.uniform(0, 3))
        span = (k - 1) * d + 1
        h = span + s * int(r.uniform(0, 20)) - 2 * p_
        wdt = span + s * int(r.uniform(0, 20)) - 2 * p_
        if h < 1 or wdt < 1:
            continue
        x = r.uniform_f32(fi * h * wdt).reshape(fi, h, wdt)
        w = r.gaussian_f32(fo * fi * k * k, 0.0, 0.3)
        b = r.uniform_f32(fo)
        assert_bitwise(run_conv(x, w, b, fo, k, d, s, p_), O.conv(x, w, b, fo, k, d, s, p_),
                       f"trial {t}")


def test_conv_rejects_mismatched_weights():
    # proj/tests/test_layers.cpp:379-389
    st = g.LayerState()
    st.init_conv(3, 2 * 9)
    with pytest.raises(g.SizeError, match="weight count"):
        g.conv_sk_forward(g.Blob(2, 5, 5), st, 3, g.ConvGeometry.from_input(5, 1, 1, 0, 5, 5),
                          g.ColumnBuffer(), g.Blob())


def test_maxpool_and_ties(glayers):
    for i in range(4):
        k, d, s, hw = (int(v) for v in glayers[f"pool{i}_cfg"])
        st, out = g.LayerState(), g.Blob()
        g.maxpool_sk_forward(blob(glayers[f"pool{i}_in"]), st,
                             g.ConvGeometry.from_input(k, d, s, 0, hw, hw), out)
        assert_bitwise(out.view(), glayers[f"pool{i}_out"], f"pool {i}")
        assert np.array_equal(st.argmax, glayers[f"pool{i}_argmax"])
    st, out = g.LayerState(), g.Blob()
    flat = g.Blob.from_array(np.full((1, 4, 4), 2.5, np.float32))
    g.maxpool_sk_forward(flat, st, g.ConvGeometry.from_input(2, 1, 2, 0, 4, 4), out)
    assert st.argmax.tolist() == [flat.index(0, 0, 0), flat.index(0, 0, 2), flat.index(0, 2, 0),
                                  flat.index(0, 2, 2)]


def test_elementwise_layers(glayers):
    out = g.Blob()
    g.relu_forward(blob(glayers["relu_in"]), out)
    assert_bitwise(out.view(), glayers["relu_out"], "relu")
    g.upconv_forward(blob(glayers["up_in"]), out)
    assert_bitwise(out.view(), glayers["up_out"], "upconv")
    g.mergecrop_forward(blob(glayers["mc_a"]), blob(glayers["mc_b"]), out)
    assert_bitwise(out.view(), glayers["mc_out"], "mergecrop")
    with pytest.raises(g.SizeError):
        g.mergecrop_forward(blob(glayers["mc_a"]), g.Blob(1, 1, 1), out)


def test_softmax(glayers):
    # tolerance stated: <= 1 ulp f32 (glibc exp vs the device's correctly rounded exp);
    # 0 ulp expected and asserted on these fixtures.
    for name in ("sm3", "sm2", "sm_ext"):
        out = g.Blob()
        g.softmax_forward(blob(glayers[name + "_in"]), out)
        assert_bitwise(out.view(), glayers[name + "_out"], name)
    r = O.Rng(41)
    x = (r.uniform_f32(2 * 256 * 256, -1, 1) * np.float32(2e-3)).reshape(2, 256, 256)
    out = g.Blob()
    g.softmax_forward(blob(x), out)
    want = O.softmax(x)
    ulps = np.abs(out.view().view(np.int32).astype(np.int64) - want.view(np.int32).astype(np.int64))
    assert ulps.max() <= 1
    assert (ulps != 0).sum() == 0


def test_im2col(glayers):
    for i, (c, h, w, k, d, s, p_) in enumerate(glayers["im2col_cases"]):
        col = g.ColumnBuffer()
        g.im2col_sk(blob(glayers[f"im2col{i}_in"]), g.ConvGeometry.from_input(k, d, s, p_, h, w),
                    col)
        assert_bitwise(col.data[:col.rows * col.cols].reshape(col.rows, col.cols),
                       glayers[f"im2col{i}_out"], f"im2col {i}")


def test_gemm_frozen_and_variants(glayers):
    c = np.full(4, -1, np.float32)
    g.gemm(False, False, 2, 2, 2, 1.0, np.array([1, 2, 3, 4], np.float32),
           np.array([5, 6, 7, 8], np.float32), 0.0, c)
    assert c.tolist() == [19.0, 22.0, 43.0, 50.0]
    m, n, k = 4, 5, 3
    A, B, Cin = glayers["gemm_A"], glayers["gemm_B"], glayers["gemm_C"]
    for ta in (0, 1):
        for tb in (0, 1):
            a = A.reshape(m, k).T.copy().ravel() if ta else A
            b = B.reshape(k, n).T.copy().ravel() if tb else B
            for alpha, beta in ((1.0, 0.0), (2.0, 1.0), (-0.5, 0.25)):
                c = Cin.copy()
                g.gemm(ta, tb, m, n, k, alpha, a, b, beta, c)
                assert_bitwise(c, glayers[f"gemm_{ta}{tb}_{alpha}_{beta}"], "gemm")
    c = glayers["gemm64_C"].copy()
    g.gemm(False, False, m, n, k, 2.0, glayers["gemm64_A"], glayers["gemm64_B"], 1.0, c)
    assert_bitwise(c, glayers["gemm64_out"], "gemm f64")
    c = np.zeros(6 * 32, np.float32)
    g.gemm(False, False, 6, 32, 50, 1.0, glayers["gemmcc_A"], glayers["gemmcc_B"], 0.0, c)
    assert_bitwise(c, glayers["gemmcc_out"], "gemm chunk")


def test_pad_normalize(glayers):
    img = g.Plane.from_array(glayers["pad_img"])
    for v in (0, 1, 5, 10):
        assert np.array_equal(g.mirror_pad(img, v).view(), glayers[f"pad_v{v}"])
    lut = g.normalize_image(g.Plane.from_array(np.arange(256, dtype=np.uint8).reshape(16, 16)))
    assert_bitwise(lut.pix, glayers["normalize_lut"])
    with pytest.raises(g.SizeError, match="needs an image larger"):
        g.mirror_pad(g.Plane(5, 5), 10)
