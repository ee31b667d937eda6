"""Layer-level backward API on the B200 (include/graft_cuda.h, paper_1509_03371_b200/layers.py)
against the reference's own functions (oracle/_ref), bit for bit, with nonzero accumulators
(the reference adds into weight_diff / bias_diff / in.diff). Cases follow
proj/tests/test_layers.cpp:107-389, test_tensor.cpp:110-147 and test_pipeline.cpp:336-395."""
import ctypes as C

import numpy as np
import pytest

from conftest import assert_bitwise

import paper_1509_03371_b200 as g
from paper_1509_03371_b200 import layers as L
from oracle import oracle as O

pytestmark = pytest.mark.gpu

if not O.ref_available():
    pytest.skip("oracle/_ref not built", allow_module_level=True)

P = O.p
R = O.ref


def rnd(r, n, lo=-1.0, hi=1.0):
    return r.uniform_f32(n, lo, hi)


CONV = [(3, 4, 9, 9, 3, 1, 1, 0), (2, 5, 11, 11, 3, 2, 1, 0), (4, 2, 8, 8, 2, 1, 2, 0),
        (1, 3, 7, 7, 7, 1, 1, 0), (2, 2, 6, 6, 3, 1, 1, 1), (12, 130, 40, 40, 10, 3, 1, 0),
        (48, 64, 30, 30, 5, 2, 1, 0)]


@pytest.mark.parametrize("case", CONV)
@pytest.mark.parametrize("propagate", [True, False])
def test_conv_sk_backward(case, propagate):
    fi, fo, h, w, k, d, s, p_ = case
    r = O.Rng(100 + fi * fo + k)
    oh = O.out_extent(h, k, d, s, p_)
    ow = O.out_extent(w, k, d, s, p_)
    x = rnd(r, fi * h * w)
    W = rnd(r, fo * fi * k * k)
    dout = rnd(r, fo * oh * ow)
    dw0, db0, din0 = rnd(r, W.size), rnd(r, fo), rnd(r, x.size)  # accumulators
    dw, db, din = dw0.copy(), db0.copy(), din0.copy()
    assert R().ref_conv_backward_f32(P(x), fi, h, w, P(W), fo, k, d, s, p_, P(dout), P(dw), P(db),
                                     P(din) if propagate else None) == 0
    # the Python mirror over Blob / LayerState, like the reference's call
    xin = g.Blob.from_array(x.reshape(fi, h, w))
    if propagate:
        xin.diff = din0.copy()
    st = g.LayerState()
    st.init_conv(fo, fi * k * k)
    st.weights, st.weight_diff, st.bias_diff = W.copy(), dw0.copy(), db0.copy()
    out = g.Blob(fo, oh, ow)
    out.diff = dout.copy()
    geo = g.ConvGeometry.from_input(k, d, s, p_, h, w)
    L.conv_sk_backward(xin, st, fo, geo, g.ColumnBuffer(), g.ColumnBuffer(), out, propagate)
    assert_bitwise(st.weight_diff, dw, "weight_diff")
    assert_bitwise(st.bias_diff, db, "bias_diff")
    if propagate:
        assert_bitwise(xin.diff, din, "in.diff")


@pytest.mark.parametrize("case", [(2, 9, 9, 3, 1, 1, 0), (3, 9, 9, 2, 2, 2, 1), (1, 7, 5, 3, 2, 1, 0)])
def test_col2im(case):
    c, h, w, k, d, s, p_ = case
    oh, ow = O.out_extent(h, k, d, s, p_), O.out_extent(w, k, d, s, p_)
    col = rnd(O.Rng(3), c * k * k * oh * ow)
    want = np.empty(c * h * w, np.float32)
    assert R().ref_col2im_f32(P(col), c, h, w, k, d, s, p_, P(want)) == 0
    cb = g.ColumnBuffer()
    cb.resize(c * k * k, oh * ow)
    cb.data = col.copy()
    out = g.Blob()
    L.col2im_sk(cb, g.ConvGeometry.from_input(k, d, s, p_, h, w), c, out)
    assert_bitwise(out.data, want, "col2im_sk")
    with pytest.raises(g.SizeError, match="col2im_sk: column buffer"):
        L.col2im_sk(cb, g.ConvGeometry.from_input(k, d, s, p_, h, w), c + 1, out)


@pytest.mark.parametrize("geo", [(2, 1, 1), (2, 2, 1), (2, 4, 1), (2, 1, 2), (3, 2, 2)])
def test_maxpool_backward_with_ties(geo):
    """Forward argmax (ties -> smallest index) from the reference, then backward both ways:
    with the geometry (per-window gather) and without (the serial scatter)."""
    k, d, s = geo
    span = (k - 1) * d + 1
    h = next(v for v in range(13, 40) if (v - span) % s == 0)
    w = next(v for v in range(12, 40) if (v - span) % s == 0)
    c = 3
    r = O.Rng(21 + k + d)
    x = np.round(rnd(r, c * h * w) * 2) / 2  # few distinct values -> many ties
    x = x.astype(np.float32)
    oh, ow = O.out_extent(h, k, d, s, 0), O.out_extent(w, k, d, s, 0)
    out = np.empty(c * oh * ow, np.float32)
    am = np.empty(c * oh * ow, np.uint64)
    assert R().ref_maxpool_f32(P(x), c, h, w, k, d, s, P(out), P(am)) == 0
    dout = rnd(r, out.size)
    din0 = rnd(r, x.size)
    want = din0.copy()
    assert R().ref_maxpool_backward_f32(P(am), P(dout), out.size, c, h, w, P(want)) == 0
    for geom in (g.ConvGeometry.from_input(k, d, s, 0, h, w), None):
        xin = g.Blob.from_array(x.reshape(c, h, w))
        xin.diff = din0.copy()
        st = g.LayerState()
        st.argmax = am.copy()
        ob = g.Blob(c, oh, ow)
        ob.diff = dout.copy()
        L.maxpool_sk_backward(xin, st, ob, geom)
        assert_bitwise(xin.diff, want, f"maxpool backward geometry={geom is not None}")


def test_elementwise_backwards():
    r = O.Rng(77)
    n = 5 * 6 * 7
    x = rnd(r, n)
    x[::7] = 0.0  # relu subgradient at exactly 0 is 0 (test_layers.cpp:219-252)
    dout, din0 = rnd(r, n), rnd(r, n)
    want = din0.copy()
    R().ref_relu_backward_f32(P(x), P(dout), n, P(want))
    a = g.Blob.from_array(x.reshape(5, 6, 7))
    a.diff = din0.copy()
    o = g.Blob(5, 6, 7)
    o.diff = dout.copy()
    L.relu_backward(a, o)
    assert_bitwise(a.diff, want, "relu_backward")

    up = rnd(r, 5 * 12 * 14)
    want = din0.copy()
    R().ref_upconv_backward_f32(P(up), 5, 6, 7, P(want))
    a = g.Blob(5, 6, 7)
    a.diff = din0.copy()
    o = g.Blob(5, 12, 14)
    o.diff = up.copy()
    L.upconv_backward(a, o)
    assert_bitwise(a.diff, want, "upconv_backward")

    mc = rnd(r, (5 + 3) * 6 * 7)
    want = din0.copy()
    R().ref_mergecrop_backward_f32(P(mc), 5, 3, 6, 7, P(want))
    a = g.Blob(5, 6, 7)
    a.diff = din0.copy()
    o = g.Blob(8, 6, 7)
    o.diff = mc.copy()
    L.mergecrop_backward(a, o)
    assert_bitwise(a.diff, want, "mergecrop_backward")

    scores = rnd(r, 3 * 4 * 5, -3, 3)
    probs = np.empty_like(scores)
    R().ref_softmax_f32(P(scores), 3, 4, 5, P(probs))
    dsm, din1 = rnd(r, scores.size), rnd(r, scores.size)
    want = din1.copy()
    R().ref_softmax_backward_f32(P(probs), P(dsm), 3, 4, 5, P(want))
    a = g.Blob(3, 4, 5)
    a.diff = din1.copy()
    o = g.Blob.from_array(probs.reshape(3, 4, 5))
    o.diff = dsm.copy()
    L.softmax_backward(a, o)
    assert_bitwise(a.diff, want, "softmax_backward")


@pytest.mark.parametrize("masked", [False, True])
def test_softmax_loss_layer(masked):
    r = O.Rng(5 + masked)
    c, h, w = 3, 9, 11
    scores = rnd(r, c * h * w, -4, 4)
    labels = r.index_u8(h * w, c).astype(np.int32)
    mask = r.index_u8(h * w, 2) if masked else None
    d0 = rnd(r, scores.size)
    want = d0.copy()
    lw = C.c_double()
    assert R().ref_softmax_loss_f32(P(scores), c, h, w, P(labels), P(mask), P(want), C.byref(lw)) == 0
    b = g.Blob.from_array(scores.reshape(c, h, w))
    b.diff = d0.copy()
    loss = L.softmax_loss(b, labels.reshape(h, w), None if mask is None else mask.reshape(h, w))
    assert np.float64(loss).view(np.uint64) == np.float64(lw.value).view(np.uint64)
    assert_bitwise(b.diff, want, "softmax_loss diff")
    with pytest.raises(g.SpecError, match="outside"):
        L.softmax_loss(b, np.full((h, w), c, np.int32))


def test_sgd_step_array():
    """sgd_step (pipeline.hpp:483-500; test_pipeline.cpp:336-395) on one parameter array."""
    r = O.Rng(9)
    n = 10007
    w, mom, diff = rnd(r, n), rnd(r, n), rnd(r, n)
    ww, mm, dd = w.copy(), mom.copy(), diff.copy()
    R().ref_sgd_step_f32(P(ww), P(mm), P(dd), n, 0.01, 0.9, 5e-4)
    from paper_1509_03371_b200 import _lib
    _lib.check(_lib.lib().graft_sgd_step_f32(P(w), P(mom), P(diff), n, 0.01, 0.9, 5e-4, _lib.MEM_HOST))
    assert_bitwise(w, ww, "weights")
    assert_bitwise(mom, mm, "momentum")
    assert_bitwise(diff, dd, "diff zeroed")
