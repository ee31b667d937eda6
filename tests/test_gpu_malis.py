"""Batched MALIS on the B200 (malis.hpp) against the reference.

* reference-made fixtures (tests/golden/malis.npz, make_golden.py malis): affinity graphs,
  components, malis_gradient (gradients, per-edge pair counts, totals, losses),
  affinity_backward and the composed malis_softmax_loss, float and double, bit for bit;
* random batches against the reference itself (oracle/_ref), every patch of the batch;
* the reference's own test cases (proj/tests/test_malis.cpp): closed forms, the
  zero-gradient fixpoint, degenerate instances, relabeling invariance, input validation;
* the training runner's device MALIS loss (pipeline.hpp:599-606) against the reference's
  malis_softmax_loss on the same score blob.
"""
import numpy as np
import pytest

import paper_1509_03371_b200 as g
from paper_1509_03371_b200 import malis as M
from conftest import assert_bitwise, load_golden
from oracle import oracle as O

pytestmark = pytest.mark.gpu

FIELDS = ("da_x", "da_y", "pos_x", "pos_y", "neg_x", "neg_y")


def graph(ax, ay, mx=None, my=None):
    mx = np.zeros(np.shape(ax), np.uint8) if mx is None else mx
    my = np.zeros(np.shape(ax), np.uint8) if my is None else my
    return M.AffinityGraph(np.asarray(ax), np.asarray(ay), mx, my)


def test_malis_reference_goldens():
    gold = load_golden("malis.npz")
    for ci, (h, w) in enumerate(gold["cases"]):
        key = f"c{ci}"
        fg = gold[f"{key}_fg"]
        assert np.array_equal(M.connected_components(fg), gold[f"{key}_comp"]), key
        for t in ("f32", "f64"):
            k = f"{key}_{t}"
            pg = M.affinity_forward(gold[f"{k}_probs"])
            for n, a in (("pax", pg.a_x), ("pay", pg.a_y), ("pmx", pg.m_x), ("pmy", pg.m_y)):
                assert_bitwise(a, gold[f"{k}_{n}"], f"{k} {n}")
            r = M.malis_gradient(pg, graph(gold[f"{k}_tax"], gold[f"{k}_tay"]), gold[f"{key}_comp"])
            for n in FIELDS:
                assert_bitwise(getattr(r, n), gold[f"{k}_{n}"], f"{k} {n}")
            assert [r.total_pos, r.total_neg] == list(gold[f"{k}_totals"]), k
            assert_bitwise(np.array([r.loss_pos, r.loss_neg, r.loss]), gold[f"{k}_losses"], f"{k} losses")
            dp, dn = M.affinity_backward(gold[f"{k}_dgx"], gold[f"{k}_dgy"], pg)
            assert_bitwise(dp, gold[f"{k}_dpos"], f"{k} dpos")
            assert_bitwise(dn, gold[f"{k}_dneg"], f"{k} dneg")
            losses, d = M.malis_softmax_loss_batch(gold[f"{k}_scores"][None], fg[None], gold[f"{k}_diff0"][None])
            assert_bitwise(losses, gold[f"{k}_loss"], f"{k} loss")
            assert_bitwise(d[0], gold[f"{k}_diff"], f"{k} diff")


def random_batch(rng, B, h, w, density, dt):
    fg = (rng.random((B, h, w)) < density).astype(np.uint8)
    probs = rng.uniform(0.01, 0.99, (B, h, w)).astype(dt)
    if rng.random() < 0.5:  # ties: quantised probabilities exercise the (value, index) order
        probs = (np.round(probs * 8) / 8).clip(0.01, 0.99).astype(dt)
    return fg, probs


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("shape,B,density", [((64, 64), 12, 0.5), ((17, 33), 9, 0.3), ((40, 24), 8, 0.9),
                                             ((1, 50), 4, 0.5), ((30, 1), 4, 0.5), ((8, 8), 6, 0.0),
                                             ((8, 8), 6, 1.0)])
def test_malis_batches_match_reference(dt, shape, B, density):
    h, w = shape
    rng = np.random.default_rng(h * 1000 + w + B)
    fg, probs = random_batch(rng, B, h, w, density, dt)
    pred = M.affinity_forward_batch(probs)
    truth = M.affinity_forward_batch(fg.astype(dt))
    comp = M.connected_components_batch(fg)
    r = M.malis_gradient_batch(pred, truth, comp)
    scores = rng.uniform(-2.0, 2.0, (B, 2, h, w)).astype(dt)
    diff0 = rng.uniform(-1.0, 1.0, (B, 2, h, w)).astype(dt)
    losses, diff = M.malis_softmax_loss_batch(scores, fg, diff0)
    for b in range(B):
        rp = O.malis_affinity_forward(probs[b], "ref")
        for got, want in zip((pred.a_x[b], pred.a_y[b], pred.m_x[b], pred.m_y[b]), rp):
            assert_bitwise(got, want, f"pred graph {b}")
        assert np.array_equal(comp[b], O.malis_components(fg[b], "ref"))
        rt = O.malis_affinity_forward(fg[b].astype(dt), "ref")
        want = O.malis_gradient(rp[0], rp[1], rt[0], rt[1], comp[b], "ref")
        for n in FIELDS:
            assert_bitwise(getattr(r, n)[b], want[n], f"patch {b} {n}")
        assert [r.total_pos[b], r.total_neg[b]] == list(want["totals"])
        assert_bitwise(np.array([r.loss_pos[b], r.loss_neg[b], r.loss[b]]), want["losses"], f"patch {b} losses")
        lw, dw = O.malis_softmax_loss(scores[b], fg[b], diff0[b], "ref")
        assert_bitwise(np.array([losses[b]]), np.array([lw]), f"patch {b} composed loss")
        assert_bitwise(diff[b], dw, f"patch {b} composed diff")


def test_single_pair_closed_form():
    """test_malis.cpp: 'maximin gradient: single-pair closed form'."""
    probs = np.array([[0.4, 0.7]])
    fg = np.ones((1, 2), np.uint8)
    r = M.malis_gradient(M.affinity_forward(probs), M.affinity_forward(fg.astype(np.float64)),
                         M.connected_components(fg))
    assert r.total_pos == 1 and r.total_neg == 0 and r.pos_x[0, 0] == 1
    assert r.loss_pos == pytest.approx(0.36, rel=1e-12) and r.loss_neg == 0.0
    assert r.da_x[0, 0] == pytest.approx(-1.2, rel=1e-12)


def test_cross_pair_lands_on_bottleneck():
    """test_malis.cpp: 'maximin gradient: cross pair lands on the bottleneck edge only'."""
    probs = np.array([[0.3, 0.8, 0.5]])
    fg = np.array([[1, 0, 1]], np.uint8)
    r = M.malis_gradient(M.affinity_forward(probs), M.affinity_forward(fg.astype(np.float64)),
                         M.connected_components(fg))
    assert r.total_pos == 0 and r.loss_pos == 0.0 and r.total_neg == 3
    assert r.neg_x[0, 1] == 1 and r.neg_x[0, 0] == 2
    assert r.da_x[0, 1] == pytest.approx(2.0 * 0.5 * 1.0 / 3.0, rel=1e-12)
    assert r.da_x[0, 0] == pytest.approx(2.0 * 0.3 * 2.0 / 3.0, rel=1e-12)


def test_perfect_predictions_and_degenerate_instances():
    """test_malis.cpp: zero-gradient fixpoint, all background, one component, 1x1."""
    rng = np.random.default_rng(77)
    for _ in range(10):
        fg = (rng.random((5, 5)) < 0.5).astype(np.uint8)
        exact = fg.astype(np.float64)
        r = M.malis_gradient(M.affinity_forward(exact), M.affinity_forward(exact), M.connected_components(fg))
        assert r.loss == 0.0 and not r.da_x.any() and not r.da_y.any()
    pred = M.affinity_forward(rng.uniform(0.01, 0.99, (3, 3)))
    none = np.zeros((3, 3), np.uint8)
    r = M.malis_gradient(pred, M.affinity_forward(none.astype(np.float64)), M.connected_components(none))
    assert r.total_pos == 0 and r.loss_pos == 0.0 and r.total_neg == 0
    full = np.ones((3, 3), np.uint8)
    r = M.malis_gradient(pred, M.affinity_forward(full.astype(np.float64)), M.connected_components(full))
    assert r.total_neg == 0 and r.total_pos == 36
    one = np.ones((1, 1), np.uint8)
    r = M.malis_gradient(M.affinity_forward(np.full((1, 1), 0.5)), M.affinity_forward(one.astype(np.float64)),
                         M.connected_components(one))
    assert r.loss == 0.0


def test_relabeling_invariance():
    """test_malis.cpp: 'maximin gradient is invariant under component relabeling'."""
    for seed in range(404, 500):
        rng = np.random.default_rng(seed)
        fg = (rng.random((5, 5)) < 0.5).astype(np.uint8)
        comp = M.connected_components(fg)
        if comp.max() >= 2:  # otherwise the permutation below is trivial
            break
    pred = M.affinity_forward(rng.uniform(0.01, 0.99, (5, 5)))
    truth = M.affinity_forward(fg.astype(np.float64))
    assert comp.max() >= 2
    perm = np.where(comp > 0, comp.max() + 1 - comp, 0).astype(np.int32)
    a, b = M.malis_gradient(pred, truth, comp), M.malis_gradient(pred, truth, perm)
    assert a.total_pos == b.total_pos and a.total_neg == b.total_neg and a.loss == b.loss
    assert_bitwise(a.da_x, b.da_x, "da_x")
    assert_bitwise(a.da_y, b.da_y, "da_y")


def test_components_reference_cases():
    """test_malis.cpp: 'connected components: 4-connectivity, raster numbering'."""
    assert not M.connected_components(np.zeros((3, 3), np.uint8)).any()
    blobs = np.zeros((3, 5), np.uint8)
    blobs[:, 0:2] = 1
    blobs[:, 3:5] = 1
    c = M.connected_components(blobs)
    assert c[0, 0] == 1 and c[2, 1] == 1 and c[0, 3] == 2 and c[2, 4] == 2 and c[1, 2] == 0
    diag = np.array([[1, 0], [0, 1]], np.uint8)
    c = M.connected_components(diag)
    assert c[0, 0] == 1 and c[1, 1] == 2
    assert (M.connected_components(np.ones((2, 2), np.uint8)) == 1).all()


def test_composed_loss_validation():
    """test_malis.cpp: 'composed loss input validation' (SizeError, the reference's messages)."""
    fg = np.ones((2, 2), np.uint8)
    three = g.Blob(3, 2, 2, np.float64)
    with pytest.raises(g.SizeError, match="needs exactly 2 score channels, got 3"):
        M.malis_softmax_loss(three, fg)
    wrong = g.Blob(2, 3, 3, np.float64)
    with pytest.raises(g.SizeError, match="label plane does not match score extent"):
        M.malis_softmax_loss(wrong, fg)
    # the C ABI rejects C != 2 with the same message
    with pytest.raises(g.SizeError, match="needs exactly 2 score channels"):
        from paper_1509_03371_b200 import _lib

        sc = np.zeros((1, 3, 2, 2), np.float32)
        d = np.zeros_like(sc)
        loss = np.zeros(1)
        _lib.check(_lib.lib().graft_malis_softmax_loss_f32(_lib.ptr(sc), 1, 3, 2, 2, _lib.ptr(fg), _lib.ptr(d),
                                                           _lib.ptr(loss), _lib.MEM_HOST))


def test_composed_loss_blob_accumulates():
    rng = np.random.default_rng(550)
    fg = (rng.random((4, 4)) < 0.5).astype(np.uint8)
    b = g.Blob(2, 4, 4, np.float64)
    b.data = rng.uniform(-1.0, 1.0, b.size())
    b.diff = rng.uniform(-1.0, 1.0, b.size())
    d0 = b.diff.copy()
    loss = M.malis_softmax_loss(b, fg)
    lw, dw = O.malis_softmax_loss(b.data.reshape(2, 4, 4), fg, d0.reshape(2, 4, 4))
    assert loss == lw
    assert_bitwise(b.diff.reshape(2, 4, 4), dw, "accumulated diff")


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_net_runner_malis_loss_matches_reference():
    """The device training step's MALIS loss on the score blob of a small net (float)."""
    text = ("input w=12 f=1\n"
            "layer conv1 conv_sk k=3 fout=4 in=data out=conv1 init=gaussian:0.5\n"
            "layer relu1 relu in=conv1 out=relu1\n"
            "layer conv2 conv_sk k=3 fout=2 in=relu1 out=conv2 init=gaussian:0.5\n"
            "layer prob softmax_loss in=conv2 out=prob\n")
    ref = O.RefNet(text, seed=9)
    spec = g.parse_netspec_or_throw(text)
    states = g.init_weights(spec, 9)
    runner = g.NetRunner(spec, states)
    x = O.Rng(3).uniform_f32(1 * 24 * 24).reshape(1, 24, 24)
    runner.forward(g.Blob.from_array(x))
    ref.forward(x)
    scores = ref.blob("conv2")
    assert_bitwise(runner.blob("conv2").view(), scores, "scores")
    fg = (np.random.default_rng(5).random(scores.shape[1:]) < 0.5).astype(np.uint8)
    runner.zero_blob_diffs()
    loss = runner.malis_softmax_loss("conv2", fg)
    lw, dw = O.malis_softmax_loss(scores, fg, np.zeros_like(scores), "ref")
    assert loss == lw
    assert_bitwise(runner.blob_diff("conv2").reshape(scores.shape), dw, "conv2 diff")
