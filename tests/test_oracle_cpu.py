"""Pins the CPU oracle (oracle/pixelseg_oracle.c) before it is trusted as the checker:
against the reference's own known-answer values (the frozen numbers in proj/tests) and against
golden vectors produced by the reference itself (tests/golden/*.npz, made by
tests/golden/make_golden.py from oracle/_ref). CPU only."""
import numpy as np
import pytest

from conftest import assert_bitwise, config_text
from oracle import oracle as O
from paper_1509_03371_b200.netspec import (LayerKind, flop_estimate, parse_netspec_or_throw,
                                           propagate_sizes)


# ---- frozen known answers of the reference's tests ----------------------------------------
def test_frozen_strided_gather():
    # proj/tests/test_tensor.cpp:59-76: 7x7 k=3 d=2, tap (2,2) of output (0,0) reads (4,4) = 44
    x = np.array([[10.0 * y + x for x in range(7)] for y in range(7)], np.float32)[None]
    col = O.im2col(x, 3, 2)
    assert col.shape == (9, 9)
    assert col[(0 * 3 + 2) * 3 + 2, 0] == x[0, 4, 4] == 44.0


def test_frozen_gemm_2x2():
    # proj/tests/test_tensor.cpp:161-170
    a = np.array([1, 2, 3, 4], np.float32)
    b = np.array([5, 6, 7, 8], np.float32)
    c = np.full(4, -1, np.float32)
    O.gemm(0, 0, 2, 2, 2, 1.0, a, b, 0.0, c)
    assert c.tolist() == [19.0, 22.0, 43.0, 50.0]


def test_gemm_column_chunk_invariance(glayers):
    # proj/tests/test_tensor.cpp:198-219: a column subset is bit-identical
    m, n, k = 6, 32, 50
    A, B = glayers["gemmcc_A"], glayers["gemmcc_B"]
    c = np.zeros(m * n, np.float32)
    O.gemm(0, 0, m, n, k, 1.0, A, B, 0.0, c)
    assert_bitwise(c, glayers["gemmcc_out"], "gemm")
    n1 = 13
    Bs = np.ascontiguousarray(B.reshape(k, n)[:, :n1])
    cs = np.zeros(m * n1, np.float32)
    O.gemm(0, 0, m, n1, k, 1.0, A, Bs, 0.0, cs)
    assert_bitwise(cs.reshape(m, n1), c.reshape(m, n)[:, :n1], "gemm subset")


def test_identity_kernels():
    # proj/tests/test_layers.cpp:60-78
    x = O.Rng(3).uniform_f32(25).reshape(1, 5, 5)
    assert_bitwise(O.conv(x, np.ones(1, np.float32), np.zeros(1, np.float32), 1, 1), x)
    w = np.zeros(9, np.float32)
    w[4] = 1.0
    assert_bitwise(O.conv(x, w, np.zeros(1, np.float32), 1, 3, p_=1), x)


# ---- oracle == reference, bit for bit, on the golden vectors ---------------------------------
def test_conv_cases(glayers):
    for i, (fi, fo, h, w, k, d, s, p_) in enumerate(glayers["conv_cases"]):
        out = O.conv(glayers[f"conv{i}_in"], glayers[f"conv{i}_w"], glayers[f"conv{i}_b"], fo, k,
                     d, s, p_)
        assert_bitwise(out, glayers[f"conv{i}_out"], f"conv case {i}")
        out64 = O.conv(glayers[f"conv64_{i}_in"], glayers[f"conv64_{i}_w"],
                       glayers[f"conv64_{i}_b"], fo, k, d, s, p_)
        assert_bitwise(out64, glayers[f"conv64_{i}_out"], f"conv f64 case {i}")


def test_sk_shaped_conv_cases(glayers):
    for i, (fi, fo, h, w, k, d) in enumerate(glayers["sk_cases"]):
        out = O.conv(glayers[f"sk{i}_in"], glayers[f"sk{i}_w"], glayers[f"sk{i}_b"], fo, k, d,
                     threads=4)
        assert_bitwise(out, glayers[f"sk{i}_out"], f"sk case {i}")


def test_pool_and_ties(glayers):
    for i in range(4):
        k, d, s, hw = glayers[f"pool{i}_cfg"]
        out, am = O.maxpool(glayers[f"pool{i}_in"], k, d, s, want_argmax=True)
        assert_bitwise(out, glayers[f"pool{i}_out"], f"pool {i}")
        assert np.array_equal(am, glayers[f"pool{i}_argmax"])
    out, am = O.maxpool(np.full((1, 4, 4), 2.5, np.float32), 2, 1, 2, want_argmax=True)
    assert am.tolist() == [0, 2, 8, 10]  # test_layers.cpp:185-191: smallest linear index
    assert np.array_equal(am, glayers["pool_flat_argmax"])


def test_elementwise(glayers):
    assert_bitwise(O.relu(glayers["relu_in"]), glayers["relu_out"], "relu")
    assert_bitwise(O.upconv(glayers["up_in"]), glayers["up_out"], "upconv")
    assert_bitwise(O.mergecrop(glayers["mc_a"], glayers["mc_b"]), glayers["mc_out"], "mergecrop")
    for name in ("sm3", "sm2", "sm_ext"):
        assert_bitwise(O.softmax(glayers[name + "_in"]), glayers[name + "_out"], name)


def test_im2col_cases(glayers):
    for i, (c, h, w, k, d, s, p_) in enumerate(glayers["im2col_cases"]):
        assert_bitwise(O.im2col(glayers[f"im2col{i}_in"], k, d, s, p_), glayers[f"im2col{i}_out"],
                       f"im2col {i}")


def test_gemm_variants(glayers):
    m, n, k = 4, 5, 3
    A, B, Cin = glayers["gemm_A"], glayers["gemm_B"], glayers["gemm_C"]
    for ta in (0, 1):
        for tb in (0, 1):
            a = A.reshape(m, k).T.copy().ravel() if ta else A
            b = B.reshape(k, n).T.copy().ravel() if tb else B
            for alpha, beta in ((1.0, 0.0), (2.0, 1.0), (-0.5, 0.25)):
                c = Cin.copy()
                O.gemm(ta, tb, m, n, k, alpha, a, b, beta, c)
                assert_bitwise(c, glayers[f"gemm_{ta}{tb}_{alpha}_{beta}"], "gemm")
    c = glayers["gemm64_C"].copy()
    O.gemm(0, 0, m, n, k, 2.0, glayers["gemm64_A"], glayers["gemm64_B"], 1.0, c)
    assert_bitwise(c, glayers["gemm64_out"], "gemm f64")


def test_pad_normalize(glayers):
    img = glayers["pad_img"]
    for v in (0, 1, 5, 10):
        assert np.array_equal(O.mirror_pad(img, v), glayers[f"pad_v{v}"])
    assert_bitwise(O.normalize(np.arange(256, dtype=np.uint8)), glayers["normalize_lut"])
    with pytest.raises(O.OracleError, match="needs an image larger"):
        O.mirror_pad(img[:5, :5], 10)


def test_rng_matches_reference_init(gnets):
    # init_weights(spec, 7) of the hand-chained net == the reference's (fixture came from it)
    spec = parse_netspec_or_throw(bytes(gnets["chain_spec"]).decode())
    params = O.init_weights(spec, 7)
    out = O.forward_net(spec, params, gnets["chain_in"], keep=True)
    for name in ("conv1", "relu1", "pool1", "conv2", "prob"):
        assert_bitwise(out[name], gnets[f"chain_{name}"], name)


# ---- nets / process restated over the C layers == reference ---------------------------------
def _spec(gnets, key):
    return parse_netspec_or_throw(bytes(gnets[key]).decode())


def test_unet_small(gnets):
    spec = _spec(gnets, "unet_spec")
    out = O.forward_net(spec, O.init_weights(spec, 11), gnets["unet_in"], keep=True)
    for name in ("conv1", "pool1", "conv2", "upconv1", "merge1", "conv3", "prob"):
        assert_bitwise(out[name], gnets[f"unet_{name}"], name)


def _sk_small():
    spec = parse_netspec_or_throw(config_text("sk.net"))
    fo = {"conv1": 6, "conv2": 8, "conv3": 12, "ip1": 16, "ip2": 8, "ip3": 2}
    for l in spec.layers:
        if l.name in fo:
            l.f_out = fo[l.name]
            l.init_sigma = 0.1
    return spec


def test_sk_small_and_crop(gnets):
    # proj/tests/test_netgraph.cpp:277-308 with every blob pinned
    spec = _sk_small()
    params = O.init_weights(spec, 3)
    out = O.forward_net(spec, params, gnets["sksmall_in"], keep=True)
    for name in ("conv1", "relu1", "pool1", "conv2", "pool2", "conv3", "pool3", "ip1", "relu4",
                 "ip2", "ip3", "prob"):
        assert_bitwise(out[name], gnets[f"sksmall_{name}"], name)
    crop = O.forward_net(spec, params, np.ascontiguousarray(gnets["sksmall_in"][:, :102, :102]))
    assert_bitwise(crop, gnets["sksmall_crop_prob"], "crop")
    assert np.abs(crop[:, 0, 0] - out["prob"][:, 0, 0]).max() <= 1e-5


def test_sw_net(gnets):
    spec = _spec(gnets, "sw_spec")
    out = O.forward_net(spec, O.init_weights(spec, 1), gnets["sw_in"], keep=True, threads=8)
    for name in ("ip1", "ip3", "prob"):
        assert_bitwise(out[name], gnets[f"sw_{name}"], name)


def test_tiled_process(gnets):
    spec = _spec(gnets, "tile_spec")
    params = O.init_weights(spec, 17)
    for key, img, w in (("w16", "tile_img", 16), ("w8", "tile_img", 8), ("o13", "tile_odd", 13),
                        ("o6", "tile_odd", 6)):
        lab, pr = O.process(spec, params, gnets[img], w, 5)
        assert np.array_equal(lab, gnets[f"tile_{key}_labels"])
        assert_bitwise(pr, gnets[f"tile_{key}_probs"], key)
    # the reference's own invariance: tile size does not change a bit
    assert_bitwise(gnets["tile_w16_probs"], gnets["tile_w8_probs"])
    assert_bitwise(gnets["tile_o13_probs"], gnets["tile_o6_probs"])


def test_sk_small_process(gnets):
    spec = _sk_small()
    params = O.init_weights(spec, 3)
    lab, pr = O.process(spec, params, gnets["skproc_img"], 16, 101)
    assert np.array_equal(lab, gnets["skproc_w16_labels"])
    assert_bitwise(pr, gnets["skproc_w16_probs"])
    assert_bitwise(gnets["skproc_w9_probs"], gnets["skproc_w16_probs"])


# ---- size / cost model (convert.hpp) against the paper's published table ---------------------
def test_sk_sizes_and_flops():
    spec = parse_netspec_or_throw(config_text("sk.net"))
    rows = {r.name: r for r in propagate_sizes(spec, 229)}
    assert [rows[n].w_out for n in ("conv1", "pool1", "conv2", "pool2", "conv3", "pool3", "ip1",
                                    "ip3")] == [223, 222, 214, 212, 204, 200, 128, 128]
    fl = flop_estimate(spec, 229)
    # PAPER.md:2015-2020 (GFLOP 0.70, 14.06, 18.40, 644.23, 17.17, 0.03)
    assert [round(fl[n] / 1e9, 2) for n in ("conv1", "conv2", "conv3", "ip1", "ip2", "ip3")] == \
        [0.70, 14.06, 18.40, 644.23, 17.17, 0.03]
    assert fl["ip1"] == 644228317184  # test_tensor.cpp:223
    assert fl["total"] == 694596973808


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference)")
def test_oracle_vs_live_reference_random_geometries():
    r = O.Rng(123)
    for t in range(30):
        fi = 1 + int(r.uniform(0, 5))
        fo = 1 + int(r.uniform(0, 6))
        k = 1 + int(r.uniform(0, 4))
        d = 1 + int(r.uniform(0, 3))
        s = 1 + int(r.uniform(0, 2))
        p_ = int(r.uniform(0, 2))
        span = (k - 1) * d + 1
        h = span + s * int(r.uniform(0, 6)) - 2 * p_
        if h < 1:
            continue
        x = r.uniform_f32(fi * h * h).reshape(fi, h, h)
        w = r.uniform_f32(fo * fi * k * k)
        b = r.uniform_f32(fo)
        out = O.conv(x, w, b, fo, k, d, s, p_)
        ref = np.empty_like(out)
        assert O.ref().ref_conv_f32(O.p(x), fi, h, h, O.p(w), O.p(b), fo, k, d, s, p_,
                                    O.p(ref)) == 0
        assert_bitwise(out, ref, f"trial {t}")


# ---- MALIS (malis.hpp): the C restatement against the reference-made fixtures ------------
def test_oracle_malis_matches_reference_goldens():
    from conftest import load_golden

    gold = load_golden("malis.npz")
    for ci, (h, w) in enumerate(gold["cases"]):
        key = f"c{ci}"
        fg = gold[f"{key}_fg"]
        comp = O.malis_components(fg)
        assert np.array_equal(comp, gold[f"{key}_comp"]), key
        for t in ("f32", "f64"):
            k = f"{key}_{t}"
            pax, pay, pmx, pmy = O.malis_affinity_forward(gold[f"{k}_probs"])
            for n, a in (("pax", pax), ("pay", pay), ("pmx", pmx), ("pmy", pmy)):
                assert_bitwise(a, gold[f"{k}_{n}"], f"{k} {n}")
            r = O.malis_gradient(pax, pay, gold[f"{k}_tax"], gold[f"{k}_tay"], comp)
            for n in ("da_x", "da_y", "pos_x", "pos_y", "neg_x", "neg_y", "totals", "losses"):
                assert_bitwise(r[n], gold[f"{k}_{n}"], f"{k} {n}")
            dp, dn = O.malis_affinity_backward(gold[f"{k}_dgx"], gold[f"{k}_dgy"], pmx, pmy)
            assert_bitwise(dp, gold[f"{k}_dpos"], f"{k} dpos")
            assert_bitwise(dn, gold[f"{k}_dneg"], f"{k} dneg")
            loss, d = O.malis_softmax_loss(gold[f"{k}_scores"], fg, gold[f"{k}_diff0"])
            assert_bitwise(np.array([loss]), gold[f"{k}_loss"], f"{k} loss")
            assert_bitwise(d, gold[f"{k}_diff"], f"{k} diff")
