"""Generates the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Every output array below is produced by the unmodified reference headers
(/root/reference/proj/include/pixelseg), compiled into oracle/_ref/libpixelseg_ref.so by
oracle/Makefile and called through oracle/ref_shim.cpp. Inputs are drawn with the reference's
own Rng in the order the reference's tests draw them (file:line cited per fixture), so the
fixtures are the reference tests' own data.

    python tests/golden/make_golden.py small     # seconds: layers.npz, nets.npz
    python tests/golden/make_golden.py sk229     # ~10 min: full sk.net at 229 (pixelseg bench)
    python tests/golden/make_golden.py u572 usk692
    python tests/golden/make_golden.py strided     # ~1 min: multi-tile u.net/usk.net process()
    python tests/golden/make_golden.py skproc      # ~75 min: full sk.net process() 260x230
    python tests/golden/make_golden.py malis       # seconds: MALIS (malis.hpp) instances

Runs only where /root/reference exists (the dev container); the .npz files are committed.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

CONFIGS = "/root/reference/proj/configs"
OUT = os.path.dirname(os.path.abspath(__file__))
P = O.p


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_conv(x, w, b, fo, k, d, s, p_):
    fn = O.ref().ref_conv_f64 if x.dtype == np.float64 else O.ref().ref_conv_f32
    oh = O.out_extent(x.shape[1], k, d, s, p_, "height")
    ow = O.out_extent(x.shape[2], k, d, s, p_, "width")
    out = np.empty((fo, oh, ow), x.dtype)
    assert fn(P(x), *x.shape, P(w), P(b), fo, k, d, s, p_, P(out)) == 0
    return out


def small():
    f = {}
    # conv forward == direct loop bit for bit (proj/tests/test_layers.cpp:80-105), Rng(5)
    cases = [(3, 4, 9, 9, 3, 1, 1, 0), (2, 5, 11, 11, 3, 2, 1, 0), (4, 2, 8, 8, 2, 1, 2, 0),
             (1, 3, 7, 7, 7, 1, 1, 0), (2, 2, 6, 6, 3, 1, 1, 1)]
    f["conv_cases"] = np.array(cases, np.int32)
    r = O.Rng(5)
    for i, (fi, fo, h, w, k, d, s, p_) in enumerate(cases):
        x = r.uniform_f32(fi * h * w).reshape(fi, h, w)
        W = r.uniform_f32(fo * fi * k * k)
        b = r.uniform_f32(fo)
        f[f"conv{i}_in"], f[f"conv{i}_w"], f[f"conv{i}_b"] = x, W, b
        f[f"conv{i}_out"] = ref_conv(x, W, b, fo, k, d, s, p_)
    # the same geometries in S=double
    r = O.Rng(6)
    for i, (fi, fo, h, w, k, d, s, p_) in enumerate(cases):
        x = r.uniform_f64(fi * h * w).reshape(fi, h, w)
        W = r.uniform_f64(fo * fi * k * k)
        b = r.uniform_f64(fo)
        f[f"conv64_{i}_in"], f[f"conv64_{i}_w"], f[f"conv64_{i}_b"] = x, W, b
        f[f"conv64_{i}_out"] = ref_conv(x, W, b, fo, k, d, s, p_)
    # sk.net-shaped layers at reduced extents (dilations 2,4,8 and a 10x10 spanning kernel)
    sk_layers = [(3, 16, 40, 40, 7, 1), (16, 24, 30, 30, 5, 2), (24, 32, 30, 30, 3, 4),
                 (12, 40, 80, 80, 10, 8), (64, 33, 9, 9, 1, 1), (520, 2, 5, 5, 1, 1)]
    f["sk_cases"] = np.array(sk_layers, np.int32)
    r = O.Rng(29)
    for i, (fi, fo, h, w, k, d) in enumerate(sk_layers):
        x = r.uniform_f32(fi * h * w).reshape(fi, h, w)
        W = r.gaussian_f32(fo * fi * k * k, 0.0, 0.05)
        b = r.uniform_f32(fo, -0.1, 0.1)
        f[f"sk{i}_in"], f[f"sk{i}_w"], f[f"sk{i}_b"] = x, W, b
        f[f"sk{i}_out"] = ref_conv(x, W, b, fo, k, d, 1, 0)
    # max pool + ties (proj/tests/test_layers.cpp:166-192), Rng(11)
    r = O.Rng(11)
    for i, (k, d, s, hw) in enumerate([(2, 1, 2, 8), (2, 2, 1, 9), (2, 4, 1, 13), (3, 1, 3, 9)]):
        x = r.uniform_f32(3 * hw * hw).reshape(3, hw, hw)
        oh = O.out_extent(hw, k, d, s, 0)
        out = np.empty((3, oh, oh), np.float32)
        am = np.empty(out.size, np.uint64)
        assert O.ref().ref_maxpool_f32(P(x), 3, hw, hw, k, d, s, P(out), P(am)) == 0
        f[f"pool{i}_cfg"] = np.array([k, d, s, hw], np.int32)
        f[f"pool{i}_in"], f[f"pool{i}_out"], f[f"pool{i}_argmax"] = x, out, am
    flat = np.full((1, 4, 4), 2.5, np.float32)
    out = np.empty((1, 2, 2), np.float32)
    am = np.empty(4, np.uint64)
    assert O.ref().ref_maxpool_f32(P(flat), 1, 4, 4, 2, 1, 2, P(out), P(am)) == 0
    f["pool_flat_out"], f["pool_flat_argmax"] = out, am
    # relu with -0, NaN, +-inf, subnormals
    x = np.array([-1.0, -0.0, 0.0, 0.5, 2.0, np.inf, -np.inf, np.nan, 1e-45, -1e-45],
                 np.float32).reshape(1, 1, -1)
    out = np.empty_like(x)
    O.ref().ref_relu_f32(P(x), 1, 1, x.shape[2], P(out))
    f["relu_in"], f["relu_out"] = x, out
    # upconv / mergecrop (test_layers.cpp:219-280)
    r = O.Rng(19)
    x = r.uniform_f32(2 * 3 * 5).reshape(2, 3, 5)
    out = np.empty((2, 6, 10), np.float32)
    O.ref().ref_upconv_f32(P(x), 2, 3, 5, P(out))
    f["up_in"], f["up_out"] = x, out
    a = r.uniform_f32(3 * 4 * 5).reshape(3, 4, 5)
    b = r.uniform_f32(2 * 9 * 8).reshape(2, 9, 8)
    out = np.empty((5, 4, 5), np.float32)
    assert O.ref().ref_mergecrop_f32(P(a), 3, 4, 5, P(b), 2, 9, 8, P(out)) == 0
    f["mc_a"], f["mc_b"], f["mc_out"] = a, b, out
    # softmax: random 3-class (test_layers.cpp:334-357 shape), 2-class sk-like small scores,
    # and extremes
    r = O.Rng(23)
    for name, x in [("sm3", r.uniform_f32(3 * 4 * 4, -2, 2).reshape(3, 4, 4)),
                    ("sm2", (r.uniform_f32(2 * 64 * 64, -1, 1) * 3e-4).reshape(2, 64, 64)),
                    ("sm_ext", np.array([[[0, 100, -100, 1e-30, 88.0, -87.0, 50.0, 0.5]],
                                         [[0, -100, 100, -1e-30, -88.0, 87.0, -60.0, 0.5]]],
                                        np.float32))]:
        out = np.empty_like(x)
        O.ref().ref_softmax_f32(P(x), *x.shape, P(out))
        f[name + "_in"], f[name + "_out"] = x, out
    # im2col (test_tensor.cpp:78-98 geometries), Rng(11) in float
    geos = [(1, 7, 7, 3, 2, 1, 0), (2, 9, 8, 3, 1, 1, 1), (3, 10, 10, 2, 1, 2, 0),
            (2, 11, 11, 3, 3, 1, 0), (1, 7, 7, 2, 2, 2, 0), (4, 5, 5, 5, 1, 1, 2)]
    f["im2col_cases"] = np.array(geos, np.int32)
    r = O.Rng(11)
    for i, (c, h, w, k, d, s, p_) in enumerate(geos):
        x = r.uniform_f32(c * h * w).reshape(c, h, w)
        oh, ow = O.out_extent(h, k, d, s, p_), O.out_extent(w, k, d, s, p_)
        col = np.empty((c * k * k, oh * ow), np.float32)
        assert O.ref().ref_im2col_f32(P(x), c, h, w, k, d, s, p_, P(col)) == 0
        f[f"im2col{i}_in"], f[f"im2col{i}_out"] = x, col
    # gemm: transposes + alpha/beta (test_tensor.cpp:172-196), column-chunk (198-219)
    r = O.Rng(17)
    m, n, k = 4, 5, 3
    A = r.uniform_f32(m * k)
    B = r.uniform_f32(k * n)
    Cin = r.uniform_f32(m * n)
    for ta in (0, 1):
        for tb in (0, 1):
            a = A.reshape(m, k).T.copy().ravel() if ta else A
            b = B.reshape(k, n).T.copy().ravel() if tb else B
            for alpha, beta in ((1.0, 0.0), (2.0, 1.0), (-0.5, 0.25)):
                c = Cin.copy()
                O.ref().ref_gemm_f32(ta, tb, m, n, k, alpha, P(a), P(b), beta, P(c))
                f[f"gemm_{ta}{tb}_{alpha}_{beta}"] = c
    f["gemm_A"], f["gemm_B"], f["gemm_C"] = A, B, Cin
    r = O.Rng(18)
    A64, B64, C64 = r.uniform_f64(m * k), r.uniform_f64(k * n), r.uniform_f64(m * n)
    c = C64.copy()
    O.ref().ref_gemm_f64(0, 0, m, n, k, 2.0, P(A64), P(B64), 1.0, P(c))
    f["gemm64_A"], f["gemm64_B"], f["gemm64_C"], f["gemm64_out"] = A64, B64, C64, c
    r = O.Rng(19)
    m, n, k = 6, 32, 50
    A, B = r.uniform_f32(m * k), r.uniform_f32(k * n)
    c = np.zeros(m * n, np.float32)
    O.ref().ref_gemm_f32(0, 0, m, n, k, 1.0, P(A), P(B), 0.0, P(c))
    f["gemmcc_A"], f["gemmcc_B"], f["gemmcc_out"] = A, B, c
    # mirror_pad + normalize (pipeline.hpp:36-93)
    r = O.Rng(55)
    img = r.index_u8(13 * 11, 256).reshape(13, 11)
    for v in (0, 1, 5, 10):
        out = np.empty((13 + v, 11 + v), np.uint8)
        assert O.ref().ref_mirror_pad_u8(P(img), 13, 11, v, P(out)) == 0
        f[f"pad_v{v}"] = out
    f["pad_img"] = img
    allv = np.arange(256, dtype=np.uint8)
    out = np.empty(256, np.float32)
    O.ref().ref_normalize_f32(P(allv), 256, P(out))
    f["normalize_lut"] = out
    np.savez_compressed(os.path.join(OUT, "layers.npz"), **f)
    print("layers.npz", len(f), "arrays")


def net_fixture(f, key, text, seed, x, fout=None, sigma=0.0, names=None):
    net = O.RefNet(text, seed=seed, fout=fout, sigma=sigma)
    net.forward(x)
    f[key + "_in"] = x
    for nm in names:
        f[f"{key}_{nm}"] = net.blob(nm)
    return net


def nets():
    f = {}
    # hand-chained small net (proj/tests/test_netgraph.cpp:156-218), float instantiation
    t1 = ("input w=8 f=2\n"
          "layer conv1 conv_sk k=3 fout=3 in=data out=conv1 init=gaussian:0.5\n"
          "layer relu1 relu in=conv1 out=relu1\n"
          "layer pool1 pool_max k=2 s=2 in=relu1 out=pool1\n"
          "layer conv2 conv_sk k=3 fout=2 in=pool1 out=conv2 init=gaussian:0.5\n"
          "layer prob softmax_loss in=conv2 out=prob\n")
    r = O.Rng(99)
    net_fixture(f, "chain", t1, 7, r.uniform_f32(2 * 8 * 8).reshape(2, 8, 8),
                names=["conv1", "relu1", "pool1", "conv2", "prob"])
    f["chain_spec"] = np.frombuffer(t1.encode(), np.uint8)
    # u-topology (proj/tests/test_netgraph.cpp:238-275)
    t2 = ("input w=16 f=1\n"
          "layer conv1 conv_sk k=3 fout=2 in=data out=conv1 init=gaussian:0.4\n"
          "layer pool1 pool_max k=2 s=2 in=conv1 out=pool1\n"
          "layer conv2 conv_sk k=3 fout=4 in=pool1 out=conv2 init=gaussian:0.4\n"
          "layer upconv1 upconv in=conv2 out=upconv1\n"
          "layer merge1 mergecrop in=upconv1,conv1 out=merge1\n"
          "layer conv3 conv_sk k=3 fout=2 in=merge1 out=conv3 init=gaussian:0.4\n"
          "layer prob softmax_loss in=conv3 out=prob\n")
    r = O.Rng(5)
    net_fixture(f, "unet", t2, 11, r.uniform_f32(16 * 16).reshape(1, 16, 16),
                names=["conv1", "pool1", "conv2", "upconv1", "merge1", "conv3", "prob"])
    f["unet_spec"] = np.frombuffer(t2.encode(), np.uint8)
    # reduced sk.net at 110 and its 102 crop (proj/tests/test_netgraph.cpp:277-308)
    sk = open(os.path.join(CONFIGS, "sk.net")).read()
    fo = {"conv1": 6, "conv2": 8, "conv3": 12, "ip1": 16, "ip2": 8, "ip3": 2}
    r = O.Rng(17)
    big = r.uniform_f32(3 * 110 * 110).reshape(3, 110, 110)
    names = ["conv1", "relu1", "pool1", "conv2", "pool2", "conv3", "pool3", "ip1", "relu4",
             "ip2", "ip3", "prob"]
    net = net_fixture(f, "sksmall", sk, 3, big, fout=fo, sigma=0.1, names=names)
    net.forward(np.ascontiguousarray(big[:, :102, :102]))
    f["sksmall_crop_prob"] = net.blob("prob")
    f["sksmall_crop_ip3"] = net.blob("ip3")
    # corrected sw.net at its corrected w0 (convert.hpp:175-195): one label
    sw = O.correct_sw(open(os.path.join(CONFIGS, "sw.net")).read())
    f["sw_spec"] = np.frombuffer(sw.encode(), np.uint8)
    w0 = int(sw.split("w=")[1].split()[0])
    r = O.Rng(1 ^ 0x9e3779b97f4a7c15)
    x = r.uniform_f32(3 * w0 * w0).reshape(3, w0, w0)
    net_fixture(f, "sw", sw, 1, x, names=["ip1", "ip3", "prob"])
    # tiled inference (proj/tests/test_pipeline.cpp:535-588)
    t3 = ("input w=21 f=1\n"
          "layer c1 conv_sk k=3 fout=4 in=data out=c1 init=he\n"
          "layer r1 relu in=c1 out=r1\n"
          "layer p1 pool_max k=2 s=1 in=r1 out=p1\n"
          "layer c2 conv_sk k=2 d=2 fout=3 in=p1 out=c2 init=he\n"
          "layer prob softmax_loss in=c2 out=prob\n")
    f["tile_spec"] = np.frombuffer(t3.encode(), np.uint8)
    net = O.RefNet(t3, seed=17)
    net.n_classes = 3
    r = O.Rng(55)
    img = r.index_u8(16 * 16).reshape(16, 16)
    odd = r.index_u8(14 * 13).reshape(14, 13)
    f["tile_img"], f["tile_odd"] = img, odd
    for key, im, w in (("w16", img, 16), ("w8", img, 8), ("o13", odd, 13), ("o6", odd, 6)):
        lab, pr = net.process(im, w, 5)
        f[f"tile_{key}_labels"], f[f"tile_{key}_probs"] = lab, pr
    # reduced sk.net process() over a 60x57 image with 9- and 16-pixel tiles
    net = O.RefNet(sk, seed=3, fout=fo, sigma=0.1)
    r = O.Rng(77)
    img = r.index_u8(60 * 57).reshape(60, 57)
    f["skproc_img"] = img
    for w in (9, 16):
        lab, pr = net.process(img, w, 101)
        f[f"skproc_w{w}_labels"], f[f"skproc_w{w}_probs"] = lab, pr
    np.savez_compressed(os.path.join(OUT, "nets.npz"), **f)
    print("nets.npz", len(f), "arrays")


FULL = {"sk229": ("sk.net", 229), "u572": ("u.net", 572), "usk692": ("usk.net", 692)}


def full(key):
    """pixelseg bench --net <cfg> --seed 1 input (proj/tools/pixelseg.cpp:203-207), full net."""
    cfg, w0 = FULL[key]
    text = open(os.path.join(CONFIGS, cfg)).read()
    from paper_1509_03371_b200.netspec import parse_netspec_or_throw

    spec = parse_netspec_or_throw(text)
    net = O.RefNet(text, seed=1)
    r = O.Rng(1 ^ 0x9e3779b97f4a7c15)
    x = r.uniform_f32(3 * w0 * w0).reshape(3, w0, w0)
    net.forward(x)
    f = {"in_sha": np.frombuffer(sha(x).encode(), np.uint8)}
    rng = np.random.default_rng(0)
    for l in spec.layers[1:]:
        b = net.blob(l.output)
        f[f"sha_{l.output}"] = np.frombuffer(sha(b).encode(), np.uint8)
        f[f"shape_{l.output}"] = np.array(b.shape, np.int64)
        idx = rng.integers(0, b.size, 4096)
        f[f"sampidx_{l.output}"] = idx
        f[f"sampval_{l.output}"] = b.ravel()[idx]
    last = spec.layers[-1]
    f["prob"] = net.blob(last.output)
    f["scores"] = net.blob(last.inputs[0])
    np.savez_compressed(os.path.join(OUT, f"{key}.npz"), **f)
    print(f"{key}.npz written")


def configs():
    """The four proj/configs net descriptions (the parity workloads), as fixture data."""
    f = {}
    for name in ("sk.net", "sw.net", "u.net", "usk.net"):
        f[name.split(".")[0]] = np.frombuffer(open(os.path.join(CONFIGS, name), "rb").read(), np.uint8)
    np.savez_compressed(os.path.join(OUT, "configs.npz"), **f)
    print("configs.npz", len(f), "arrays")


CLI_NET = """input w=229 f=3
layer conv1 conv_sk k=7 d=1 fout=6 in=data out=conv1 init=gaussian:0.1
layer relu1 relu in=conv1 out=relu1
layer pool1 pool_max k=2 s=1 d=1 in=relu1 out=pool1
layer conv2 conv_sk k=5 d=2 fout=8 in=pool1 out=conv2 init=gaussian:0.1
layer relu2 relu in=conv2 out=relu2
layer pool2 pool_max k=2 s=1 d=2 in=relu2 out=pool2
layer conv3 conv_sk k=3 d=4 fout=12 in=pool2 out=conv3 init=gaussian:0.1
layer relu3 relu in=conv3 out=relu3
layer pool3 pool_max k=2 s=1 d=4 in=relu3 out=pool3
layer ip1 conv_sk k=10 d=8 fout=16 in=pool3 out=ip1 init=gaussian:0.1
layer relu4 relu in=ip1 out=relu4
layer ip2 conv_sk k=1 d=1 fout=8 in=relu4 out=ip2 init=gaussian:0.1
layer relu5 relu in=ip2 out=relu5
layer ip3 conv_sk k=1 d=1 fout=2 in=relu5 out=ip3 init=gaussian:0.1
layer prob softmax_loss in=ip3 out=prob
"""


def write_png_gray(path, img):
    """8-bit grayscale, non-interlaced PNG (filter 0 rows), read by image_io.hpp:95-174."""
    import struct
    import zlib

    def chunk(tag, data):
        return (struct.pack(">I", len(data)) + tag + data +
                struct.pack(">I", zlib.crc32(tag + data) & 0xFFFFFFFF))

    h, w = img.shape
    raw = b"".join(b"\x00" + img[y].tobytes() for y in range(h))
    with open(path, "wb") as fh:
        fh.write(b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, 8, 0, 0, 0, 0))
                 + chunk(b"IDAT", zlib.compress(raw)) + chunk(b"IEND", b""))


def cli():
    """Fixtures for `pixelseg_gpu process` (proj/tools/pixelseg.cpp:161-191): a reduced-channel
    sk.net spec file, its PXSG weights written by the reference's save_weights
    (weights_io.hpp), a 300x260 gray scan written by the reference's write_pgm (and the same
    pixels as PNG), and the expected output files: labels from the reference's process<float>
    at the CLI's default tile (128) and the 8-bit probability maps the CLI derives from the
    probs (clamp to [0,1], lround(p*255), pixelseg.cpp:179-183)."""
    d = os.path.join(OUT, "cli")
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, "sk_small.net"), "w") as fh:
        fh.write(CLI_NET)
    net = O.RefNet(CLI_NET, seed=3)
    net.save_weights(os.path.join(d, "sk_small.pxsg"))
    img = O.Rng(55).index_u8(300 * 260).reshape(300, 260)
    O.write_pgm(os.path.join(d, "scan.pgm"), img)
    write_png_gray(os.path.join(d, "scan.png"), img)
    labels, probs = net.process(img, 128, 101)
    O.write_pgm(os.path.join(d, "expect_scan_labels.pgm"), labels)
    for c in range(probs.shape[0]):
        m = np.floor(np.clip(probs[c].astype(np.float64), 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)
        O.write_pgm(os.path.join(d, f"expect_scan_prob{c}.pgm"), m)
    np.save(os.path.join(d, "expect_scan_probs.npy"), probs)


# Reduced-channel u.net / usk.net (the configs' own topology, strided pools and upconvs) for
# multi-tile process(). Odd image sizes make the snapped edge tiles start at an odd offset, so
# overlapping tiles see the strided pools at the opposite parity and produce different values:
# the planes then pin both the reference's tile origins and its later-tile-wins stitch
# (pipeline.hpp:662-672, 685-694).
U_FOUT = {"conv1": 4, "conv2": 4, "conv3": 8, "conv4": 8, "conv5": 16, "conv6": 16, "conv7": 32,
          "conv8": 32, "conv9": 64, "conv10": 64, "conv11": 32, "conv12": 32, "conv13": 32,
          "conv14": 16, "conv15": 16, "conv16": 16, "conv17": 8, "conv18": 8, "conv19": 8,
          "conv20": 4, "conv21": 4, "conv22": 4, "ip1": 2}
USK_FOUT = {"conv1": 8, "conv2": 8, "conv3": 16, "conv4": 16, "conv5": 16, "ip1": 64, "ip2": 32,
            "conv6": 16, "conv7": 16, "conv8": 8, "ip3": 2}
STRIDED = (("u", "u.net", U_FOUT, 0.0, 36, 184, 101, 97),
           ("usk", "usk.net", USK_FOUT, 0.05, 40, 180, 97, 93))


def strided():
    f = {}
    for key, cfg, fout, sigma, w, v, H, W in STRIDED:
        text = open(os.path.join(CONFIGS, cfg)).read()
        net = O.RefNet(text, seed=5, fout=fout, sigma=sigma)
        img = O.Rng(61).index_u8(H * W).reshape(H, W)
        lab, pr = net.process(img, w, v)
        f[f"{key}_img"], f[f"{key}_labels"], f[f"{key}_probs"] = img, lab, pr
        f[f"{key}_geom"] = np.array([w, v, H, W], np.int32)
        print(key, "tiles", O.tile_offsets(H, w), O.tile_offsets(W, w),
              "label histogram", np.bincount(lab.ravel(), minlength=2))
    np.savez_compressed(os.path.join(OUT, "strided.npz"), **f)
    print("strided.npz", len(f), "arrays")


# Full-width sk.net process() at the CLI's tile (w=128, v=101) on a non-square image whose
# right and bottom tiles snap inward. The GPU retiles it internally (one 230-px tile column)
# and runs ip1 (K = 19200) on the int8 certify-or-recompute path, so this pins that path on
# the full net against the reference's own process(). Weights: init_weights(sk, 1), the bench's.
SKPROC = (128, 101, 260, 230)


def skproc():
    w, v, H, W = SKPROC
    text = open(os.path.join(CONFIGS, "sk.net")).read()
    net = O.RefNet(text, seed=1)
    img = O.Rng(55).index_u8(H * W).reshape(H, W)
    lab, pr = net.process(img, w, v)
    np.savez_compressed(os.path.join(OUT, "skproc.npz"), img=img, labels=lab, probs=pr,
                        geom=np.array(SKPROC, np.int32),
                        labels_sha=np.frombuffer(sha(lab).encode(), np.uint8),
                        probs_sha=np.frombuffer(sha(pr).encode(), np.uint8))
    print("skproc.npz written; labels", np.bincount(lab.ravel(), minlength=2))


# MALIS instances (malis.hpp): per case an h x w foreground plane and predicted probabilities
# (numpy default_rng(seed), inputs stored), through the reference's affinity_forward,
# connected_components, malis_gradient, affinity_backward and malis_softmax_loss, in float and
# double. Shapes cover the degenerate extents (1x1, 1xn, nx1) and multi-component patches.
MALIS_CASES = [(1, 1), (1, 7), (9, 1), (2, 2), (5, 5), (6, 9), (16, 16), (31, 24), (48, 48)]


def malis():
    f = {}
    for ci, (h, w) in enumerate(MALIS_CASES):
        rng = np.random.default_rng(1000 + ci)
        fg = (rng.random((h, w)) < 0.55).astype(np.uint8)
        probs = rng.uniform(0.01, 0.99, (h, w))
        scores = rng.uniform(-1.0, 1.0, (2, h, w))
        diff0 = rng.uniform(-1.0, 1.0, (2, h, w))
        dgx, dgy = rng.uniform(-1.0, 1.0, (h, w)), rng.uniform(-1.0, 1.0, (h, w))
        key = f"c{ci}"
        f[f"{key}_fg"] = fg
        f[f"{key}_comp"] = O.malis_components(fg, "ref")
        for dt in (np.float32, np.float64):
            t = "f32" if dt == np.float32 else "f64"
            pr = probs.astype(dt)
            pax, pay, pmx, pmy = O.malis_affinity_forward(pr, "ref")
            tax, tay, _, _ = O.malis_affinity_forward(fg.astype(dt), "ref")
            g = O.malis_gradient(pax, pay, tax, tay, f[f"{key}_comp"], "ref")
            f[f"{key}_{t}_probs"] = pr
            for n, a in (("pax", pax), ("pay", pay), ("pmx", pmx), ("pmy", pmy), ("tax", tax), ("tay", tay)):
                f[f"{key}_{t}_{n}"] = a
            for n, a in g.items():
                f[f"{key}_{t}_{n}"] = a
            dp, dn = O.malis_affinity_backward(dgx.astype(dt), dgy.astype(dt), pmx, pmy, "ref")
            f[f"{key}_{t}_dgx"], f[f"{key}_{t}_dgy"] = dgx.astype(dt), dgy.astype(dt)
            f[f"{key}_{t}_dpos"], f[f"{key}_{t}_dneg"] = dp, dn
            sc, d0 = scores.astype(dt), diff0.astype(dt)
            loss, d = O.malis_softmax_loss(sc, fg, d0, "ref")
            f[f"{key}_{t}_scores"], f[f"{key}_{t}_diff0"] = sc, d0
            f[f"{key}_{t}_loss"], f[f"{key}_{t}_diff"] = np.array([loss]), d
    np.savez_compressed(os.path.join(OUT, "malis.npz"), cases=np.array(MALIS_CASES, np.int32), **f)
    print("malis.npz written:", len(MALIS_CASES), "cases")


if __name__ == "__main__":
    for arg in sys.argv[1:] or ["small"]:
        if arg == "cli":
            cli()
        elif arg == "strided":
            strided()
        elif arg == "skproc":
            skproc()
        elif arg == "malis":
            malis()
        elif arg == "small":
            configs()
            small()
            nets()
        else:
            full(arg)
