"""Training step on the B200 against the reference itself (oracle/_ref:
the unmodified reference headers): NetRunner::backward (netgraph.hpp:88-98) through every
backward layer function (layers.hpp:68-95, 134-139, 149-155, 178-190, 214-221, 246-262),
softmax_loss (layers.hpp:269-307) and sgd_step (pipeline.hpp:483-500), two SGD iterations
per net. Blob diffs, parameter diffs, momenta and updated weights must be bit-identical; the
loss is a libm-log sum (log_cr) and must match to the last bit as well."""
import numpy as np
import pytest

from conftest import assert_bitwise, config_text

import paper_1509_03371_b200 as g
from oracle import oracle as O

pytestmark = pytest.mark.gpu

if not O.ref_available():
    pytest.skip("oracle/_ref not built", allow_module_level=True)

CHAIN = ("input w=12 f=2\n"
         "layer conv1 conv_sk k=3 fout=4 in=data out=conv1 init=gaussian:0.5\n"
         "layer relu1 relu in=conv1 out=relu1\n"
         "layer pool1 pool_max k=2 s=2 in=relu1 out=pool1\n"
         "layer conv2 conv_sk k=3 fout=3 in=pool1 out=conv2 init=gaussian:0.5\n"
         "layer prob softmax_loss in=conv2 out=prob\n")
UNET = ("input w=16 f=1\n"
        "layer conv1 conv_sk k=3 fout=2 in=data out=conv1 init=gaussian:0.4\n"
        "layer pool1 pool_max k=2 s=2 in=conv1 out=pool1\n"
        "layer conv2 conv_sk k=3 fout=4 in=pool1 out=conv2 init=gaussian:0.4\n"
        "layer up1 upconv in=conv2 out=up1\n"
        "layer merge1 mergecrop in=up1,conv1 out=merge1\n"
        "layer conv3 conv_sk k=3 fout=2 in=merge1 out=conv3 init=gaussian:0.4\n"
        "layer prob softmax_loss in=conv3 out=prob\n")
SK_SMALL_FOUT = {"conv1": 6, "conv2": 8, "conv3": 12, "ip1": 16, "ip2": 8, "ip3": 2}


def sk_small_text():
    spec = g.parse_netspec_or_throw(config_text("sk"))
    lines = []
    for line in config_text("sk").splitlines():
        for name, f in SK_SMALL_FOUT.items():
            if line.startswith(f"layer {name} "):
                import re
                line = re.sub(r"fout=\d+", f"fout={f}", line)
                line = re.sub(r"init=\S+", "init=gaussian:0.1", line)
        lines.append(line)
    del spec
    return "\n".join(lines) + "\n"


def make_pair(text, seed):
    ref = O.RefNet(text, seed=seed)
    spec = g.parse_netspec_or_throw(text)
    states = g.init_weights(spec, seed)
    for i, (w, b) in ref.params().items():  # same init stream -> same parameters
        assert_bitwise(states.layers[i].weights, w, f"init layer {i}")
    return ref, spec, g.NetRunner(spec, states)


def compare_state(ref, spec, runner, what):
    for l in spec.layers:
        assert_bitwise(runner.blob_diff(l.output), ref.blob_diff(l.output), f"{what}: diff of {l.output}")
    for i, l in enumerate(spec.layers):
        if l.kind != g.LayerKind.ConvSK:
            continue
        st = runner.states.layers[i]
        rw, rb = ref.param_state(i, 1)
        assert_bitwise(st.weight_diff, rw, f"{what}: weight_diff {l.name}")
        assert_bitwise(st.bias_diff, rb, f"{what}: bias_diff {l.name}")


def compare_params(ref, spec, runner, what):
    rp = ref.params()
    for i, l in enumerate(spec.layers):
        if l.kind != g.LayerKind.ConvSK:
            continue
        st = runner.states.layers[i]
        assert_bitwise(st.weights, rp[i][0], f"{what}: weights {l.name}")
        assert_bitwise(st.bias, rp[i][1], f"{what}: bias {l.name}")
        mw, mb = ref.param_state(i, 2)
        assert_bitwise(st.weight_mom, mw, f"{what}: weight_mom {l.name}")
        assert_bitwise(st.bias_mom, mb, f"{what}: bias_mom {l.name}")
        dw, db = ref.param_state(i, 1)
        assert_bitwise(st.weight_diff, dw, f"{what}: zeroed weight_diff {l.name}")


@pytest.mark.parametrize("name,text,w0,seed", [
    ("chain", CHAIN, 12, 7),
    ("unet", UNET, 16, 9),
    ("sk_small", None, 110, 3),
])
@pytest.mark.parametrize("masked", [False, True])
def test_two_sgd_iterations_bit_identical(name, text, w0, seed, masked):
    text = text or sk_small_text()
    ref, spec, runner = make_pair(text, seed)
    scores = spec.layers[-1].inputs[0]
    rng = O.Rng(1000 + seed)
    cfg = g.SolverConfig(lr=0.05, momentum=0.9, weight_decay=5e-4)
    for it in range(2):
        x = rng.uniform_f32(spec.f0 * w0 * w0).reshape(spec.f0, w0, w0)
        ref.forward(x)
        out = runner.forward(g.Blob.from_array(x)).view()
        assert_bitwise(out, ref.blob(spec.layers[-1].output), f"{name} it{it}: forward")
        h, w = out.shape[1:]
        labels = (rng.index_u8(h * w, out.shape[0]).astype(np.int32)).reshape(h, w)
        mask = (rng.index_u8(h * w, 2) if masked else np.ones(h * w, np.uint8)).reshape(h, w)
        ref.zero_blob_diffs()
        runner.zero_blob_diffs()
        lr_ = ref.softmax_loss(scores, labels, mask if masked else None)
        lg = runner.softmax_loss(scores, labels, mask if masked else None)
        assert np.float64(lg).view(np.uint64) == np.float64(lr_).view(np.uint64), (lg, lr_)
        ref.backward()
        runner.backward()
        compare_state(ref, spec, runner, f"{name} it{it}")
        ref.sgd_step(cfg.lr, cfg.momentum, cfg.weight_decay)
        g.sgd_step(runner, cfg)
        compare_params(ref, spec, runner, f"{name} it{it}")


def test_backward_through_softmax_head_and_accumulation():
    """A diff seeded at the probability blob flows through softmax_backward
    (layers.hpp:246-262); a second backward without zeroing accumulates (diffs += ...)."""
    ref, spec, runner = make_pair(CHAIN, 11)
    x = O.Rng(5).uniform_f32(2 * 12 * 12).reshape(2, 12, 12)
    ref.forward(x)
    runner.forward(g.Blob.from_array(x))
    prob = spec.layers[-1].output
    seed = O.Rng(6).uniform_f32(3 * 3 * 3).reshape(3, 3, 3)
    ref.set_blob_diff(prob, seed)
    runner.set_blob_diff(prob, seed)
    ref.backward()
    runner.backward()
    compare_state(ref, spec, runner, "softmax head")
    ref.backward()
    runner.backward()
    compare_state(ref, spec, runner, "second backward")


def test_backward_errors():
    spec = g.parse_netspec_or_throw(CHAIN)
    runner = g.NetRunner(spec, g.init_weights(spec, 1))
    with pytest.raises(g.SpecError):
        runner.backward()  # no forward yet
    runner.forward(g.Blob.from_array(np.zeros((2, 12, 12), np.float32)))
    with pytest.raises(g.SizeError, match="does not match scores"):
        runner.softmax_loss("conv2", np.zeros((2, 2), np.int32))
    with pytest.raises(g.SpecError, match="outside"):
        runner.softmax_loss("conv2", np.full((3, 3), 3, np.int32))
