"""Graph executor on the B200: NetStates, init_weights and NetRunner, mirroring netgraph.hpp
(/root/reference/proj/include/pixelseg/netgraph.hpp:19-206).

NetRunner owns a device-resident ``graft_net`` (the C++ host driver in csrc/net.cu): the blob
table lives in HBM, conv weights live there as f64 tiles, and ``blob(name)`` reads a blob back
on demand. Weights stay in the caller's NetStates; the runner re-uploads a layer whenever its
host arrays changed since the last upload (compared on every forward).
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List

import numpy as np

from . import _lib
from .blob import Blob, LayerState
from .errors import SizeError, SpecError
from .netspec import InitKind, LayerKind, NetSpec, compute_channels
from .rng import Rng


class NetStates:
    """NetStates<S> (netgraph.hpp:19-22): one LayerState per NetSpec layer."""

    def __init__(self, n: int = 0, dtype=np.float32):
        self.layers: List[LayerState] = [LayerState(dtype) for _ in range(n)]


def init_weights(spec: NetSpec, seed: int, dtype=np.float32) -> NetStates:
    """init_weights<S> (netgraph.hpp:27-46): one seeded mt19937_64 stream, layer by layer;
    sigma = init_sigma (gaussian), sqrt(2/fan_in) (he), 0.01 (unspecified); biases zero.
    Host-only; bit-identical to the reference's parameters."""
    if np.dtype(dtype) != np.float32:
        raise TypeError("init_weights: the B200 path runs S=float nets")
    states = NetStates(len(spec.layers), dtype)
    rng = Rng(seed)
    channels = compute_channels(spec)
    for i, l in enumerate(spec.layers):
        if not l.has_weights():
            continue
        fin = sum(channels[b] for b in l.inputs)
        fan_in = fin * l.k * l.k
        states.layers[i].init_conv(l.f_out, fan_in)
        sigma = l.init_sigma
        if l.init == InitKind.He:
            sigma = float(np.sqrt(2.0 / float(fan_in)))
        if l.init == InitKind.None_:
            sigma = 0.01
        states.layers[i].weights = rng.gaussian_array(l.f_out * fan_in, 0.0, sigma)
    return states


def net_descs(spec: NetSpec):
    """LayerSpec list -> graft_layer_desc array (plus the byte strings it points to)."""
    keep = []

    def b(s):
        if s is None:
            return None
        v = s.encode()
        keep.append(v)
        return v

    arr = (_lib.LayerDesc * len(spec.layers))()
    for i, l in enumerate(spec.layers):
        d = arr[i]
        d.name = b(l.name)
        d.kind = int(l.kind)
        d.k, d.s, d.d, d.p, d.f_out = l.k, l.s, l.d, l.p, l.f_out
        d.in0 = b(l.inputs[0]) if len(l.inputs) > 0 else None
        d.in1 = b(l.inputs[1]) if len(l.inputs) > 1 else None
        d.out = b(l.output)
        d.init = {InitKind.None_: _lib.INIT_NONE, InitKind.Gaussian: _lib.INIT_GAUSSIAN,
                  InitKind.He: _lib.INIT_HE}[l.init]
        d.init_sigma = l.init_sigma
    return arr, keep


class DeviceNet:
    """RAII owner of one graft_net handle on the current device."""

    def __init__(self, spec: NetSpec):
        if not spec.layers or spec.layers[0].kind != LayerKind.Data:
            raise SpecError("missing input directive")
        arr, keep = net_descs(spec)
        h = C.c_void_p()
        _lib.check(_lib.lib().graft_net_create(spec.f0, len(spec.layers), arr, C.byref(h)))
        self.h = h
        self._keep = keep
        self._uploaded: Dict[int, tuple] = {}

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            _lib.lib().graft_net_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, opt: int, value: int) -> None:
        _lib.check(_lib.lib().graft_net_set_option(self.h, opt, int(value)))

    def get_option(self, opt: int) -> int:
        v = _lib.C.c_longlong(0)
        _lib.check(_lib.lib().graft_net_get_option(self.h, opt, _lib.C.byref(v)))
        return int(v.value)

    def sync_params(self, spec: NetSpec, states: NetStates) -> None:
        """Uploads every conv layer whose parameters were assigned since its last upload
        (LayerState.generation; O(layers), no weight is read unless it changed)."""
        for i, l in enumerate(spec.layers):
            if l.kind != LayerKind.ConvSK:
                continue
            st = states.layers[i]
            if self._uploaded.get(i) == (id(st), st.generation):
                continue
            w = np.ascontiguousarray(st.weights, np.float32)
            bb = np.ascontiguousarray(st.bias, np.float32)
            _lib.check(_lib.lib().graft_net_set_params_f32(self.h, i, _lib.ptr(w), w.size,
                                                           _lib.ptr(bb), bb.size))
            self.mark_synced(i, st)

    def mark_synced(self, i: int, st) -> None:
        """Records st's current parameters as the device's (after an upload or a device-side
        update) and freezes the host arrays."""
        st.freeze_params()
        self._uploaded[i] = (id(st), st.generation)


class NetRunner:
    """NetRunner<float> (netgraph.hpp:49-206), forward path on the B200."""

    def __init__(self, spec: NetSpec, states: NetStates):
        if len(states.layers) != len(spec.layers):
            raise SpecError(f"net runner: state table has {len(states.layers)} entries for "
                            f"{len(spec.layers)} layers")
        self.spec = spec
        self.states = states
        self.net = DeviceNet(spec)
        # the reference's forward always records what backward needs (pool argmax)
        self.net.set_option(_lib.OPT_TRAINING, 1)
        self._layer_seconds: List[float] = [0.0] * len(spec.layers)
        self._last = None

    def forward(self, input: Blob, timed: bool = False) -> Blob:
        """NetRunner::forward (netgraph.hpp:64-84); returns the last layer's blob (a host copy)."""
        if input.channels != self.spec.f0:
            raise SizeError(f"forward: input has {input.channels} channels, net expects {self.spec.f0}")
        if np.dtype(input.dtype) != np.float32:
            raise TypeError("NetRunner on the B200 runs S=float nets")
        self.net.sync_params(self.spec, self.states)
        self.net.set_option(_lib.OPT_TIMED, 1 if timed else 0)
        x = np.ascontiguousarray(input.data, np.float32)
        oc, oh, ow = C.c_int(), C.c_int(), C.c_int()
        _lib.check(_lib.lib().graft_net_forward_f32(self.net.h, _lib.ptr(x), input.channels,
                                                    input.height, input.width, _lib.MEM_HOST,
                                                    C.byref(oc), C.byref(oh), C.byref(ow)))
        if timed:
            ms = (C.c_double * len(self.spec.layers))()
            _lib.check(_lib.lib().graft_net_layer_ms(self.net.h, ms, len(self.spec.layers)))
            self._layer_seconds = [v * 1e-3 for v in ms]
        else:
            self._layer_seconds = [0.0] * len(self.spec.layers)
        self._last = self.blob(self.spec.layers[-1].output)
        return self._last

    def has_blob(self, name: str) -> bool:
        c = C.c_int()
        return _lib.lib().graft_net_blob_shape(self.net.h, name.encode(), C.byref(c), None, None) == 0

    def blob(self, name: str) -> Blob:
        """NetRunner::blob (netgraph.hpp:108-112): SpecError if absent."""
        c, h, w = C.c_int(), C.c_int(), C.c_int()
        _lib.check(_lib.lib().graft_net_blob_shape(self.net.h, name.encode(), C.byref(c),
                                                   C.byref(h), C.byref(w)))
        b = Blob(c.value, h.value, w.value, np.float32)
        if b.size():
            _lib.check(_lib.lib().graft_net_blob_f32(self.net.h, name.encode(), _lib.ptr(b.data),
                                                     _lib.MEM_HOST))
        return b

    def layer_seconds(self) -> List[float]:
        return list(self._layer_seconds)

    # ---- training step: backward, softmax_loss, sgd_step ------------
    def zero_blob_diffs(self) -> None:
        """NetRunner::zero_blob_diffs (netgraph.hpp:100-105)."""
        _lib.check(_lib.lib().graft_net_zero_blob_diffs(self.net.h))

    def blob_diff(self, name: str) -> np.ndarray:
        """Blob::diff of a blob as a (C, H, W) float32 array (zeros when cleared)."""
        b = self.blob(name)
        out = np.zeros((b.channels, b.height, b.width), np.float32)
        if out.size:
            _lib.check(_lib.lib().graft_net_blob_diff_f32(self.net.h, name.encode(), _lib.ptr(out),
                                                          _lib.MEM_HOST))
        return out

    def set_blob_diff(self, name: str, diff: np.ndarray) -> None:
        """blob_mut(name).diff = diff: the caller's seeding before backward (netgraph.hpp:85-87)."""
        d = np.ascontiguousarray(diff, np.float32)
        _lib.check(_lib.lib().graft_net_set_blob_diff_f32(self.net.h, name.encode(), _lib.ptr(d),
                                                          _lib.MEM_HOST))

    def _push_param_state(self) -> None:
        for i, l in enumerate(self.spec.layers):
            if l.kind != LayerKind.ConvSK:
                continue
            st = self.states.layers[i]
            for which, (w, b) in ((_lib.PARAM_DIFF, (st.weight_diff, st.bias_diff)),
                                  (_lib.PARAM_MOMENTUM, (st.weight_mom, st.bias_mom))):
                w = np.ascontiguousarray(w, np.float32)
                b = np.ascontiguousarray(b, np.float32)
                if w.size == st.weights.size and b.size == st.bias.size:
                    _lib.check(_lib.lib().graft_net_set_param_state_f32(
                        self.net.h, i, which, _lib.ptr(w), _lib.ptr(b)))

    def _pull_param_state(self, weights: bool) -> None:
        for i, l in enumerate(self.spec.layers):
            if l.kind != LayerKind.ConvSK:
                continue
            st = self.states.layers[i]
            for which, names in ((_lib.PARAM_DIFF, ("weight_diff", "bias_diff")),
                                 (_lib.PARAM_MOMENTUM, ("weight_mom", "bias_mom"))):
                w = np.empty(st.weights.size, np.float32)
                b = np.empty(st.bias.size, np.float32)
                _lib.check(_lib.lib().graft_net_get_param_state_f32(self.net.h, i, which,
                                                                    _lib.ptr(w), _lib.ptr(b)))
                setattr(st, names[0], w)
                setattr(st, names[1], b)
            if weights:
                w = np.empty(st.weights.size, np.float32)
                b = np.empty(st.bias.size, np.float32)
                _lib.check(_lib.lib().graft_net_get_params_f32(self.net.h, i, _lib.ptr(w),
                                                               _lib.ptr(b)))
                st.weights, st.bias = w, b
                self.net.mark_synced(i, st)

    def backward(self) -> None:
        """NetRunner::backward (netgraph.hpp:88-98) on the device: reverse sweep over the blob
        diffs seeded since the last forward; parameter diffs accumulate into the NetStates."""
        self._push_param_state()
        _lib.check(_lib.lib().graft_net_backward(self.net.h))
        self._pull_param_state(weights=False)

    def softmax_loss(self, scores: str, labels: np.ndarray, mask=None) -> float:
        """softmax_loss (layers.hpp:269-307) on this runner's blob `scores` (diff += gradient)."""
        lab = np.ascontiguousarray(labels, np.int32)
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        loss = C.c_double()
        _lib.check(_lib.lib().graft_net_softmax_loss_f32(self.net.h, scores.encode(), _lib.ptr(lab),
                                                         _lib.ptr(m), lab.shape[0], lab.shape[1],
                                                         C.byref(loss)))
        return loss.value

    def malis_softmax_loss(self, scores: str, fg: np.ndarray) -> float:
        """malis_softmax_loss (malis.hpp:311-346) on this runner's blob `scores`: the training
        step's MALIS loss (pipeline.hpp:599-606); diff += gradient, on the device."""
        from .malis import malis_softmax_loss_device

        return malis_softmax_loss_device(self.net.h, scores, fg)


class SolverConfig:
    """The SGD fields of SolverConfig (pipeline.hpp:324-339) that sgd_step reads."""

    def __init__(self, lr: float = 0.01, momentum: float = 0.9, weight_decay: float = 0.0):
        self.lr = lr
        self.momentum = momentum
        self.weight_decay = weight_decay


def sgd_step(runner: NetRunner, cfg: SolverConfig) -> None:
    """sgd_step<float> (pipeline.hpp:483-500) on the device copy of runner.states:
    v = mom*v - lr*(diff + wd*w); w += v; diffs zeroed. The NetStates arrays are updated."""
    runner._push_param_state()
    _lib.check(_lib.lib().graft_net_sgd_step(runner.net.h, cfg.lr, cfg.momentum, cfg.weight_decay))
    runner._pull_param_state(weights=True)
