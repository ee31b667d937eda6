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

    def sync_params(self, spec: NetSpec, states: NetStates) -> None:
        """Uploads every conv layer whose host weights/bias differ from the last upload."""
        for i, l in enumerate(spec.layers):
            if l.kind != LayerKind.ConvSK:
                continue
            st = states.layers[i]
            w = np.ascontiguousarray(st.weights, np.float32)
            bb = np.ascontiguousarray(st.bias, np.float32)
            prev = self._uploaded.get(i)
            if prev is not None and prev[0].shape == w.shape and prev[1].shape == bb.shape \
                    and np.array_equal(prev[0], w) and np.array_equal(prev[1], bb):
                continue
            _lib.check(_lib.lib().graft_net_set_params_f32(self.h, i, _lib.ptr(w), w.size,
                                                           _lib.ptr(bb), bb.size))
            self._uploaded[i] = (w.copy(), bb.copy())


class NetRunner:
    """NetRunner<float> (netgraph.hpp:49-206), forward path on the B200."""

    def __init__(self, spec: NetSpec, states: NetStates):
        if len(states.layers) != len(spec.layers):
            raise SpecError(f"net runner: state table has {len(states.layers)} entries for "
                            f"{len(spec.layers)} layers")
        self.spec = spec
        self.states = states
        self.net = DeviceNet(spec)
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
