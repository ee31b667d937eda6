"""Tiled whole-image inference on the B200: process(), mirror_pad(), normalize_image(),
mirroring pipeline.hpp (/root/reference/proj/include/pixelseg/pipeline.hpp:36-93, 618-698).

``process`` validates exactly like the reference, then hands the whole tile loop to the C++
driver (graft_process): tiles are batched on the device, the tile input is built from the raw
u8 image (mirror pad + normalize fused), and softmax + argmax + stitch are one kernel. Any tile
size gives bit-identical planes (the reference's own guarantee, tests/test_pipeline.cpp:535-588).
"""
from __future__ import annotations

from typing import List, Optional

import numpy as np

from . import _lib
from .blob import Plane
from .errors import SizeError, SpecError
from .netgraph import DeviceNet, NetStates
from .netspec import NetSpec, compute_channels, output_extent


def mirror_pad(img: Plane, v: int) -> Plane:
    """mirror_pad<uint8_t> (pipeline.hpp:36-58), run on the device."""
    if v < 0:
        raise SizeError("mirror_pad: negative padding")
    if v == 0:
        return Plane.from_array(img.view())
    src = np.ascontiguousarray(img.pix, np.uint8)
    out = Plane(img.height + v, img.width + v)
    _lib.check(_lib.lib().graft_mirror_pad_u8(_lib.ptr(src), img.height, img.width, v,
                                              _lib.ptr(out.pix), _lib.MEM_HOST))
    return out


def normalize_image(img: Plane) -> Plane:
    """normalize_image<float> (pipeline.hpp:86-93): float(x/127.5 - 1.0), on the device."""
    src = np.ascontiguousarray(img.pix, np.uint8)
    out = Plane(img.height, img.width, 0, np.float32)
    _lib.check(_lib.lib().graft_normalize_image_f32(_lib.ptr(src), src.size, _lib.ptr(out.pix),
                                                    _lib.MEM_HOST))
    return out


class ProcessResult:
    """ProcessResult<S> (pipeline.hpp:620-624)."""

    def __init__(self, labels: Plane, probs: List[Plane]):
        self.labels = labels
        self.probs = probs


def validate_process(spec: NetSpec, H: int, W: int, w: int, v: int) -> None:
    """The checks of process() (pipeline.hpp:633-653) in the reference's order."""
    if spec.loss_head() is None:
        raise SpecError("process: net has no probability head as its last layer")
    try:
        out = output_extent(spec, w + v)
    except SpecError as e:  # Error in the reference; SizeError is a SpecError here
        raise SpecError(f"process: tile + context is not a valid input size: {e}") from None
    if out != w:
        raise SpecError(f"process: input {w + v} produces output {out}, not the tile size {w}")
    if H < w or W < w:
        raise SizeError(f"process: image {H}x{W} is smaller than one {w}-tile")


class Processor:
    """A device-resident net for repeated process() calls (one upload of the weights)."""

    def __init__(self, spec: NetSpec, states: NetStates, tile_batch: int = 0,
                 retile: Optional[int] = None, tensor_cores: Optional[str] = None):
        """retile: largest internal tile process() may use (default 1024; 0 = exactly the
        caller's w). Every tiling gives bit-identical planes.

        tensor_cores: None (default) = the exact fp64 path, bit-identical to the reference;
        "bf16" / "tf32" / "bf16x3" (split bf16, ~fp32 operands) = TOLERANCE MODE: eligible convs run on the tcgen05 tensor cores and the
        planes are only within the tolerance DESIGN.md states (labels may differ on near-ties)."""
        self.spec = spec
        self.states = states
        self.net = DeviceNet(spec)
        self.net.sync_params(spec, states)
        if tile_batch:
            self.net.set_option(_lib.OPT_TILE_BATCH, tile_batch)
        if retile is not None:
            self.net.set_option(_lib.OPT_RETILE, retile)
        if tensor_cores is not None:
            kinds = {"bf16": _lib.TC_BF16, "tf32": _lib.TC_TF32, "bf16x3": _lib.TC_BF16X3}
            if tensor_cores not in kinds:
                raise ValueError(f"tensor_cores must be None, 'bf16', 'tf32' or 'bf16x3', "
                                 f"not {tensor_cores!r}")
            self.net.set_option(_lib.OPT_TC_KIND, kinds[tensor_cores])
        self.n_classes = compute_channels(spec)[spec.layers[-1].output]

    def run(self, image: np.ndarray, w: int, v: int, labels: Optional[np.ndarray] = None,
            probs: Optional[np.ndarray] = None, rows: Optional[tuple] = None, mem: int = 0):
        """Raw entry: image (H, W) uint8 -> labels (H, W) uint8, probs (C, H, W) float32.
        With mem=MEM_DEVICE the three arguments are device pointers / tensors."""
        if mem == _lib.MEM_HOST:
            image = np.ascontiguousarray(image, np.uint8)
            H, W = image.shape
            if labels is None:
                labels = np.zeros((H, W), np.uint8)
            if probs is None:
                probs = np.zeros((self.n_classes, H, W), np.float32)
        else:
            H, W = image.shape
        self.net.sync_params(self.spec, self.states)
        if rows is None:
            _lib.check(_lib.lib().graft_process(self.net.h, _lib.ptr(image), H, W, w, v,
                                                _lib.ptr(labels), _lib.ptr(probs), mem))
        else:
            _lib.check(_lib.lib().graft_process_band(self.net.h, _lib.ptr(image), H, W, w, v,
                                                     rows[0], rows[1], _lib.ptr(labels),
                                                     _lib.ptr(probs), mem))
        return labels, probs


    def run_batch(self, images, w: int, v: int, labels=None, probs=None, mem: int = 0):
        """process() of N same-size images (N, H, W) in shared launches -> labels (N, H, W) u8,
        probs (N, C, H, W) f32, bit-identical to N separate run() calls."""
        if mem == _lib.MEM_HOST:
            images = np.ascontiguousarray(images, np.uint8)
            N, H, W = images.shape
            if labels is None:
                labels = np.zeros((N, H, W), np.uint8)
            if probs is None:
                probs = np.zeros((N, self.n_classes, H, W), np.float32)
        else:
            N, H, W = images.shape
        self.net.sync_params(self.spec, self.states)
        _lib.check(_lib.lib().graft_process_batch(self.net.h, _lib.ptr(images), N, H, W, w, v,
                                                  _lib.ptr(labels), _lib.ptr(probs), mem))
        return labels, probs

    def last_tile(self) -> int:
        """Internal tile size the last run() used."""
        import ctypes as C
        v = C.c_longlong()
        _lib.check(_lib.lib().graft_net_get_option(self.net.h, _lib.OPT_LAST_TILE, C.byref(v)))
        return v.value


def process(spec: NetSpec, states: NetStates, image: Plane, w: int, v: int) -> ProcessResult:
    """process<float> (pipeline.hpp:630-698) on the B200."""
    validate_process(spec, image.height, image.width, w, v)
    proc = Processor(spec, states)
    img = np.ascontiguousarray(image.pix, np.uint8).reshape(image.height, image.width)
    labels, probs = proc.run(img, w, v)
    lab = Plane.from_array(labels)
    pl = [Plane.from_array(probs[c]) for c in range(probs.shape[0])]
    return ProcessResult(lab, pl)


def tile_rows(H: int, w: int) -> int:
    """Number of tile rows process() visits (pipeline.hpp:662-672)."""
    import ctypes as C
    n = C.c_int()
    _lib.check(_lib.lib().graft_tile_rows(H, w, C.byref(n)))
    return n.value


def band_rows(H: int, w: int, r0: int, r1: int) -> tuple:
    """Output rows [y0, y1) owned by tile rows [r0, r1) (disjoint across a partition)."""
    import ctypes as C
    y0, y1 = C.c_int(), C.c_int()
    _lib.check(_lib.lib().graft_band_rows(H, w, r0, r1, C.byref(y0), C.byref(y1)))
    return y0.value, y1.value
