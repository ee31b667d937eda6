"""Host containers mirroring blob.hpp / tensor.hpp / layers.hpp (reference paths under
/root/reference/proj/include/pixelseg/): ``Blob`` (C x H x W, channel slowest), ``Plane``,
``ConvGeometry``, ``ColumnBuffer`` and ``LayerState``. numpy-backed; the layout is identical
to the reference's ``std::vector`` so buffers pass straight to the C ABI.
"""
from __future__ import annotations

import itertools
from typing import Optional

import numpy as np

from .errors import SizeError
from .netspec import out_extent


class Blob:
    """Blob<S> (blob.hpp:13-52): data and diff, C x H x W row-major, channel slowest."""

    def __init__(self, f: int = 0, h: int = 0, w: int = 0, dtype=np.float32):
        self.dtype = np.dtype(dtype)
        self.channels = 0
        self.height = 0
        self.width = 0
        self.data = np.zeros(0, self.dtype)
        self.diff = np.zeros(0, self.dtype)
        if f or h or w:
            self.resize(f, h, w)

    def resize(self, f: int, h: int, w: int) -> None:
        if f < 0 or h < 0 or w < 0:
            raise SizeError("Blob: negative dimension")
        self.channels, self.height, self.width = f, h, w
        self.data = np.zeros(f * h * w, self.dtype)
        self.diff = np.zeros(0, self.dtype)

    def ensure_diff(self) -> None:
        """Blob::ensure_diff (blob.hpp:43-45): a diff of the wrong size becomes zeros."""
        if self.diff.size != self.size():
            self.diff = np.zeros(self.size(), self.dtype)

    def zero_diff(self) -> None:
        self.diff = np.zeros(self.size(), self.dtype)

    def plane(self) -> int:
        return self.height * self.width

    def size(self) -> int:
        return self.channels * self.plane()

    def index(self, c: int, y: int, x: int) -> int:
        return (c * self.height + y) * self.width + x

    def view(self) -> np.ndarray:
        return self.data.reshape(self.channels, self.height, self.width)

    def at(self, c: int, y: int, x: int):
        return self.data[self.index(c, y, x)]

    def copy(self) -> "Blob":
        b = Blob(dtype=self.dtype)
        b.channels, b.height, b.width = self.channels, self.height, self.width
        b.data = self.data.copy()
        b.diff = self.diff.copy()
        return b

    @staticmethod
    def from_array(a: np.ndarray, dtype=None) -> "Blob":
        a = np.asarray(a)
        if dtype is not None:
            a = a.astype(dtype)
        if a.ndim != 3:
            raise SizeError("Blob.from_array: need a C x H x W array")
        b = Blob(dtype=a.dtype)
        b.channels, b.height, b.width = a.shape
        b.data = np.ascontiguousarray(a).reshape(-1).copy()
        return b


class Plane:
    """Plane<T> (blob.hpp:55-66)."""

    def __init__(self, h: int = 0, w: int = 0, fill=0, dtype=np.uint8):
        self.height, self.width = h, w
        self.pix = np.full(h * w, fill, dtype=dtype)

    def size(self) -> int:
        return self.pix.size

    def at(self, y: int, x: int):
        return self.pix[y * self.width + x]

    def view(self) -> np.ndarray:
        return self.pix.reshape(self.height, self.width)

    @staticmethod
    def from_array(a: np.ndarray) -> "Plane":
        a = np.ascontiguousarray(a)
        p = Plane()
        p.height, p.width = a.shape
        p.pix = a.reshape(-1).copy()
        return p


class ConvGeometry:
    """ConvGeometry (tensor.hpp:14-56)."""

    def __init__(self):
        self.k = 1
        self.d = 1
        self.s = 1
        self.p = 0
        self.in_h = 0
        self.in_w = 0
        self.out_h = 0
        self.out_w = 0

    def span(self) -> int:
        return (self.k - 1) * self.d + 1

    out_extent = staticmethod(out_extent)

    @staticmethod
    def from_input(k: int, d: int, s: int, p: int, in_h: int, in_w: int) -> "ConvGeometry":
        g = ConvGeometry()
        g.k, g.d, g.s, g.p, g.in_h, g.in_w = k, d, s, p, in_h, in_w
        g.out_h = out_extent(in_h, k, d, s, p, "height")
        g.out_w = out_extent(in_w, k, d, s, p, "width")
        return g


class ColumnBuffer:
    """ColumnBuffer<S> (tensor.hpp:60-75): rows = C*k*k taps, cols = out_h*out_w; grows only."""

    def __init__(self, dtype=np.float32):
        self.dtype = np.dtype(dtype)
        self.rows = 0
        self.cols = 0
        self.data = np.zeros(0, self.dtype)

    def resize(self, r: int, c: int) -> None:
        self.rows, self.cols = r, c
        if self.data.size < r * c:
            self.data = np.zeros(r * c, self.dtype)

    def at(self, r: int, c: int):
        return self.data[r * self.cols + c]


_GENERATION = itertools.count(1)


class LayerState:
    """LayerState<S> (layers.hpp:19-37).

    `weights` and `bias` carry a generation number that changes whenever either attribute is
    assigned, so a device net re-uploads a layer's parameters only when its generation moved:
    O(layers) per call instead of comparing every weight. Once uploaded, the arrays are marked
    read-only; an in-place write (`st.weights[0] = x`) raises instead of leaving a stale device
    copy. Change parameters by assignment (`st.weights = new_array`)."""

    @property
    def weights(self) -> np.ndarray:
        return self._weights

    @weights.setter
    def weights(self, a) -> None:
        self._weights = a
        self.generation = next(_GENERATION)

    @property
    def bias(self) -> np.ndarray:
        return self._bias

    @bias.setter
    def bias(self, a) -> None:
        self._bias = a
        self.generation = next(_GENERATION)

    def freeze_params(self) -> None:
        """Marks weights and bias read-only (called once they are resident on a device)."""
        for a in (self._weights, self._bias):
            if isinstance(a, np.ndarray):
                a.flags.writeable = False

    def __init__(self, dtype=np.float32):
        self.dtype = np.dtype(dtype)
        self.weights = np.zeros(0, self.dtype)
        self.bias = np.zeros(0, self.dtype)
        self.weight_diff = np.zeros(0, self.dtype)
        self.bias_diff = np.zeros(0, self.dtype)
        self.weight_mom = np.zeros(0, self.dtype)
        self.bias_mom = np.zeros(0, self.dtype)
        self.argmax: Optional[np.ndarray] = np.zeros(0, np.uint64)

    def init_conv(self, f_out: int, fan_in: int) -> None:
        self.weights = np.zeros(f_out * fan_in, self.dtype)
        self.bias = np.zeros(f_out, self.dtype)
        self.weight_diff = np.zeros_like(self.weights)
        self.bias_diff = np.zeros_like(self.bias)
        self.weight_mom = np.zeros_like(self.weights)
        self.bias_mom = np.zeros_like(self.bias)
