"""Rng (rng.hpp:12-54) over libgraft_cuda's host-only generator: std::mt19937_64 with the
reference's hand-rolled uniform / gaussian (Box-Muller with a cached spare) transforms, so
streams are identical to the reference's for the same seed. Bulk fills run in C++."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


class Rng:
    def __init__(self, seed: int):
        h = C.c_void_p()
        _lib.check(_lib.lib().graft_rng_create(C.c_uint64(seed & (2**64 - 1)), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if self.h:
                _lib.lib().graft_rng_destroy(self.h)
        except Exception:
            pass

    def gaussian_array(self, n: int, mean: float = 0.0, sigma: float = 1.0) -> np.ndarray:
        """n draws of float(mean + sigma * gaussian()), in stream order."""
        out = np.empty(n, np.float32)
        _lib.check(_lib.lib().graft_rng_fill_gaussian_f32(self.h, _lib.ptr(out), n, mean, sigma))
        return out

    def uniform_array(self, n: int, lo: float, hi: float, dtype=np.float32) -> np.ndarray:
        """n draws of S(lo + (hi - lo) * uniform()), in stream order."""
        if np.dtype(dtype) == np.float64:
            out = np.empty(n, np.float64)
            _lib.check(_lib.lib().graft_rng_fill_uniform_f64(self.h, _lib.ptr(out), n, lo, hi))
        else:
            out = np.empty(n, np.float32)
            _lib.check(_lib.lib().graft_rng_fill_uniform_f32(self.h, _lib.ptr(out), n, lo, hi))
        return out

    def index_array_u8(self, n: int, m: int) -> np.ndarray:
        """n draws of uint8(uniform_index(m))."""
        out = np.empty(n, np.uint8)
        _lib.check(_lib.lib().graft_rng_fill_index_u8(self.h, _lib.ptr(out), n, m))
        return out
