"""Layer-level API on the B200: the forward functions of layers.hpp and the primitives of
tensor.hpp (/root/reference/proj/include/pixelseg/), same names, argument meaning, output
resizing and error behaviour. Each call runs the sm_100a kernel through the C ABI
(include/graft_cuda.h) on host numpy buffers; results are bit-identical to the reference.
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .blob import Blob, ColumnBuffer, ConvGeometry, LayerState
from .errors import SizeError

_H = _lib.MEM_HOST


def _sfx(dtype) -> str:
    dt = np.dtype(dtype)
    if dt == np.float32:
        return "f32"
    if dt == np.float64:
        return "f64"
    raise TypeError(f"unsupported scalar type {dt} (the reference instantiates float and double)")


def _c(a: np.ndarray, dtype) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


def conv_sk_forward(in_: Blob, state: LayerState, f_out: int, g: ConvGeometry,
                    colbuf: ColumnBuffer, out: Blob) -> None:
    """conv_sk_forward (layers.hpp:43-64). ``colbuf`` is accepted for signature parity; the B200
    kernel is an implicit GEMM and never materialises the column matrix."""
    fan_in = in_.channels * g.k * g.k
    if state.weights.size != f_out * fan_in:
        raise SizeError(f"conv: weight count {state.weights.size} != f_out*f_in*k*k = {f_out * fan_in}")
    if state.bias.size != f_out:
        raise SizeError("conv: bias count mismatch")
    if in_.height != g.in_h or in_.width != g.in_w:
        raise SizeError(f"im2col_sk: blob is {in_.height}x{in_.width} but geometry expects "
                        f"{g.in_h}x{g.in_w}")
    dt = in_.dtype
    x, w, b = _c(in_.data, dt), _c(state.weights, dt), _c(state.bias, dt)
    out.dtype = dt
    out.resize(f_out, g.out_h, g.out_w)
    fn = getattr(_lib.lib(), f"graft_conv_sk_forward_{_sfx(dt)}")
    _lib.check(fn(_lib.ptr(x), in_.channels, in_.height, in_.width, _lib.ptr(w), w.size,
                  _lib.ptr(b), b.size, f_out, g.k, g.d, g.s, g.p, _lib.ptr(out.data), _H))


def maxpool_sk_forward(in_: Blob, state: LayerState, g: ConvGeometry, out: Blob) -> None:
    """maxpool_sk_forward (layers.hpp:102-132); fills state.argmax (uint64 linear indices)."""
    dt = in_.dtype
    out.dtype = dt
    out.resize(in_.channels, g.out_h, g.out_w)
    state.argmax = np.zeros(out.size(), np.uint64)
    x = _c(in_.data, dt)
    fn = getattr(_lib.lib(), f"graft_maxpool_sk_forward_{_sfx(dt)}")
    _lib.check(fn(_lib.ptr(x), in_.channels, in_.height, in_.width, g.k, g.d, g.s, g.p,
                  _lib.ptr(out.data), _lib.ptr(state.argmax), _H))


def relu_forward(in_: Blob, out: Blob) -> None:
    """relu_forward (layers.hpp:143-147)."""
    dt = in_.dtype
    out.dtype = dt
    out.resize(in_.channels, in_.height, in_.width)
    x = _c(in_.data, dt)
    fn = getattr(_lib.lib(), f"graft_relu_forward_{_sfx(dt)}")
    _lib.check(fn(_lib.ptr(x), x.size, _lib.ptr(out.data), _H))


def upconv_forward(in_: Blob, out: Blob) -> None:
    """upconv_forward (layers.hpp:162-176): nearest-neighbour 2x."""
    dt = in_.dtype
    out.dtype = dt
    out.resize(in_.channels, in_.height * 2, in_.width * 2)
    x = _c(in_.data, dt)
    fn = getattr(_lib.lib(), f"graft_upconv_forward_{_sfx(dt)}")
    _lib.check(fn(_lib.ptr(x), in_.channels, in_.height, in_.width, _lib.ptr(out.data), _H))


def mergecrop_forward(a: Blob, b: Blob, out: Blob) -> None:
    """mergecrop_forward (layers.hpp:196-212): A's channels then B center-cropped."""
    if b.height < a.height or b.width < a.width:
        raise SizeError(f"mergecrop: second input {b.height}x{b.width} smaller than first "
                        f"{a.height}x{a.width}")
    dt = a.dtype
    out.dtype = dt
    out.resize(a.channels + b.channels, a.height, a.width)
    xa, xb = _c(a.data, dt), _c(b.data, dt)
    fn = getattr(_lib.lib(), f"graft_mergecrop_forward_{_sfx(dt)}")
    _lib.check(fn(_lib.ptr(xa), a.channels, a.height, a.width, _lib.ptr(xb), b.channels,
                  b.height, b.width, _lib.ptr(out.data), _H))


def softmax_forward(in_: Blob, out: Blob) -> None:
    """softmax_forward (layers.hpp:227-244): per-pixel channel softmax, fp64 exp/sum."""
    dt = in_.dtype
    out.dtype = dt
    out.resize(in_.channels, in_.height, in_.width)
    x = _c(in_.data, dt)
    fn = getattr(_lib.lib(), f"graft_softmax_forward_{_sfx(dt)}")
    _lib.check(fn(_lib.ptr(x), in_.channels, in_.height, in_.width, _lib.ptr(out.data), _H))


def im2col_sk(in_: Blob, g: ConvGeometry, col: ColumnBuffer) -> None:
    """im2col_sk (tensor.hpp:80-110)."""
    if in_.height != g.in_h or in_.width != g.in_w:
        raise SizeError(f"im2col_sk: blob is {in_.height}x{in_.width} but geometry expects "
                        f"{g.in_h}x{g.in_w}")
    dt = in_.dtype
    col.dtype = dt
    rows, cols = in_.channels * g.k * g.k, g.out_h * g.out_w
    col.rows, col.cols = rows, cols
    if col.data.size < rows * cols or col.data.dtype != dt:
        col.data = np.zeros(rows * cols, dt)
    x = _c(in_.data, dt)
    fn = getattr(_lib.lib(), f"graft_im2col_sk_{_sfx(dt)}")
    _lib.check(fn(_lib.ptr(x), in_.channels, in_.height, in_.width, g.k, g.d, g.s, g.p,
                  _lib.ptr(col.data), _H))


def gemm(transpose_a: bool, transpose_b: bool, m: int, n: int, k: int, alpha, a: np.ndarray,
         b: np.ndarray, beta, c: np.ndarray) -> None:
    """gemm (tensor.hpp:151-169): C = S(alpha*sum_kk A*B [+ beta*C]) with an fp64 accumulator
    in ascending kk. ``c`` is updated in place (a contiguous numpy array of m*n)."""
    dt = c.dtype
    if not c.flags.c_contiguous:
        raise ValueError("gemm: c must be contiguous")
    aa, bb = _c(a, dt), _c(b, dt)
    fn = getattr(_lib.lib(), f"graft_gemm_{_sfx(dt)}")
    _lib.check(fn(int(bool(transpose_a)), int(bool(transpose_b)), m, n, k, alpha, _lib.ptr(aa),
                  _lib.ptr(bb), beta, _lib.ptr(c), _H))


def gemm_flops(m: int, n: int, k: int) -> int:  # tensor.hpp:173-175
    return m * n * (2 * k - 1)
