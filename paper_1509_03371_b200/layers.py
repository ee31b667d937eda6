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


# ---- backward functions, S = float ------------------------------------
def _f32(dtype):
    if np.dtype(dtype) != np.float32:
        raise TypeError("the B200 backward path runs S=float")


def conv_sk_backward(in_: Blob, state: LayerState, f_out: int, g: ConvGeometry, colbuf: ColumnBuffer,
                     col_grad: ColumnBuffer, out: Blob, propagate_input: bool = True) -> None:
    """conv_sk_backward (layers.hpp:68-95): dW += dOut col^T, db += row sums, in.diff +=
    col2im(W^T dOut) (when propagate_input). Column buffers are accepted for signature parity."""
    _f32(in_.dtype)
    if out.diff.size != out.size():
        raise SizeError("conv backward: output diff missing")
    fan_in = in_.channels * g.k * g.k
    if state.weights.size != f_out * fan_in:
        raise SizeError(f"conv: weight count {state.weights.size} != f_out*f_in*k*k = {f_out * fan_in}")
    if state.weight_diff.size != state.weights.size:
        state.weight_diff = np.zeros(state.weights.size, np.float32)
    if state.bias_diff.size != f_out:
        state.bias_diff = np.zeros(f_out, np.float32)
    if propagate_input:
        in_.ensure_diff()
    dw = _c(state.weight_diff, np.float32)
    db = _c(state.bias_diff, np.float32)
    din = _c(in_.diff, np.float32) if propagate_input else None
    _lib.check(_lib.lib().graft_conv_sk_backward_f32(
        _lib.ptr(_c(in_.data, np.float32)), in_.channels, in_.height, in_.width,
        _lib.ptr(_c(state.weights, np.float32)), f_out, g.k, g.d, g.s, g.p,
        _lib.ptr(_c(out.diff, np.float32)), _lib.ptr(dw), _lib.ptr(db), _lib.ptr(din), _H))
    state.weight_diff, state.bias_diff = dw, db
    if propagate_input:
        in_.diff = din


def col2im_sk(col: ColumnBuffer, g: ConvGeometry, channels: int, out: Blob) -> None:
    """col2im_sk (tensor.hpp:113-145): out = the exact adjoint scatter of col."""
    if col.rows != channels * g.k * g.k or col.cols != g.out_h * g.out_w:
        raise SizeError(f"col2im_sk: column buffer is {col.rows}x{col.cols}, expected "
                        f"{channels * g.k * g.k}x{g.out_h * g.out_w}")
    out.resize(channels, g.in_h, g.in_w)
    data = np.zeros(out.size(), np.float32)
    _lib.check(_lib.lib().graft_col2im_sk_f32(_lib.ptr(_c(col.data[:col.rows * col.cols], np.float32)),
                                              channels, g.in_h, g.in_w, g.k, g.d, g.s, g.p,
                                              _lib.ptr(data), _H))
    out.data = data


def maxpool_sk_backward(in_: Blob, state: LayerState, out: Blob, g: ConvGeometry = None) -> None:
    """maxpool_sk_backward (layers.hpp:134-139): in.diff[argmax[o]] += out.diff[o], o ascending.
    With the forward's geometry `g` the device gathers per pooling window; without it any
    argmax table is replayed in the reference's scatter order."""
    _f32(in_.dtype)
    if state.argmax is None or state.argmax.size != out.size():
        raise SizeError("pool backward: stale argmax cache")
    in_.ensure_diff()
    din = _c(in_.diff, np.float32)
    k, d, s = (g.k, g.d, g.s) if g is not None else (0, 1, 1)
    _lib.check(_lib.lib().graft_maxpool_sk_backward_f32(
        _lib.ptr(_c(state.argmax, np.uint64)), _lib.ptr(_c(out.diff, np.float32)), out.size(),
        in_.channels, in_.height, in_.width, k, d, s, _lib.ptr(din), _H))
    in_.diff = din


def relu_backward(in_: Blob, out: Blob) -> None:
    """relu_backward (layers.hpp:149-155): in.diff += out.diff where in.data > 0."""
    _f32(in_.dtype)
    in_.ensure_diff()
    din = _c(in_.diff, np.float32)
    _lib.check(_lib.lib().graft_relu_backward_f32(_lib.ptr(_c(in_.data, np.float32)),
                                                  _lib.ptr(_c(out.diff, np.float32)), in_.size(),
                                                  _lib.ptr(din), _H))
    in_.diff = din


def upconv_backward(in_: Blob, out: Blob) -> None:
    """upconv_backward (layers.hpp:178-190)."""
    _f32(in_.dtype)
    in_.ensure_diff()
    din = _c(in_.diff, np.float32)
    _lib.check(_lib.lib().graft_upconv_backward_f32(_lib.ptr(_c(out.diff, np.float32)), in_.channels,
                                                    in_.height, in_.width, _lib.ptr(din), _H))
    in_.diff = din


def mergecrop_backward(a: Blob, out: Blob) -> None:
    """mergecrop_backward (layers.hpp:214-221): gradient into the first input only."""
    _f32(a.dtype)
    a.ensure_diff()
    da = _c(a.diff, np.float32)
    _lib.check(_lib.lib().graft_mergecrop_backward_f32(
        _lib.ptr(_c(out.diff[:a.size()], np.float32)), a.channels, a.height, a.width,
        _lib.ptr(da), _H))
    a.diff = da


def softmax_backward(in_: Blob, out: Blob) -> None:
    """softmax_backward (layers.hpp:246-262): in.diff += J^T out.diff."""
    _f32(in_.dtype)
    in_.ensure_diff()
    din = _c(in_.diff, np.float32)
    _lib.check(_lib.lib().graft_softmax_backward_f32(_lib.ptr(_c(out.data, np.float32)),
                                                     _lib.ptr(_c(out.diff, np.float32)), in_.channels,
                                                     in_.height, in_.width, _lib.ptr(din), _H))
    in_.diff = din


def softmax_loss(scores: Blob, labels, mask=None) -> float:
    """softmax_loss (layers.hpp:269-307): returns the loss, scores.diff += gradient. labels: int
    plane (H, W); mask: u8 plane or None (all pixels count)."""
    import ctypes as C

    _f32(scores.dtype)
    lab = np.ascontiguousarray(getattr(labels, "pix", labels), np.int32).reshape(-1)
    if lab.size != scores.plane():
        raise SizeError(f"softmax_loss: label plane does not match scores")
    m = None
    if mask is not None:
        m = np.ascontiguousarray(getattr(mask, "pix", mask), np.uint8).reshape(-1)
        if m.size == 0:
            m = None
        elif m.size != scores.plane():
            raise SizeError("softmax_loss: mask plane does not match scores")
    scores.ensure_diff()
    d = _c(scores.diff, np.float32)
    loss = C.c_double()
    _lib.check(_lib.lib().graft_softmax_loss_layer_f32(
        _lib.ptr(_c(scores.data, np.float32)), scores.channels, scores.height, scores.width,
        _lib.ptr(lab), _lib.ptr(m), _lib.ptr(d), C.byref(loss), _H))
    scores.diff = d
    return loss.value
