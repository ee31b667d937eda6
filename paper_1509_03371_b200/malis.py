"""MALIS (malis.hpp) on the B200: the reference's functions, and batched forms of them.

Each call runs through libgraft_cuda.so (csrc/malis.cu): one CTA per patch, the union-find of
a pass on one thread of that CTA, everything around it (keys, sort, affinity graphs,
components, gradients, softmax) on the CTA's threads. The single-patch functions keep the
reference's signatures and messages; the ``*_batch`` forms take a leading batch axis, which
is what the device parallelises over. Results are bit-identical to the reference for float32
and float64 (tests/test_gpu_malis.py).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Tuple

import numpy as np

from . import _lib
from .blob import Blob
from .errors import SizeError


def _sfx(dtype) -> str:
    dt = np.dtype(dtype)
    if dt == np.float32:
        return "f32"
    if dt == np.float64:
        return "f64"
    raise TypeError(f"MALIS runs float32 or float64, not {dt}")


def _batched(a: np.ndarray, dtype=None) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype)
    return a[None] if a.ndim == 2 else a


@dataclass
class AffinityGraph:
    """AffinityGraph<S> (malis.hpp:19-29): edge maps of the image extent (a leading batch axis
    in the batched forms). a_x(y, x) joins (y, x)-(y, x+1); a_y(y, x) joins (y, x)-(y+1, x);
    the unused last column / row hold 1; m_* record which endpoint supplied the min."""
    a_x: np.ndarray
    a_y: np.ndarray
    m_x: np.ndarray
    m_y: np.ndarray

    @property
    def height(self) -> int:
        return self.a_x.shape[-2]

    @property
    def width(self) -> int:
        return self.a_x.shape[-1]


@dataclass
class MalisResult:
    """MalisResult<S> (malis.hpp:113-121); batched forms carry a leading batch axis."""
    da_x: np.ndarray
    da_y: np.ndarray
    pos_x: np.ndarray
    pos_y: np.ndarray
    neg_x: np.ndarray
    neg_y: np.ndarray
    total_pos: np.ndarray
    total_neg: np.ndarray
    loss_pos: np.ndarray
    loss_neg: np.ndarray
    loss: np.ndarray


def affinity_forward_batch(fg: np.ndarray) -> AffinityGraph:
    """affinity_forward (malis.hpp:34-52) of B planes (B, h, w)."""
    x = _batched(fg)
    B, h, w = x.shape
    ax, ay = np.empty_like(x), np.empty_like(x)
    mx, my = np.empty(x.shape, np.uint8), np.empty(x.shape, np.uint8)
    fn = getattr(_lib.lib(), f"graft_affinity_forward_{_sfx(x.dtype)}")
    _lib.check(fn(_lib.ptr(x), B, h, w, _lib.ptr(ax), _lib.ptr(ay), _lib.ptr(mx), _lib.ptr(my), _lib.MEM_HOST))
    return AffinityGraph(ax, ay, mx, my)


def affinity_forward(fg: np.ndarray) -> AffinityGraph:
    g = affinity_forward_batch(np.asarray(fg)[None])
    return AffinityGraph(g.a_x[0], g.a_y[0], g.m_x[0], g.m_y[0])


def affinity_backward_batch(da_x, da_y, g: AffinityGraph) -> Tuple[np.ndarray, np.ndarray]:
    """affinity_backward (malis.hpp:58-80): (d_pos, d_neg)."""
    dx, dy = _batched(da_x), _batched(da_y)
    mx, my = _batched(g.m_x, np.uint8), _batched(g.m_y, np.uint8)
    if dx.shape != mx.shape or dy.shape != mx.shape:
        raise SizeError("affinity_backward: gradient maps must match the graph extent")
    B, h, w = dx.shape
    dp, dn = np.empty_like(dx), np.empty_like(dx)
    fn = getattr(_lib.lib(), f"graft_affinity_backward_{_sfx(dx.dtype)}")
    _lib.check(fn(_lib.ptr(dx), _lib.ptr(dy), _lib.ptr(mx), _lib.ptr(my), B, h, w, _lib.ptr(dp), _lib.ptr(dn),
                  _lib.MEM_HOST))
    return dp, dn


def affinity_backward(da_x, da_y, g: AffinityGraph) -> Tuple[np.ndarray, np.ndarray]:
    dp, dn = affinity_backward_batch(np.asarray(da_x)[None], np.asarray(da_y)[None],
                                     AffinityGraph(*(np.asarray(a)[None] for a in (g.a_x, g.a_y, g.m_x, g.m_y))))
    return dp[0], dn[0]


def connected_components_batch(labels: np.ndarray) -> np.ndarray:
    """connected_components (malis.hpp:84-111) of B label planes (nonzero = foreground)."""
    lab = (_batched(labels) != 0).astype(np.uint8)
    B, h, w = lab.shape
    comp = np.empty(lab.shape, np.int32)
    _lib.check(_lib.lib().graft_connected_components_u8(_lib.ptr(lab), B, h, w, _lib.ptr(comp), _lib.MEM_HOST))
    return comp


def connected_components(labels: np.ndarray) -> np.ndarray:
    return connected_components_batch(np.asarray(labels)[None])[0]


def malis_gradient_batch(pred: AffinityGraph, truth: AffinityGraph, comp: np.ndarray) -> MalisResult:
    """malis_gradient (malis.hpp:197-298) of B independent patches."""
    pax, pay = _batched(pred.a_x), _batched(pred.a_y)
    dt = pax.dtype
    tax, tay = _batched(truth.a_x, dt), _batched(truth.a_y, dt)
    cp = _batched(comp, np.int32)
    if not (pax.shape == pay.shape == tax.shape == tay.shape == cp.shape):
        raise SizeError("malis_gradient: pred, truth and component shapes must agree")
    B, h, w = cp.shape
    dax, day = np.empty(cp.shape, dt), np.empty(cp.shape, dt)
    cnt = [np.empty(cp.shape, np.int64) for _ in range(4)]
    totals = np.zeros((B, 2), np.int64)
    losses = np.zeros((B, 3), np.float64)
    fn = getattr(_lib.lib(), f"graft_malis_gradient_{_sfx(dt)}")
    _lib.check(fn(_lib.ptr(pax), _lib.ptr(pay), _lib.ptr(tax), _lib.ptr(tay), _lib.ptr(cp), B, h, w, _lib.ptr(dax),
                  _lib.ptr(day), *[_lib.ptr(c) for c in cnt], _lib.ptr(totals), _lib.ptr(losses), _lib.MEM_HOST))
    return MalisResult(dax, day, cnt[0], cnt[1], cnt[2], cnt[3], totals[:, 0], totals[:, 1], losses[:, 0],
                       losses[:, 1], losses[:, 2])


def malis_gradient(pred: AffinityGraph, truth: AffinityGraph, comp: np.ndarray) -> MalisResult:
    if not (np.shape(pred.a_x) == np.shape(truth.a_x) == np.shape(comp)):
        raise SizeError("malis_gradient: pred, truth and component shapes must agree")
    r = malis_gradient_batch(AffinityGraph(*(np.asarray(a)[None] for a in (pred.a_x, pred.a_y, pred.m_x, pred.m_y))),
                             AffinityGraph(*(np.asarray(a)[None] for a in (truth.a_x, truth.a_y, truth.m_x,
                                                                           truth.m_y))),
                             np.asarray(comp)[None])
    return MalisResult(*(v[0] for v in (r.da_x, r.da_y, r.pos_x, r.pos_y, r.neg_x, r.neg_y)),
                       int(r.total_pos[0]), int(r.total_neg[0]), float(r.loss_pos[0]), float(r.loss_neg[0]),
                       float(r.loss[0]))


def malis_softmax_loss_batch(scores: np.ndarray, fg: np.ndarray, diff: np.ndarray = None):
    """malis_softmax_loss (malis.hpp:311-346) of B patches: scores (B, 2, h, w), fg (B, h, w).
    Returns (losses (B,), diff + gradient): a new array; `diff` (zeros if None) is not modified."""
    sc = np.ascontiguousarray(scores)
    if sc.ndim != 4:
        raise SizeError("malis loss: scores must be (B, C, h, w)")
    B, nc, h, w = sc.shape
    if nc != 2:
        raise SizeError(f"malis loss: needs exactly 2 score channels, got {nc}")
    f = np.ascontiguousarray(fg, np.uint8)
    if f.shape != (B, h, w):
        raise SizeError("malis loss: label plane does not match score extent")
    d = np.zeros_like(sc) if diff is None else np.array(diff, sc.dtype, order="C", copy=True)
    losses = np.zeros(B, np.float64)
    fn = getattr(_lib.lib(), f"graft_malis_softmax_loss_{_sfx(sc.dtype)}")
    _lib.check(fn(_lib.ptr(sc), B, nc, h, w, _lib.ptr(f), _lib.ptr(d), _lib.ptr(losses), _lib.MEM_HOST))
    return losses, d


def malis_softmax_loss(scores: Blob, fg: np.ndarray) -> float:
    """malis_softmax_loss<S>(scores, fg): the loss; the gradient accumulates into scores.diff."""
    if scores.channels != 2:
        raise SizeError(f"malis loss: needs exactly 2 score channels, got {scores.channels}")
    f = np.asarray(fg)
    if f.shape != (scores.height, scores.width):
        raise SizeError("malis loss: label plane does not match score extent")
    scores.ensure_diff()
    x = scores.data.reshape(1, 2, scores.height, scores.width)
    losses, d = malis_softmax_loss_batch(x, f[None], scores.diff.reshape(x.shape).copy())
    scores.diff = d.reshape(-1)
    return float(losses[0])


def malis_softmax_loss_device(net_handle, scores_blob: str, fg: np.ndarray) -> float:
    """The training runner's MALIS loss on its device score blob (graft_net_malis_softmax_loss_f32)."""
    f = np.ascontiguousarray(fg, np.uint8)
    H, W = f.shape
    loss = C.c_double()
    _lib.check(_lib.lib().graft_net_malis_softmax_loss_f32(net_handle, scores_blob.encode(), _lib.ptr(f), H, W,
                                                           C.byref(loss)))
    return loss.value
