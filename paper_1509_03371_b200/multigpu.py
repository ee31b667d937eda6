"""Multi-GPU partitioner and final combine (one process per GPU, torch.distributed).

The path shards without any exchange: process()'s tiles are independent and tiling is
bit-exact (pipeline.hpp:626-629; proj/tests/test_pipeline.cpp:535-588), so

  * one image:   rank r runs the tile rows ``split_rows(n_rows, world)[r]`` through
                 graft_process_band, reading the full u8 image (the 101-px context halo comes
                 from the image itself -- no halo exchange);
  * a batch:     image i goes to rank i % world.

The only collective is the final combine: the ranks' label/probability bands (or per-image
planes) are gathered to rank 0 (NCCL over NVLink on GPUs; gloo in the CPU tests) and assembled
there. The same partition and combine exist in the C ABI for one process driving all GPUs
(graft_multi_process / graft_multi_process_batch, csrc/multi.cu; MultiProcessor below). Nothing here touches the compute; it is exercised on CPU with gloo by
tests/test_multiproc_cpu.py and on GPUs by bench.py.
"""
from __future__ import annotations

from typing import Callable, List, Sequence, Tuple


def split_rows(n_rows: int, world: int) -> List[Tuple[int, int]]:
    """Balanced contiguous split of tile rows [0, n_rows) into `world` ranges (some may be
    empty when n_rows < world)."""
    base, extra = divmod(n_rows, world)
    out, r0 = [], 0
    for r in range(world):
        r1 = r0 + base + (1 if r < extra else 0)
        out.append((r0, r1))
        r0 = r1
    return out


def band_rows_py(H: int, w: int, r0: int, r1: int) -> Tuple[int, int]:
    """Output rows owned by tile rows [r0, r1) (the same rule as graft_band_rows): tile row r
    starts at min(r*w, H-w); a band owns [start(r0), start(r1)) with start(0)=0, start(n)=H."""
    n = (H + w - 1) // w
    if r0 >= r1:
        s = 0 if r0 <= 0 else min(r0 * w, H - w)
        return s, s
    y0 = 0 if r0 <= 0 else min(r0 * w, H - w)
    y1 = H if r1 >= n else min(r1 * w, H - w)
    return y0, y1


def _gather(t, rank: int, world: int, dst: int, group):
    """dist.gather of equal-shape tensors to `dst` (None on other ranks); NCCL runs it as a
    group of point-to-point sends to the destination, gloo natively."""
    import torch
    import torch.distributed as dist

    out = [torch.empty_like(t) for _ in range(world)] if rank == dst else None
    dist.gather(t, out, dst=dst, group=group)
    return out


def combine_bands(labels, probs, bands: Sequence[Tuple[int, int]], rank: int, world: int,
                  group=None, dst: int = 0):
    """Gathers every rank's rows [y0, y1) of (labels H x W, probs C x H x W) into rank `dst`'s
    planes (the final combine goes to one rank; other ranks keep only their own
    rows). Works on CUDA tensors (NCCL) and CPU tensors (gloo); bands are padded to the largest
    band height for the collective."""
    import torch

    H, W = labels.shape
    C = probs.shape[0]
    hmax = max(y1 - y0 for y0, y1 in bands)
    if hmax == 0:
        return labels, probs
    y0, y1 = bands[rank]
    lab_band = torch.zeros((hmax, W), dtype=labels.dtype, device=labels.device)
    prob_band = torch.zeros((C, hmax, W), dtype=probs.dtype, device=probs.device)
    lab_band[: y1 - y0] = labels[y0:y1]
    prob_band[:, : y1 - y0] = probs[:, y0:y1]
    lab_all = _gather(lab_band, rank, world, dst, group)
    prob_all = _gather(prob_band, rank, world, dst, group)
    if rank == dst:
        for r, (a, b) in enumerate(bands):
            labels[a:b] = lab_all[r][: b - a]
            probs[:, a:b] = prob_all[r][:, : b - a]
    return labels, probs


def process_image(run_band: Callable, H: int, w: int, rank: int, world: int, labels, probs,
                  group=None):
    """Strong-scaling process() of one image: `run_band(r0, r1)` fills rows of its tile rows
    [r0, r1) into labels/probs (graft_process_band); then the bands are combined."""
    n_rows = (H + w - 1) // w
    splits = split_rows(n_rows, world)
    bands = [band_rows_py(H, w, r0, r1) for r0, r1 in splits]
    r0, r1 = splits[rank]
    if r1 > r0:
        run_band(r0, r1)
    if world > 1:
        combine_bands(labels, probs, bands, rank, world, group)
    return labels, probs


def batch_assignment(n_images: int, world: int, rank: int) -> List[int]:
    """Images of a batch owned by `rank` (round robin)."""
    return list(range(rank, n_images, world))


def gather_batch(per_image: dict, n_images: int, shape_lab, shape_prob, rank: int, world: int,
                 device, group=None):
    """All-gathers the per-image (labels, probs) computed by each rank (weak scaling): returns
    lists indexed by image on every rank."""
    import torch
    import torch.distributed as dist

    labs, probs = [None] * n_images, [None] * n_images
    for i in range(0, n_images, world):
        own = i + rank
        if own < n_images:
            lab, pr = per_image[own]
        else:
            lab = torch.zeros(shape_lab, dtype=torch.uint8, device=device)
            pr = torch.zeros(shape_prob, dtype=torch.float32, device=device)
        la = [torch.empty_like(lab) for _ in range(world)]
        pa = [torch.empty_like(pr) for _ in range(world)]
        if world > 1:
            dist.all_gather(la, lab, group=group)
            dist.all_gather(pa, pr, group=group)
        else:
            la, pa = [lab], [pr]
        for r in range(world):
            if i + r < n_images:
                labs[i + r], probs[i + r] = la[r], pa[r]
    return labs, probs


def shard_range(n_images: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous block of a batch owned by `rank` (sizes differ by at most one)."""
    q, r = divmod(n_images, world)
    begin = rank * q + min(rank, r)
    return begin, begin + q + (1 if rank < r else 0)


def gather_shards(lab_shard, prob_shard, n_images: int, rank: int, world: int, group=None,
                  dst: int = 0):
    """Gathers per-rank batch shards (labels [n_r, H, W], probs [n_r, C, H, W], rank r owning
    shard_range(...)) into the full batch on rank `dst` (None, None elsewhere): the batch mode's
    only collective. Shards are padded to the largest size for the collective and trimmed."""
    import torch
    import torch.distributed as dist

    sizes = [shard_range(n_images, world, r) for r in range(world)]
    cap = max(e - b for b, e in sizes)

    def padded(t):
        out = torch.zeros((cap,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        out[:t.shape[0]] = t
        return out

    lp, pp = padded(lab_shard), padded(prob_shard)
    if world > 1 or (dist.is_available() and dist.is_initialized()):
        la = _gather(lp, rank, world, dst, group)
        pa = _gather(pp, rank, world, dst, group)
    else:
        la, pa = [lp], [pp]
    if rank != dst:
        return None, None
    labs = torch.cat([la[r][:e - b] for r, (b, e) in enumerate(sizes)])
    probs = torch.cat([pa[r][:e - b] for r, (b, e) in enumerate(sizes)])
    return labs, probs


def process_batch_sharded(proc, images, w: int, v: int, rank: int, world: int, device,
                          group=None):
    """Weak-scaling batch mode (BASELINE configs[3]): rank r runs graft_process_batch on its
    contiguous shard of the (N, H, W) device batch and the shards are all-gathered."""
    import torch
    from . import _lib

    n, H, W = images.shape
    b, e = shard_range(n, world, rank)
    lab = torch.empty((e - b, H, W), dtype=torch.uint8, device=device)
    prob = torch.empty((e - b, proc.n_classes, H, W), dtype=torch.float32, device=device)
    if e > b:
        proc.run_batch(images[b:e], w, v, lab, prob, mem=_lib.MEM_DEVICE)
    return gather_shards(lab, prob, n, rank, world, group)


class MultiProcessor:
    """process() across the GPUs of this node from ONE process (graft_multi_*, csrc/multi.cu):
    the net replicated on `devices`, one host thread and stream per GPU per call, tile-row
    bands (one image) or image blocks (a batch) per GPU, planes bit-identical to one GPU's.
    With device buffers (on devices[0]) the combine is one NCCL group of send/recv to rank 0
    (peer copies when ranks share a device); with host buffers each GPU copies its own rows."""

    def __init__(self, spec, states, devices=None, n_gpus: int = 0):
        import ctypes as C

        from . import _lib
        from .netgraph import net_descs
        from .netspec import LayerKind, compute_channels

        if devices is None:
            devices = list(range(n_gpus or 1))
        self.devices = list(devices)
        arr, self._keep = net_descs(spec)
        devs = (C.c_int * len(self.devices))(*self.devices)
        h = C.c_void_p()
        _lib.check(_lib.lib().graft_multi_create(spec.f0, len(spec.layers), arr, len(self.devices),
                                                 devs, C.byref(h)))
        self.h = h
        self.spec = spec
        self.n_classes = compute_channels(spec)[spec.layers[-1].output]
        import numpy as np

        for i, l in enumerate(spec.layers):
            if l.kind != LayerKind.ConvSK:
                continue
            st = states.layers[i]
            w = np.ascontiguousarray(st.weights, np.float32)
            b = np.ascontiguousarray(st.bias, np.float32)
            _lib.check(_lib.lib().graft_multi_set_params_f32(self.h, i, _lib.ptr(w), w.size,
                                                             _lib.ptr(b), b.size))

    def close(self):
        from . import _lib

        if getattr(self, "h", None) is not None and self.h.value:
            _lib.lib().graft_multi_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def combine_kind(self) -> str:
        import ctypes as C

        from . import _lib

        k = C.c_int()
        _lib.check(_lib.lib().graft_multi_combine_kind(self.h, C.byref(k)))
        return {_lib.COMBINE_NCCL: "nccl", _lib.COMBINE_PEER: "peer"}[k.value]

    def set_option(self, opt: int, value: int) -> None:
        from . import _lib

        _lib.check(_lib.lib().graft_multi_set_option(self.h, opt, int(value)))

    def run(self, image, w: int, v: int, labels=None, probs=None, mem: int = 0):
        import numpy as np

        from . import _lib

        if mem == _lib.MEM_HOST:
            image = np.ascontiguousarray(image, np.uint8)
            H, W = image.shape
            labels = np.zeros((H, W), np.uint8) if labels is None else labels
            probs = np.zeros((self.n_classes, H, W), np.float32) if probs is None else probs
        else:
            H, W = image.shape
        _lib.check(_lib.lib().graft_multi_process(self.h, _lib.ptr(image), H, W, w, v,
                                                  _lib.ptr(labels), _lib.ptr(probs), mem))
        return labels, probs

    def run_batch(self, images, w: int, v: int, labels=None, probs=None, mem: int = 0):
        import numpy as np

        from . import _lib

        if mem == _lib.MEM_HOST:
            images = np.ascontiguousarray(images, np.uint8)
            N, H, W = images.shape
            labels = np.zeros((N, H, W), np.uint8) if labels is None else labels
            probs = np.zeros((N, self.n_classes, H, W), np.float32) if probs is None else probs
        else:
            N, H, W = images.shape
        _lib.check(_lib.lib().graft_multi_process_batch(self.h, _lib.ptr(images), N, H, W, w, v,
                                                        _lib.ptr(labels), _lib.ptr(probs), mem))
        return labels, probs
