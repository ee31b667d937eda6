"""Multi-GPU partitioner and final combine (one process per GPU, torch.distributed).

The path shards without any exchange: process()'s tiles are independent and tiling is
bit-exact (pipeline.hpp:626-629; proj/tests/test_pipeline.cpp:535-588), so

  * one image:   rank r runs the tile rows ``split_rows(n_rows, world)[r]`` through
                 graft_process_band, reading the full u8 image (the 101-px context halo comes
                 from the image itself -- no halo exchange);
  * a batch:     image i goes to rank i % world.

The only collective is the final combine: the ranks' label/probability bands (or per-image
planes) are all-gathered (NCCL over NVLink on GPUs; gloo in the CPU tests) and assembled on
every rank. Nothing here touches the compute; it is exercised on CPU with gloo by
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


def combine_bands(labels, probs, bands: Sequence[Tuple[int, int]], rank: int, world: int,
                  group=None):
    """All-gathers every rank's rows [y0, y1) of (labels H x W, probs C x H x W) so that all ranks
    end with the full planes. Works on CUDA tensors (NCCL) and CPU tensors (gloo); bands are
    padded to the largest band height for the collective."""
    import torch
    import torch.distributed as dist

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
    lab_all = [torch.empty_like(lab_band) for _ in range(world)]
    prob_all = [torch.empty_like(prob_band) for _ in range(world)]
    dist.all_gather(lab_all, lab_band, group=group)
    dist.all_gather(prob_all, prob_band, group=group)
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


def gather_shards(lab_shard, prob_shard, n_images: int, rank: int, world: int, group=None):
    """All-gathers per-rank batch shards (labels [n_r, H, W], probs [n_r, C, H, W], rank r owning
    shard_range(...)) into the full batch on every rank: the batch mode's only collective.
    Shards are padded to the largest size for the NCCL all-gather and trimmed after."""
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
        la = [torch.empty_like(lp) for _ in range(world)]
        pa = [torch.empty_like(pp) for _ in range(world)]
        dist.all_gather(la, lp, group=group)
        dist.all_gather(pa, pp, group=group)
    else:
        la, pa = [lp], [pp]
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
