"""Multi-GPU sharding of the query path.

Two layouts, one process per GPU (torch.distributed, NCCL on the B200 box,
gloo in the CPU tests):

* **By camera view (config D)** -- independent units: each rank renders its
  own views of a replicated scene; the only collective is the gather of the
  final per-view results (masks / points).  ``shard_views`` + ``gather_results``.
* **By tile band of one view (config E)** -- each rank renders a band of
  tile rows plus a 5-pixel halo (the 11x11 mean filter stays local), then
  max-all-reduces of int64 keys yield select_level / localize / segment's
  global statistics.  ``band_rows`` + ``global_selection``.

Relevancy values lie in (0, 1) (positive doubles), so their IEEE bit
patterns order like the values: max/min reduce as int64 maxima of the bits
(min as the max of the negated bits), and the argmax is a second max over
negated indices restricted to the ranks that hold the global maximum -- the
reference's "lowest level, then smallest row-major index" tie rule
(query.py:111-126).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ValidationError


def shard_views(n_views: int, world_size: int, rank: int) -> list[int]:
    """Views rendered by ``rank``: round-robin, so per-rank work differs by at most one."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValidationError("bad rank / world size")
    return list(range(rank, n_views, world_size))


@dataclass(frozen=True)
class Band:
    """Rows [y0, y1) owned by a rank and the halo-extended rows it renders."""

    y0: int
    y1: int
    render_y0: int
    render_y1: int


def band_rows(height: int, world_size: int, rank: int, *, tile: int = 16, halo: int = 5) -> Band:
    """Split ``height`` into tile-aligned bands; each band renders +-halo rows."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValidationError("bad rank / world size")
    tiles_y = (height + tile - 1) // tile
    t0 = tiles_y * rank // world_size
    t1 = tiles_y * (rank + 1) // world_size
    y0, y1 = min(t0 * tile, height), min(t1 * tile, height)
    return Band(y0, y1, max(0, y0 - halo), min(height, y1 + halo))


def global_selection(level_max, level_argmax, level_min, group=None):
    """All-reduce per-level (max, argmax, min) over ranks -> (level, flat index, min, max).

    ``level_max`` / ``level_min`` are per-level float64 arrays of this rank's band,
    ``level_argmax`` the flat (global) pixel index of the band's maximum.  Two
    max-all-reduces of small int64 tensors (value/min bits, then the argmax
    index among the ranks that hold the maximum); exact on every backend.
    """
    import torch
    import torch.distributed as dist

    nl = len(level_max)
    vbits = np.asarray(level_max, dtype=np.float64).view(np.int64)        # positive -> monotone
    idx = np.asarray(level_argmax, dtype=np.int64)
    mbits = np.asarray(level_min, dtype=np.float64).view(np.int64)
    t = torch.tensor(np.concatenate([vbits, -mbits]), dtype=torch.int64)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else torch.device("cpu")
    t = t.to(dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    gmax_bits = t[:nl].cpu().numpy()
    gmin_bits = (-t[nl:]).cpu().numpy()
    # argmax: among ranks holding the global max bits, the lowest index wins
    cand = np.where(vbits == gmax_bits, idx, np.iinfo(np.int64).max)
    ti = torch.tensor(-cand, dtype=torch.int64).to(dev)
    dist.all_reduce(ti, op=dist.ReduceOp.MAX, group=group)
    gidx = (-ti).cpu().numpy()
    gmax = gmax_bits.view(np.float64)
    gmin = gmin_bits.view(np.float64)
    level = int(np.argmax(gmax))  # ties -> lowest level (query.py:111-118)
    return level, int(gidx[level]), float(gmin[level]), float(gmax[level])


def gather_results(local: "torch.Tensor", group=None) -> "torch.Tensor":
    """All-gather one equally shaped result tensor per rank (final maps / masks)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out = torch.empty((world,) + tuple(local.shape), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, local.contiguous(), group=group) if local.is_cuda else \
        dist.all_gather(list(out.unbind(0)), local.contiguous(), group=group)
    return out
