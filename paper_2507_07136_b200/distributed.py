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
    if world_size > tiles_y:
        # every rank raises here, before any collective: a rank with an empty
        # band would otherwise render nothing (or the whole frame) while the
        # others wait for it in the selection all-reduce
        raise ValidationError(f"{world_size} ranks exceed the {tiles_y} tile rows of a {height}-row image")
    t0 = tiles_y * rank // world_size
    t1 = tiles_y * (rank + 1) // world_size
    y0, y1 = min(t0 * tile, height), min(t1 * tile, height)
    return Band(y0, y1, max(0, y0 - halo), min(height, y1 + halo))


def combine_selection(level_max, level_argmax, level_min):
    """Host-side combination of per-band statistics, the single-process twin of
    ``global_selection``: lists (one entry per band) of per-level max / first
    argmax (flat, whole image) / min -> (level, flat index, min, max) of the
    reference's select_level / localize / segment (query.py:111-145)."""
    mx = np.max(np.asarray(level_max, dtype=np.float64), axis=0)
    mn = np.min(np.asarray(level_min, dtype=np.float64), axis=0)
    level = int(np.argmax(mx))  # ties -> lowest level
    cands = [int(a[level]) for m, a in zip(level_max, level_argmax) if m[level] == mx[level]]
    return level, min(cands), float(mn[level]), float(mx[level])


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


def combine_selection_many(level_max, level_argmax, level_min):
    """combine_selection for many prompts: arrays (bands, prompts, levels) ->
    one (level, flat index, min, max) per prompt."""
    mx, am, mn = (np.asarray(a) for a in (level_max, level_argmax, level_min))
    return [combine_selection(mx[:, i], am[:, i], mn[:, i]) for i in range(mx.shape[1])]


def global_selection_many(level_max, level_argmax, level_min, group=None):
    """global_selection for many prompts at once: (prompts, levels) arrays of this
    rank's band -> one (level, flat index, min, max) per prompt, with the same
    two max-all-reduces (of n_prompts x levels int64 keys) for all prompts."""
    import torch
    import torch.distributed as dist

    vbits = np.ascontiguousarray(level_max, dtype=np.float64).view(np.int64)
    idx = np.asarray(level_argmax, dtype=np.int64)
    mbits = np.ascontiguousarray(level_min, dtype=np.float64).view(np.int64)
    n, nl = vbits.shape
    t = torch.tensor(np.concatenate([vbits.ravel(), -mbits.ravel()]), dtype=torch.int64)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else torch.device("cpu")
    t = t.to(dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    tt = t.cpu().numpy()
    gmax_bits = tt[:n * nl].reshape(n, nl)
    gmin_bits = (-tt[n * nl:]).reshape(n, nl)
    cand = np.where(vbits == gmax_bits, idx, np.iinfo(np.int64).max)
    ti = torch.tensor(-cand.ravel(), dtype=torch.int64).to(dev)
    dist.all_reduce(ti, op=dist.ReduceOp.MAX, group=group)
    gidx = (-ti).cpu().numpy().reshape(n, nl)
    gmax = gmax_bits.view(np.float64)
    gmin = gmin_bits.view(np.float64)
    out = []
    for i in range(n):
        level = int(np.argmax(gmax[i]))  # ties -> lowest level (query.py:111-118)
        out.append((level, int(gidx[i, level]), float(gmin[i, level]), float(gmax[i, level])))
    return out


def gather_results(local: "torch.Tensor", group=None) -> "torch.Tensor":
    """All-gather one equally shaped result tensor per rank (final maps / masks)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out = torch.empty((world,) + tuple(local.shape), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, local.contiguous(), group=group) if local.is_cuda else \
        dist.all_gather(list(out.unbind(0)), local.contiguous(), group=group)
    return out


@dataclass
class BandQuery:
    """One rank's share of a tile-band sharded query frame (config E)."""

    band: Band
    level: int
    point: tuple
    lo: float
    hi: float
    degenerate: bool
    out: object  # FrameOutputs: filtered maps (owned rows) and mask rows [band.y0, band.y1)


def band_statistics(out, n_levels: int):
    """(max, first argmax, min) per level over the owned rows of a band frame."""
    from . import _native as N

    st_i, st_f = out.host_stats()
    mx = [float(st_f[N.STATF_LEVEL_MAX + b]) for b in range(n_levels)]
    mn = [float(st_f[N.STATF_LEVEL_MAX + n_levels + b]) for b in range(n_levels)]
    am = [int(st_i[N.STAT_LEVEL_ARGMAX + b]) for b in range(n_levels)]
    return mx, am, mn


def mask_rows(out, level: int, lo: float, hi: float, threshold: float, y0: int, y1: int) -> None:
    """segment().mask of rows [y0, y1) with the global normalisation (sf_mask_rows)."""
    import ctypes

    from . import _native as N
    from .device import stream_ptr

    H, W = out.height, out.width
    N.check(N.load().sf_mask_rows(N.ptr(out.relevancy_filtered), H, W, int(level), ctypes.c_double(lo),
                                  ctypes.c_double(hi), ctypes.c_double(threshold), int(y0), int(y1),
                                  N.ptr(out.mask), stream_ptr()))


def band_query(engine, cam, levels, spec, world_size: int, rank: int, group=None, out=None) -> BandQuery:
    """Render and query the tile band of ``rank``.

    The rank renders the tile rows covering its band plus the 5-pixel halo of
    the 11x11 mean filter (the per-tile results are identical to the full
    frame's), reduces per-level statistics over its own rows, max-all-reduces
    them across ranks (``global_selection``; exact int64 keys) and writes its
    mask rows with the global level / min / max.  With ``group=None`` and no
    initialised process group the selection is the rank's own (world of 1)."""
    import torch.distributed as dist

    H = int(cam.height)
    band = band_rows(H, world_size, rank, halo=int(spec.window) // 2)
    if out is None:
        # the coefficient map is only materialised when the relevancy is not
        # fused into the blend (it is then computed from the map, sf_capi.cu)
        from . import _native as N
        cfg = engine.ds.config
        wide = not N.load().sf_relevancy_fused(len(levels), int(cfg.L), int(cfg.K), int(len(spec.canonicals)))
        out = engine.allocate(int(cam.width), H, levels, coeff_map=wide, features=False, query=True)
    engine.run(cam, levels, out, query=spec, band=(band.y0, band.y1))
    mx, am, mn = band_statistics(out, len(levels))
    if dist.is_available() and dist.is_initialized():
        level, idx, lo, hi = global_selection(mx, am, mn, group=group)
    else:
        level, idx, lo, hi = combine_selection([mx], [am], [mn])
    if spec.fixed_level is not None and int(spec.fixed_level) >= 0:
        level = int(spec.fixed_level)
        if dist.is_available() and dist.is_initialized():
            _, idx, lo, hi = _fixed_level_selection(mx, am, mn, level, group)
        else:
            idx, lo, hi = am[level], mn[level], mx[level]
    mask_rows(out, level, lo, hi, float(spec.threshold), band.y0, band.y1)
    W = int(cam.width)
    return BandQuery(band, level, (idx // W, idx % W), lo, hi, not (hi > lo), out)


def _fixed_level_selection(mx, am, mn, level, group):
    """global_selection restricted to one level (query_pipeline(level=...))."""
    one = [mx[level]], [am[level]], [mn[level]]
    _, idx, lo, hi = global_selection(*one, group=group)
    return level, idx, lo, hi


@dataclass
class BandSweep:
    """One rank's share of a tile-band sharded prompt sweep (config E)."""

    band: Band
    selections: list          # per prompt: (level, (row, col), lo, hi, degenerate)
    filtered: object          # (prompts, levels, H, W) fp64; owned rows valid
    masks: object             # (prompts, H, W) u8; owned rows valid


def band_sweep_statistics(engine, cam, levels, prompts, canonicals, world_size: int, rank: int, *,
                          window: int = 11, threshold: float = 0.5):
    """Render the band of ``rank`` once and run every prompt over its owned rows:
    (band, filtered, masks, per-prompt level max / first argmax / min arrays)."""
    from . import _native as N
    H, W = int(cam.height), int(cam.width)
    band = band_rows(H, world_size, rank, halo=int(window) // 2)
    out = engine.allocate(W, H, levels, coeff_map=True, mask=False)
    filt, masks, st_i, st_f = engine.sweep(cam, levels, out, np.asarray(prompts, dtype=np.float64),
                                           np.asarray(canonicals, dtype=np.float64), window=window,
                                           threshold=threshold, band=(band.y0, band.y1))
    nl = len(levels)
    mx = st_f[:, N.STATF_LEVEL_MAX:N.STATF_LEVEL_MAX + nl]
    mn = st_f[:, N.STATF_LEVEL_MAX + nl:N.STATF_LEVEL_MAX + 2 * nl]
    am = st_i[:, N.STAT_LEVEL_ARGMAX:N.STAT_LEVEL_ARGMAX + nl]
    return band, filt, masks, mx, am, mn


def finish_band_sweep(band, filt, masks, selections, threshold: float, W: int, H: int) -> BandSweep:
    """Write each prompt's mask rows of the band with its global selection."""
    import ctypes

    import torch

    from . import _native as N
    from .device import stream_ptr
    lib = N.load()
    out_sel = []
    for i, (level, idx, lo, hi) in enumerate(selections):
        N.check(lib.sf_mask_rows(N.ptr(filt[i]), H, W, int(level), ctypes.c_double(lo), ctypes.c_double(hi),
                                 ctypes.c_double(threshold), int(band.y0), int(band.y1), N.ptr(masks[i]),
                                 stream_ptr()))
        out_sel.append((level, (idx // W, idx % W), lo, hi, not (hi > lo)))
    torch.cuda.current_stream().synchronize()
    return BandSweep(band, out_sel, filt, masks)


def band_query_sweep(engine, cam, levels, prompts, canonicals, world_size: int, rank: int, *, window: int = 11,
                     threshold: float = 0.5, group=None) -> BandSweep:
    """query_sweep over the tile band of ``rank`` (config E: tile bands x prompts):
    the band is rendered once, every prompt's relevancy / filter / statistics
    cover the owned rows, one pair of all-reduces selects all prompts' level /
    point / range (``global_selection_many``), and each prompt's mask rows are
    written with its global normalisation.  Without a process group the
    selection is the rank's own (world of 1)."""
    import torch.distributed as dist

    band, filt, masks, mx, am, mn = band_sweep_statistics(engine, cam, levels, prompts, canonicals, world_size,
                                                          rank, window=window, threshold=threshold)
    if dist.is_available() and dist.is_initialized():
        sel = global_selection_many(mx, am, mn, group=group)
    else:
        sel = combine_selection_many(mx[None], am[None], mn[None])
    return finish_band_sweep(band, filt, masks, sel, threshold, int(cam.width), int(cam.height))
