"""Sparse-coefficient splatting + decode + query (drop-in for splatfield/sparse_splat.py).

Per pixel and level the blend accumulates only each Gaussian's K stored
coefficients (sparse_splat.py:138-150); ``decode`` recovers the D-dimensional
features with one contraction per level (:183-199).  Here the whole frame --
projection, depth-rank sort, binning, blend, decode, relevancy, filter,
selection, localisation, segmentation -- is one native call
(``sf_render_frame``) on the GPU; results stay in HBM and materialise as
float64 numpy arrays only when a caller reads ``.data`` / ``.maps``.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import ValidationError
from .projection import DEFAULT_TILE_SIZE
from .query import QueryEmbedding, RelevancyMap
from .rasterizer import (DEFAULT_MAX_RENDER_ELEMENTS, TAG_COEFFICIENT, RenderStats,
                         check_render_budget)


class CoefficientMap:
    """Rendered sparse-coefficient accumulator (sparse_splat.py:46-88).

    ``data`` is (H, W, len(levels) * L) float64 (materialised from the fp32
    device tensor ``dev`` on first access).
    """

    def __init__(self, data=None, L: int = 0, K: int = 0, levels=(0,), *, dev=None):
        self.L = int(L)
        self.K = int(K)
        self.levels = tuple(levels)
        self.dev = dev
        self._data = None
        if dev is None:
            self._data = np.asarray(data)
            shape = self._data.shape
        else:
            shape = tuple(dev.shape)
        if len(shape) != 3 or shape[2] != len(self.levels) * self.L:
            raise ValidationError(
                f"coefficient map shape {shape} does not match "
                f"{len(self.levels)} level(s) of {self.L} channels")

    @property
    def data(self) -> np.ndarray:
        if self._data is None:
            self._data = self.dev.double().cpu().numpy()
        return self._data

    @property
    def shape(self):
        return tuple(self.dev.shape) if self.dev is not None else self._data.shape

    @property
    def num_levels(self) -> int:
        return len(self.levels)

    def level_view(self, level: int) -> np.ndarray:
        b = self.levels.index(level)
        return self.data[:, :, b * self.L:(b + 1) * self.L]

    def device_tensor(self):
        """(H, W, n_ch) float32 CUDA tensor."""
        import torch

        from .device import require_cuda
        if self.dev is None:
            self.dev = torch.from_numpy(np.ascontiguousarray(self._data, dtype=np.float32)).to(require_cuda())
        return self.dev

    def validate(self) -> None:
        d = self.data
        if not np.all(np.isfinite(d)):
            raise ValidationError("coefficient map must be finite")
        if np.any(d < 0) or np.any(d > 1):
            raise ValidationError("coefficient channels must lie in [0, 1]")
        for level in self.levels:
            if np.any(self.level_view(level).sum(axis=2) > 1.0 + 1e-5):
                raise ValidationError("per-level channel sum exceeds 1")


class FeatureMapSet:
    """Per-level H x W x D feature buffers (sparse_splat.py:91-100).

    ``maps`` materialises float64 numpy arrays; ``dev`` is the (levels, H, W,
    D) float32 device tensor.  A lazy set decodes on first use.
    """

    def __init__(self, maps=None, levels=(0,), provenance="decoded-from-coefficients", *,
                 dev=None, thunk=None):
        self.levels = tuple(levels)
        self.provenance = provenance
        self._dev = dev
        self._thunk = thunk
        self._maps = tuple(maps) if maps is not None else None

    @property
    def dev(self):
        if self._dev is None and self._thunk is not None:
            self._dev = self._thunk()
            self._thunk = None
        return self._dev

    @property
    def maps(self):
        if self._maps is None:
            d = self.dev
            self._maps = tuple(d[b].double().cpu().numpy() for b in range(d.shape[0]))
        return self._maps

    def level_map(self, level: int):
        return self.maps[self.levels.index(level)]


def _levels_and_checks(scene, levels, tile_size, max_elements, W, H):
    cfg = scene.config
    levels = tuple(int(lv) for lv in levels)
    for lv in levels:
        if not 0 <= lv < cfg.num_levels:
            raise ValidationError(f"level {lv} out of range for {cfg.num_levels} levels")
    if tile_size != DEFAULT_TILE_SIZE:
        raise ValidationError("the sm_100a kernels are specialised for 16x16 tiles")
    check_render_budget(W, H, len(levels) * cfg.L, max_elements)
    return levels


def _splat_levels(scene, cam, levels, *, tile_size: int = DEFAULT_TILE_SIZE, early_exit: bool = True,
                  max_elements: int = DEFAULT_MAX_RENDER_ELEMENTS, workers: int = 1,
                  with_stats: bool = False):
    """Fused multi-level sparse splat (sparse_splat.py:103-170) on the GPU."""
    from .device import device_scene
    W, H = int(cam.width), int(cam.height)
    levels = _levels_and_checks(scene, levels, tile_size, max_elements, W, H)
    ds = device_scene(scene)
    if ds.bad_index:
        raise ValidationError("coefficient index >= L")
    eng = ds.engine
    out = eng.allocate(W, H, levels, coeff_map=True, final_t=with_stats)
    eng.run(cam, levels, out, early_exit=early_exit)
    cfg = scene.config
    cmap = CoefficientMap(L=cfg.L, K=cfg.K, levels=levels, dev=out.coeff_map)
    if not with_stats:
        return cmap
    st = out.stats_i64.cpu().numpy()
    stats = RenderStats(final_transmittance=out.final_t.double().cpu().numpy(),
                        pairs_blended=int(st[N.STAT_PAIRS]),
                        channels_per_gaussian=len(levels) * cfg.K, workers=workers)
    return cmap, stats


def splat_sparse(scene, cam, level: int, **kwargs):
    """One level's L-dim coefficient map at K-channel blend cost (sparse_splat.py:173-175)."""
    return _splat_levels(scene, cam, [level], **kwargs)


def splat_multilevel(scene, cam, **kwargs):
    """Every configured level in one fused pass (sparse_splat.py:178-180)."""
    return _splat_levels(scene, cam, range(scene.config.num_levels), **kwargs)


def decode(cmap: CoefficientMap, codebooks) -> FeatureMapSet:
    """Coefficient map -> feature maps, one tcgen05 contraction per level (sparse_splat.py:183-199)."""
    import torch

    from .device import require_cuda, stream_ptr
    codebooks = list(codebooks)
    dev = require_cuda()
    W = cmap.device_tensor()
    h, w, nch = W.shape
    Dims = set()
    for level in cmap.levels:
        cb = codebooks[level]
        if cb.L != cmap.L:
            raise ValidationError(f"codebook L={cb.L} does not match coefficient map L={cmap.L}")
        Dims.add(cb.D)
    if len(Dims) > 1:
        raise ValidationError("codebooks of the decoded levels must share D")
    D = Dims.pop()
    out = torch.empty((len(cmap.levels), h, w, D), dtype=torch.float32, device=dev)
    lib = N.load()
    ws = torch.empty(max(int(lib.sf_decode_workspace_bytes(cmap.L, D)), 16), dtype=torch.uint8, device=dev)
    for b, level in enumerate(cmap.levels):
        atoms = torch.from_numpy(np.ascontiguousarray(codebooks[level].atoms, dtype=np.float32)).to(dev)
        N.check(lib.sf_decode(h * w, cmap.L, D, N.ptr(W[:, :, b * cmap.L:]), nch, N.ptr(atoms),
                              N.ptr(out[b]), N.ptr(ws), ws.numel(), stream_ptr()))
        del atoms
    torch.cuda.current_stream().synchronize()
    return FeatureMapSet(levels=cmap.levels, provenance="decoded-from-coefficients", dev=out)


@dataclass(frozen=True)
class StageTimings:
    """Milliseconds of the three query stages (sparse_splat.py:202-215), CUDA-event timed."""

    render_ms: float
    decode_ms: float
    post_ms: float

    @property
    def total_ms(self) -> float:
        return self.render_ms + self.decode_ms + self.post_ms

    def as_dict(self) -> dict:
        return {"render_ms": self.render_ms, "decode_ms": self.decode_ms, "post_ms": self.post_ms}


TIMING_CSV_HEADER = "scene_id,H,W,L,K,levels,render_ms,decode_ms,post_ms"


def timing_csv_row(scene_id: str, h: int, w: int, l: int, k: int, levels: int,
                   timings: StageTimings) -> str:
    return (f"{scene_id},{h},{w},{l},{k},{levels},"
            f"{timings.render_ms:.6f},{timings.decode_ms:.6f},{timings.post_ms:.6f}")


class QueryResult:
    """Everything one query produced (sparse_splat.py:229-240).

    ``coefficient_map`` and ``feature_maps`` are produced on demand (the
    serving path -- cli.py:136-154, server.py:186-203 -- never reads them),
    unless query_pipeline(..., features="eager") materialised them.
    """

    def __init__(self, query, level_maps, level, chosen, point, timings, cmap_thunk,
                 features: FeatureMapSet, mask=None, degenerate=None):
        self.query = query
        self.level_maps = level_maps
        self.level = level
        self.chosen = chosen
        self.point = point
        self.timings = timings
        self._cmap_thunk = cmap_thunk
        self._cmap = None
        self.feature_maps = features
        self.mask = mask            # segment(chosen).mask, computed in the same frame
        self.degenerate = degenerate

    @property
    def coefficient_map(self) -> CoefficientMap:
        if self._cmap is None:
            self._cmap = self._cmap_thunk()
        return self._cmap


def query_pipeline(scene, cam, query: QueryEmbedding, canonicals, *, window: int = 11,
                   level: int | None = None, tile_size: int = DEFAULT_TILE_SIZE, workers: int = 1,
                   instrument: bool = True, threshold: float = 0.5,
                   features: str = "lazy",
                   max_elements: int = DEFAULT_MAX_RENDER_ELEMENTS, engine=None) -> QueryResult:
    """Fused multilevel splat -> decode -> post-process (sparse_splat.py:243-297).

    One ``sf_render_frame``: the blend kernel also computes the per-level
    relevancy from the coefficient tile through the projected codebook
    P = atoms @ [q; canonicals]^T (fp64) -- exactly f.q = (W @ atoms).q --
    so the 512-d features are decoded only when asked for
    (``features="eager"`` decodes them inside the timed frame).
    ``max_elements`` (extension, default = the reference's fixed budget) lets
    configurations above 2^27 coefficient elements run; ``engine`` (extension)
    runs the frame on a given FrameEngine (its own workspace) on the current
    stream, so concurrent requests need not serialise on the scene's engine.
    """
    from .device import QuerySpec, device_scene
    cfg = scene.config
    W, H = int(cam.width), int(cam.height)
    levels = tuple(range(cfg.num_levels))
    if tile_size != DEFAULT_TILE_SIZE:
        raise ValidationError("the sm_100a kernels are specialised for 16x16 tiles")
    canon = np.asarray(canonicals, dtype=np.float64)
    if canon.ndim != 2 or canon.shape[0] < 1:
        raise ValidationError("at least one canonical D-vector is required")
    if canon.shape[1] != cfg.D or query.vector.shape[0] != cfg.D:
        raise ValidationError(
            f"dimension mismatch: features D={cfg.D}, query D={query.vector.shape[0]}, "
            f"canonicals D={canon.shape[1]}")
    if window < 1 or window % 2 == 0:
        raise ValidationError(f"filter window must be odd and >= 1, got {window}")
    # the reference cannot override the render budget here (sparse_splat.py:264);
    # the keyword is an extension whose default keeps that behaviour
    check_render_budget(W, H, len(levels) * cfg.L, max_elements)
    fixed = -1
    if level is not None:
        if level not in levels:
            raise ValidationError(f"level {level} was not rendered")
        fixed = levels.index(level)
    ds = device_scene(scene)
    if ds.bad_index:
        raise ValidationError("coefficient index >= L")
    eager = features == "eager"
    fused = bool(N.load().sf_decode_fused(len(levels), cfg.L, cfg.K, cfg.D))
    rel_fused = bool(N.load().sf_relevancy_fused(len(levels), cfg.L, cfg.K, canon.shape[0]))
    need_cmap = (eager and not fused) or not rel_fused
    eng = ds.engine if engine is None else engine  # serve.py: one engine + stream per concurrent request
    out = eng.allocate(W, H, levels, coeff_map=need_cmap, features=eager, query=True)
    spec = QuerySpec(query.vector, canon, window, fixed, threshold)
    eng.run(cam, levels, out, query=spec, timing=instrument, fetch_mask=True)
    st_i, st_f = out.host_stats()
    timings = None
    if instrument:
        r, d, p = out.stage_ms()
        timings = StageTimings(render_ms=r, decode_ms=d, post_ms=p)
    maps = tuple(RelevancyMap(query=query.name, level=lv, filtered=True, window=window,
                              dev=out.relevancy_filtered[b]) for b, lv in enumerate(levels))
    chosen_b = int(st_i[N.STAT_LEVEL])
    point = (int(st_i[N.STAT_ROW]), int(st_i[N.STAT_COL]))
    mask = out.mask_host.numpy().view(np.bool_)  # 0/1 bytes; the pinned buffer is this call's own

    if need_cmap:
        cm = CoefficientMap(L=cfg.L, K=cfg.K, levels=levels, dev=out.coeff_map)
        cmap_thunk = (lambda cm=cm: cm)
    else:
        cmap_thunk = (lambda: splat_multilevel(scene, cam))
    if eager:
        fms = FeatureMapSet(levels=levels, dev=out.features)
    else:
        holder = {}

        def _decode_lazy():
            if "cm" not in holder:
                holder["cm"] = res.coefficient_map
            return decode(holder["cm"], getattr(scene, "host_codebooks", None) or scene.codebooks).dev

        fms = FeatureMapSet(levels=levels, thunk=_decode_lazy)
    res = QueryResult(query=query.name, level_maps=maps, level=levels[chosen_b], chosen=maps[chosen_b],
                      point=point, timings=timings, cmap_thunk=cmap_thunk, features=fms, mask=mask,
                      degenerate=bool(st_i[N.STAT_DEGENERATE]))
    return res


def query_sweep(scene, cam, queries, canonicals, *, window: int = 11, threshold: float = 0.5,
                tile_size: int = DEFAULT_TILE_SIZE,
                max_elements: int = DEFAULT_MAX_RENDER_ELEMENTS, engine=None) -> list:
    """Many text prompts over one view (BASELINE config E; extension).

    The reference answers each prompt with its own query_pipeline call
    (sparse_splat.py:243-297), re-rendering the frame every time.  Here the
    multilevel coefficient map is rendered once and every prompt runs only
    its post: relevancy from the map through its projected codebook (fp64),
    mean filter, select_level / localize / segment (sf_query_sweep).  Each
    returned QueryResult equals query_pipeline(scene, cam, q, canonicals,
    window=window, threshold=threshold) for its prompt (automatic level;
    timings None)."""
    from .device import device_scene
    cfg = scene.config
    W, H = int(cam.width), int(cam.height)
    levels = tuple(range(cfg.num_levels))
    if tile_size != DEFAULT_TILE_SIZE:
        raise ValidationError("the sm_100a kernels are specialised for 16x16 tiles")
    queries = list(queries)
    canon = np.asarray(canonicals, dtype=np.float64)
    if canon.ndim != 2 or canon.shape[0] < 1:
        raise ValidationError("at least one canonical D-vector is required")
    for q in queries:
        if canon.shape[1] != cfg.D or q.vector.shape[0] != cfg.D:
            raise ValidationError(
                f"dimension mismatch: features D={cfg.D}, query D={q.vector.shape[0]}, "
                f"canonicals D={canon.shape[1]}")
    if window < 1 or window % 2 == 0:
        raise ValidationError(f"filter window must be odd and >= 1, got {window}")
    check_render_budget(W, H, len(levels) * cfg.L, max_elements)
    ds = device_scene(scene)
    if ds.bad_index:
        raise ValidationError("coefficient index >= L")
    eng = ds.engine if engine is None else engine
    out = eng.allocate(W, H, levels, coeff_map=True, mask=False)
    prompts = np.stack([q.vector for q in queries]) if queries else np.zeros((0, cfg.D))
    filt, masks, st_i, _ = eng.sweep(cam, levels, out, prompts, canon, window=window, threshold=threshold)
    host_masks = masks.cpu().numpy().view(np.bool_)
    cm = CoefficientMap(L=cfg.L, K=cfg.K, levels=levels, dev=out.coeff_map)
    holder = {}

    def _decode_lazy():
        if "f" not in holder:
            holder["f"] = decode(cm, getattr(scene, "host_codebooks", None) or scene.codebooks).dev
        return holder["f"]

    results = []
    for i, q in enumerate(queries):
        maps = tuple(RelevancyMap(query=q.name, level=lv, filtered=True, window=window, dev=filt[i, b])
                     for b, lv in enumerate(levels))
        b = int(st_i[i][N.STAT_LEVEL])
        results.append(QueryResult(
            query=q.name, level_maps=maps, level=levels[b], chosen=maps[b],
            point=(int(st_i[i][N.STAT_ROW]), int(st_i[i][N.STAT_COL])), timings=None,
            cmap_thunk=(lambda cm=cm: cm), features=FeatureMapSet(levels=levels, thunk=_decode_lazy),
            mask=host_masks[i], degenerate=bool(st_i[i][N.STAT_DEGENERATE])))
    return results


@dataclass
class StreamResult:
    """What one streamed query returns (the serving fields of QueryResult)."""

    query: str
    level: int
    point: tuple
    mask: np.ndarray      # (H, W) bool, this frame's own pinned host copy
    degenerate: bool


class QueryStream:
    """Pipelined text queries over one scene at one image size (extension).

    The reference answers one query_pipeline call at a time
    (sparse_splat.py:243-297).  submit() enqueues a frame and returns at once:
    the query vector is copied from pinned host memory, the frame runs
    query_pipeline's work on the GPU (features="eager" also decodes the 3 x D
    feature maps), and the mask and statistics are copied back into pinned
    host buffers of that frame.  result() waits for that frame only.  Frames
    overlap on the GPU (device.FramePipeline): frame i+1's projection / sort /
    binning run under frame i's blend.  The canonicals are the stream's
    constant and are uploaded once.  A frame whose pairs overflowed the pair
    buffer is re-run through query_pipeline (which grows it) inside result().
    """

    def __init__(self, scene, width: int, height: int, canonicals, *, window: int = 11, threshold: float = 0.5,
                 features: str = "lazy"):
        import torch

        from .device import FramePipeline, device_scene
        cfg = scene.config
        canon = np.asarray(canonicals, dtype=np.float64)
        if canon.ndim != 2 or canon.shape[0] < 1 or canon.shape[1] != cfg.D:
            raise ValidationError("canonicals must be a non-empty (n, D) array")
        if window < 1 or window % 2 == 0:
            raise ValidationError(f"filter window must be odd and >= 1, got {window}")
        self.scene, self.W, self.H = scene, int(width), int(height)
        self.canonicals, self.window, self.threshold = canon, int(window), float(threshold)
        self.levels = tuple(range(cfg.num_levels))
        self.features = features
        self.ds = device_scene(scene)
        if self.ds.bad_index:
            raise ValidationError("coefficient index >= L")
        eager = features == "eager"
        fused = bool(N.load().sf_decode_fused(len(self.levels), cfg.L, cfg.K, cfg.D))
        rel_fused = bool(N.load().sf_relevancy_fused(len(self.levels), cfg.L, cfg.K, canon.shape[0]))
        need_cmap = (eager and not fused) or not rel_fused
        self.pipe = FramePipeline(self.ds, self.W, self.H, self.levels, coeff_map=need_cmap, features=eager,
                                  query=True)
        self.canon_dev = torch.from_numpy(canon).to(self.ds.device)
        self._began = False

    def submit(self, cam, query: QueryEmbedding):
        import torch

        from .device import QuerySpec
        if (int(cam.width), int(cam.height)) != (self.W, self.H):
            raise ValidationError("camera size differs from the stream's image size")
        if query.vector.shape[0] != self.scene.config.D:
            raise ValidationError("query dimension mismatch")
        if not self._began:
            self.pipe.begin()
            self._began = True
        hq = torch.from_numpy(np.ascontiguousarray(query.vector, dtype=np.float64)).pin_memory()
        rs = self.pipe.render[self.pipe.k % 2]
        with torch.cuda.stream(rs):
            qd = hq.to(self.ds.device, non_blocking=True)
        spec = QuerySpec(query.vector, self.canonicals, self.window, -1, self.threshold)
        out = self.pipe.enqueue(cam, self.levels, query=spec, qdev=(qd, self.canon_dev))
        hm = torch.empty((self.H, self.W), dtype=torch.uint8, pin_memory=True)
        hi = torch.empty(16, dtype=torch.int64, pin_memory=True)
        with torch.cuda.stream(rs):
            hm.copy_(out.mask, non_blocking=True)
            hi.copy_(out.stats_i64, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(rs)
        return (ev, hm, hi, hq, qd, cam, query)

    def result(self, handle) -> StreamResult:
        ev, hm, hi, _, _, cam, query = handle
        ev.synchronize()
        st = hi.numpy()
        if not int(st[N.STAT_OVERFLOW]):
            N.check_fixups(st, cam.width, cam.height)
        if int(st[N.STAT_OVERFLOW]):
            r = query_pipeline(self.scene, cam, query, self.canonicals, window=self.window,
                               threshold=self.threshold, instrument=False, features=self.features,
                               max_elements=1 << 62)
            for e in self.pipe.engines:
                e.pair_capacity = max(e.pair_capacity, self.ds.engine.pair_capacity)
            return StreamResult(query.name, r.level, r.point, r.mask, bool(r.degenerate))
        return StreamResult(query.name, self.levels[int(st[N.STAT_LEVEL])],
                            (int(st[N.STAT_ROW]), int(st[N.STAT_COL])), hm.numpy().view(np.bool_),
                            bool(st[N.STAT_DEGENERATE]))

    def close(self):
        if self._began:
            self.pipe.end()
            self._began = False
