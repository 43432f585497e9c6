"""Relevancy scoring and post-processing (drop-in for splatfield/query.py).

    score = min over canonicals c of sigmoid(f.q - f.c)       query.py:65-84

Raw dot products, no normalisation (the reference's definition).  Every
function runs on the GPU (sf_relevancy_* / sf_mean_filter /
sf_select_segment); ``RelevancyMap.data`` is a float64 numpy view that
materialises from the device tensor on first access.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import ValidationError


@dataclass(frozen=True)
class QueryEmbedding:
    """A named query vector in the scene's feature space (query.py:22-37)."""

    name: str
    vector: np.ndarray
    canonical_set_id: str = "default"

    def __post_init__(self):
        v = np.asarray(self.vector, dtype=np.float64)
        object.__setattr__(self, "vector", v)
        if v.ndim != 1:
            raise ValidationError("query vector must be 1-D")
        if not np.all(np.isfinite(v)):
            raise ValidationError("query vector must be finite")


class RelevancyMap:
    """H x W score grid plus provenance (query.py:39-52); device-backed."""

    def __init__(self, data=None, query: str = "", level: int = 0, filtered: bool = False,
                 window: int = 1, *, dev=None):
        self.query = query
        self.level = level
        self.filtered = filtered
        self.window = window
        self.dev = dev
        self._data = None
        if dev is None:
            d = np.asarray(data, dtype=np.float64)
            if d.ndim != 2:
                raise ValidationError("relevancy map must be 2-D")
            self._data = d
        elif dev.dim() != 2:
            raise ValidationError("relevancy map must be 2-D")

    @property
    def data(self) -> np.ndarray:
        if self._data is None:
            self._data = self.dev.cpu().numpy()
        return self._data

    @data.setter
    def data(self, value):
        self._data = np.asarray(value, dtype=np.float64)
        self.dev = None

    @property
    def shape(self):
        return tuple(self.dev.shape) if self.dev is not None else self._data.shape

    def device_tensor(self):
        import torch

        from .device import require_cuda
        if self.dev is None:
            self.dev = torch.from_numpy(np.ascontiguousarray(self._data)).to(require_cuda())
        return self.dev


@dataclass
class SegmentationResult:
    mask: np.ndarray
    threshold: float
    degenerate: bool


def relevancy_map(features, q: QueryEmbedding, canonicals, *, level: int = 0) -> RelevancyMap:
    """Per-pixel min-over-canonicals pairwise softmax score (query.py:65-84)."""
    import torch

    from .device import require_cuda, stream_ptr
    if isinstance(features, torch.Tensor):
        f = features
    else:
        f = np.asarray(features)
        if f.dtype not in (np.float32, np.float64):
            f = f.astype(np.float64)
    if f.ndim != 3:
        raise ValidationError("features must be H x W x D")
    h, w, d = (int(s) for s in f.shape)
    canon = np.asarray(canonicals, dtype=np.float64)
    if canon.ndim != 2 or canon.shape[0] < 1:
        raise ValidationError("at least one canonical D-vector is required")
    if canon.shape[1] != d or q.vector.shape[0] != d:
        raise ValidationError(
            f"dimension mismatch: features D={d}, query D={q.vector.shape[0]}, "
            f"canonicals D={canon.shape[1]}")
    dev = require_cuda()
    ft = f if isinstance(f, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(f))
    ft = ft.to(dev).contiguous()
    if ft.dtype not in (torch.float32, torch.float64):
        ft = ft.double()
    qt = torch.from_numpy(np.ascontiguousarray(q.vector)).to(dev)
    ct = torch.from_numpy(np.ascontiguousarray(canon)).to(dev)
    out = torch.empty((h, w), dtype=torch.float64, device=dev)
    lib = N.load()
    fn = lib.sf_relevancy_f32 if ft.dtype == torch.float32 else lib.sf_relevancy_f64
    N.check(fn(h * w, d, N.ptr(ft), N.ptr(qt), N.ptr(ct), canon.shape[0], N.ptr(out), stream_ptr()))
    return RelevancyMap(query=q.name, level=level, dev=out)


def mean_filter(m: RelevancyMap, window: int) -> RelevancyMap:
    """Edge-clamped box filter; window 1 is the identity (query.py:87-108)."""
    import torch

    from .device import stream_ptr
    if window < 1 or window % 2 == 0:
        raise ValidationError(f"filter window must be odd and >= 1, got {window}")
    src = m.device_tensor().contiguous()
    if window == 1:
        return RelevancyMap(query=m.query, level=m.level, filtered=True, window=1, dev=src.clone())
    h, w = src.shape
    out = torch.empty_like(src)
    tmp = torch.empty_like(src)
    N.check(N.load().sf_mean_filter(h, w, N.ptr(src), window, N.ptr(out), N.ptr(tmp),
                                    tmp.numel() * 8, stream_ptr()))
    return RelevancyMap(query=m.query, level=m.level, filtered=True, window=window, dev=out)


def _select(maps, fixed_level: int, threshold: float, want_mask: bool):
    import torch

    from .device import require_cuda, stream_ptr
    dev = require_cuda()
    ts = [m.device_tensor() for m in maps]
    shapes = {tuple(t.shape) for t in ts}
    if len(shapes) != 1:
        # differently sized maps: reduce one at a time (selection only compares maxima)
        return None
    h, w = ts[0].shape
    stacked = torch.stack(ts).contiguous() if len(ts) > 1 else ts[0].reshape(1, h, w).contiguous()
    lib = N.load()
    nbytes = lib.sf_select_segment_workspace_bytes(len(ts), h, w)
    ws = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=dev)
    # k_finalize_select writes stats_i64[8 + m] and stats_f64[8 + n + m] per map m
    n = len(ts)
    st_i = torch.zeros(max(16, 8 + n), dtype=torch.int64, device=dev)
    st_f = torch.zeros(8 + 2 * n, dtype=torch.float64, device=dev)
    mask = torch.empty((h, w), dtype=torch.uint8, device=dev) if want_mask else None
    N.check(lib.sf_select_segment(len(ts), h, w, N.ptr(stacked), fixed_level, float(threshold),
                                  N.ptr(mask), N.ptr(st_i), N.ptr(st_f), N.ptr(ws), ws.numel(),
                                  stream_ptr()))
    return st_i.cpu().numpy(), st_f.cpu().numpy(), mask


def select_level(maps):
    """Level whose map has the highest maximum; ties to the lowest (query.py:111-118)."""
    maps = list(maps)
    if not maps:
        raise ValidationError("at least one level map is required")
    res = _select(maps, -1, 0.5, False)
    if res is None:
        maxima = []
        for m in maps:
            st_i, st_f, _ = _select([m], 0, 0.5, False)
            maxima.append(st_f[N.STATF_MAX])
        level = int(np.argmax(np.array(maxima)))
    else:
        level = int(res[0][N.STAT_LEVEL])
    return level, maps[level]


def localize(m: RelevancyMap):
    """(row, col) of the maximum; ties to smallest row, then column (query.py:121-126)."""
    if int(np.prod(m.shape)) == 0:
        raise ValidationError("cannot localize an empty map")
    st_i, _, _ = _select([m], 0, 0.5, False)
    return int(st_i[N.STAT_ROW]), int(st_i[N.STAT_COL])


def segment(m: RelevancyMap, threshold: float = 0.5) -> SegmentationResult:
    """Mask of min-max normalised scores above ``threshold`` (query.py:136-145)."""
    if int(np.prod(m.shape)) == 0:
        return SegmentationResult(mask=np.zeros(m.shape, dtype=bool), threshold=threshold,
                                  degenerate=True)
    st_i, _, mask = _select([m], 0, threshold, True)
    degenerate = bool(st_i[N.STAT_DEGENERATE])
    return SegmentationResult(mask=mask.cpu().numpy().astype(bool), threshold=threshold,
                              degenerate=degenerate)


def iou(a, b) -> float:
    """Intersection over union of two boolean masks; empty vs empty is 1 (query.py:177-186)."""
    a = np.asarray(a, dtype=bool)
    b = np.asarray(b, dtype=bool)
    if a.shape != b.shape:
        raise ValidationError(f"mask shapes differ: {a.shape} vs {b.shape}")
    union = np.logical_or(a, b).sum()
    if union == 0:
        return 1.0
    return float(np.logical_and(a, b).sum() / union)
