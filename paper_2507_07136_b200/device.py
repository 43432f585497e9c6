"""Device plumbing: resident scenes, workspaces and the per-frame launcher.

PyTorch is used only for device memory, streams and copies.  All compute
is the native library (``_native``); this module marshals pointers into the
C structs of include/splatfield_b200.h.

* ``DeviceScene`` -- the scene uploaded once to HBM in id order (the
  canonical order tie-break of projection.py:396 then reduces to a stable
  depth sort).  Cached per scene object (scenes are immutable by contract).
* ``FrameEngine`` -- owns the per-shape workspace (grown on pair-buffer
  overflow) and launches ``sf_render_frame`` on the current torch stream.
"""

from __future__ import annotations

import ctypes
import threading
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import SplatfieldError, ValidationError

try:
    import torch
except ImportError as exc:  # pragma: no cover
    raise SplatfieldError("PyTorch is required for device memory management") from exc


def require_cuda() -> "torch.device":
    if not torch.cuda.is_available():
        raise SplatfieldError("a CUDA device is required: the sm_100a path has no CPU fallback")
    N.load()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def camera_struct(cam) -> N.SfCamera:
    c = N.SfCamera()
    R = np.ascontiguousarray(np.asarray(cam.rotation, dtype=np.float64)).reshape(9)
    t = np.asarray(cam.translation, dtype=np.float64).reshape(3)
    for i in range(9):
        c.R[i] = float(R[i])
    for i in range(3):
        c.t[i] = float(t[i])
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.near_plane = float(getattr(cam, "near", 0.01))
    c.width, c.height = int(cam.width), int(cam.height)
    return c


def _dev(a: np.ndarray, device, dtype=None) -> "torch.Tensor":
    a = np.ascontiguousarray(a if dtype is None else a.astype(dtype, copy=False))
    return torch.from_numpy(a).to(device, non_blocking=False)


class DeviceScene:
    """A scene resident on the GPU, rows ordered by id (SfScene)."""

    def __init__(self, scene, device=None):
        device = device or require_cuda()
        cfg = scene.config
        g = int(np.asarray(scene.positions).shape[0])
        ids = np.asarray(scene.ids, dtype=np.int64).reshape(g)
        if g > 1 and np.any(ids[1:] < ids[:-1]):
            perm = np.argsort(ids, kind="stable")
        else:
            perm = None
        sel = (lambda a: a) if perm is None else (lambda a: a[perm])
        ci = np.asarray(scene.coeff_indices, dtype=np.uint16).reshape(cfg.num_levels, g, cfg.K)
        cv = np.asarray(scene.coeff_values, dtype=np.float32).reshape(cfg.num_levels, g, cfg.K)
        if perm is not None:
            ci, cv = ci[:, perm], cv[:, perm]
        self.device = device
        self.num_gaussians = g
        self.config = cfg
        self.bad_index = bool(g and np.any(ci >= cfg.L))
        self.positions = _dev(sel(np.asarray(scene.positions)).reshape(g, 3), device, np.float32)
        self.rotations = _dev(sel(np.asarray(scene.rotations)).reshape(g, 4), device, np.float32)
        self.scales = _dev(sel(np.asarray(scene.scales)).reshape(g, 3), device, np.float32)
        self.opacities = _dev(sel(np.asarray(scene.opacities)).reshape(g), device, np.float32)
        self.coeff_indices = _dev(np.ascontiguousarray(ci).view(np.int16), device)
        self.coeff_values = _dev(cv, device)
        self.ids = _dev(sel(ids), device)
        self.orig_rows = None if perm is None else _dev(perm.astype(np.int64), device)
        atoms = np.stack([np.asarray(cb.atoms, dtype=np.float32) for cb in scene.codebooks]) \
            if len(scene.codebooks) else np.zeros((0, cfg.L, cfg.D), np.float32)
        self.codebooks = _dev(atoms, device)
        self.host_codebooks = tuple(scene.codebooks)
        self.colors = _dev(sel(np.asarray(scene.colors)).reshape(g, 3), device, np.float32)
        self.struct = N.SfScene(
            g, cfg.num_levels, cfg.L, cfg.K, cfg.D,
            N.ptr(self.positions), N.ptr(self.rotations), N.ptr(self.scales), N.ptr(self.opacities),
            N.ptr(self.coeff_indices), N.ptr(self.coeff_values), N.ptr(self.ids), N.ptr(self.codebooks))
        self._engine = None
        self._lock = threading.Lock()

    @classmethod
    def from_device(cls, config, tensors: dict, host_codebooks, device) -> "DeviceScene":
        """A resident scene from SoA tensors already in HBM (io.load_scene_device):
        positions, rotations, scales, opacities, colors, coeff_indices (int16 view of
        u16), coeff_values, codebooks; rows are in id order (ids = arange)."""
        self = cls.__new__(cls)
        g = int(tensors["positions"].shape[0])
        self.device = device
        self.num_gaussians = g
        self.config = config
        self.bad_index = False  # checked by the unpack kernel (SF_LSV2_INDEX_RANGE)
        for k in ("positions", "rotations", "scales", "opacities", "colors", "coeff_indices", "coeff_values",
                  "codebooks"):
            setattr(self, k, tensors[k])
        self.ids = torch.arange(g, dtype=torch.int64, device=device)
        self.orig_rows = None
        self.host_codebooks = tuple(host_codebooks)
        self.struct = N.SfScene(
            g, config.num_levels, config.L, config.K, config.D,
            N.ptr(self.positions), N.ptr(self.rotations), N.ptr(self.scales), N.ptr(self.opacities),
            N.ptr(self.coeff_indices), N.ptr(self.coeff_values), N.ptr(self.ids), N.ptr(self.codebooks))
        self._engine = None
        self._lock = threading.Lock()
        return self

    @property
    def engine(self) -> "FrameEngine":
        if self._engine is None:
            self._engine = FrameEngine(self)
        return self._engine


_scene_cache: dict = {}
_cache_lock = threading.Lock()


_SCENE_ARRAYS = ("positions", "rotations", "scales", "opacities", "colors", "coeff_indices", "coeff_values", "ids")


def _fingerprint(scene) -> tuple:
    """Identity of a scene's arrays and codebooks (object, data pointer, shape,
    dtype): reassigning any of them re-uploads.  In-place edits keep the
    identity -- call ``invalidate(scene)`` after those (the reference treats
    scenes as immutable; so does the serving path).  ~10 us per call."""
    parts = []
    for name in _SCENE_ARRAYS:
        a = getattr(scene, name, None)
        if isinstance(a, np.ndarray):
            parts.append((name, id(a), a.__array_interface__["data"][0], a.shape, a.dtype.str))
        else:
            parts.append((name, id(a)))
    cbs = tuple(getattr(scene, "codebooks", ()))
    for cb in cbs:
        a = cb.atoms
        parts.append((id(cb), id(a), a.__array_interface__["data"][0] if isinstance(a, np.ndarray) else 0))
    return tuple(parts) + ((len(cbs), id(scene.config)),)


def invalidate(scene) -> None:
    """Drop the cached device copy of ``scene`` (after editing its arrays in place)."""
    with _cache_lock:
        _scene_cache.pop(id(scene), None)


def device_scene(scene) -> DeviceScene:
    """Upload ``scene`` once and return its cached device copy (re-uploaded
    when the scene's arrays or codebooks changed, see ``_fingerprint``)."""
    if isinstance(scene, DeviceScene):
        return scene
    key = id(scene)
    fp = _fingerprint(scene)
    with _cache_lock:
        hit = _scene_cache.get(key)
        if hit is not None and hit[0]() is scene and hit[2] == fp:
            return hit[1]
    ds = DeviceScene(scene)
    with _cache_lock:
        try:
            ref = weakref.ref(scene, lambda _r, k=key: _scene_cache.pop(k, None))
        except TypeError:  # not weak-referenceable: cache without eviction hook
            ref = (lambda s=scene: s)
        _scene_cache[key] = (ref, ds, fp)
    return ds


@dataclass
class QuerySpec:
    vector: np.ndarray          # (D,) float64
    canonicals: np.ndarray      # (n, D) float64
    window: int = 11
    fixed_level: int = -1       # block index or -1
    threshold: float = 0.5


@dataclass
class FrameOutputs:
    """Device tensors of one frame (views valid until the next run with reuse)."""

    width: int
    height: int
    levels: tuple
    coeff_map: "torch.Tensor | None"
    final_t: "torch.Tensor | None"
    features: "torch.Tensor | None"
    relevancy_raw: "torch.Tensor | None"
    relevancy_filtered: "torch.Tensor | None"
    mask: "torch.Tensor | None"
    stats_i64: "torch.Tensor"
    stats_f64: "torch.Tensor"
    events: tuple | None = None

    def host_stats(self):
        if getattr(self, "_host", None) is None:
            self._host = (self.stats_i64.cpu().numpy(), self.stats_f64.cpu().numpy())
            if int(self._host[0][N.STAT_OVERFLOW]) == 0:
                N.check_fixups(self._host[0], self.width, self.height)
        return self._host

    def stage_ms(self):
        if not self.events:
            return None
        lib = N.load()
        e = self.events
        return (lib.sf_event_elapsed_ms(e[0], e[1]), lib.sf_event_elapsed_ms(e[1], e[2]),
                lib.sf_event_elapsed_ms(e[2], e[3]))

    def blend_ms(self):
        """Time of the blend kernel alone (it includes the decode when it is fused)."""
        if not self.events:
            return None
        return N.load().sf_event_elapsed_ms(self.events[4], self.events[1])


class FrameEngine:
    """Launches frames of one DeviceScene; owns a growable workspace."""

    def __init__(self, dscene: DeviceScene):
        self.ds = dscene
        g = dscene.num_gaussians
        self.pair_capacity = max(1 << 16, 6 * g)
        self._ws = None
        self._ws_key = None
        # re-entrant: render_dense holds it across its channel passes, which
        # reuse the first pass's tile lists (SfFrame.reuse_lists)
        self._lock = threading.RLock()
        self._events = None
        self._handoff = None
        self._plans = {}

    def channel_plan(self, levels) -> "torch.Tensor":
        """Cached per-row scatter plan of a level selection (a scene constant)."""
        key = tuple(int(x) for x in levels)
        plan = self._plans.get(key)
        if plan is None:
            lib = N.load()
            cfg = self.ds.config
            nbytes = int(lib.sf_channel_plan_bytes(self.ds.num_gaussians, len(key), cfg.K))
            plan = torch.empty(nbytes, dtype=torch.uint8, device=self.ds.device)
            lv = (ctypes.c_int32 * len(key))(*key)
            N.check(lib.sf_pack_channels(ctypes.byref(self.ds.struct), ctypes.cast(lv, ctypes.c_void_p), len(key),
                                         N.ptr(plan), nbytes, stream_ptr()))
            self._plans[key] = plan
        return plan

    def decode_image(self, levels):
        """Cached codebook image of the fused decode for a level selection (or None)."""
        key = ("dec",) + tuple(int(x) for x in levels)
        if key not in self._plans:
            lib = N.load()
            cfg = self.ds.config
            nbytes = int(lib.sf_decode_image_bytes(len(levels), cfg.L, cfg.K, cfg.D))
            img = None
            if nbytes:
                img = torch.empty(nbytes, dtype=torch.uint8, device=self.ds.device)
                lv = (ctypes.c_int32 * len(levels))(*key[1:])
                N.check(lib.sf_pack_decode_image(ctypes.byref(self.ds.struct), ctypes.cast(lv, ctypes.c_void_p),
                                                 len(levels), N.ptr(img), nbytes, stream_ptr()))
            self._plans[key] = img
        return self._plans[key]

    def workspace(self, W: int, H: int, n_levels: int, L: int | None = None, K: int | None = None) -> "torch.Tensor":
        cfg = self.ds.config
        L = cfg.L if L is None else L
        K = cfg.K if K is None else K
        key = (W, H, n_levels, L, K, self.pair_capacity)
        if self._ws is None or self._ws_key != key:
            nbytes = ctypes.c_size_t(0)
            N.check(N.load().sf_frame_workspace_bytes(self.ds.num_gaussians, W, H, n_levels, L,
                                                      K, cfg.D, self.pair_capacity,
                                                      ctypes.byref(nbytes)))
            if self._ws is None or self._ws.numel() < nbytes.value:
                self._ws = None
                self._ws = torch.empty(nbytes.value, dtype=torch.uint8, device=self.ds.device)
            self._ws_key = key
        return self._ws

    def allocate(self, W, H, levels, *, coeff_map=True, final_t=False, features=False,
                 query=False, mask=True) -> FrameOutputs:
        cfg = self.ds.config
        dev = self.ds.device
        nl = len(levels)
        f32, f64 = torch.float32, torch.float64
        return FrameOutputs(
            W, H, tuple(levels),
            torch.empty((H, W, nl * cfg.L), dtype=f32, device=dev) if coeff_map else None,
            torch.empty((H, W), dtype=f32, device=dev) if final_t else None,
            torch.empty((nl, H, W, cfg.D), dtype=f32, device=dev) if features else None,
            torch.empty((nl, H, W), dtype=f64, device=dev) if query else None,
            torch.empty((nl, H, W), dtype=f64, device=dev) if query else None,
            torch.empty((H, W), dtype=torch.uint8, device=dev) if (query and mask) else None,
            torch.zeros(16, dtype=torch.int64, device=dev),
            torch.zeros(8 + 2 * 8, dtype=torch.float64, device=dev),
        )

    def enqueue(self, cam, levels, out: FrameOutputs, *, query: QuerySpec | None = None,
                early_exit: bool = True, qdev=None, timing: bool = False, band=None, prep_stream=None,
                dense=None, reuse_lists: bool = False):
        """Launch one frame on the current stream (no host synchronisation).

        ``band=(y0, y1)``: tile-band mode -- only pixel rows [y0, y1) are owned
        (SfFrame.band_y0/1); ``None`` renders the whole image.
        ``prep_stream``: run projection / sort / binning there instead
        (sf_render_frame_split); the rest stays on the current stream.
        ``dense=(plan, C)``: blend C <= 16 dense channels per Gaussian from a
        ready scatter plan (render_dense) instead of the scene's coefficients.
        ``reuse_lists``: skip projection and binning and blend with the lists
        the previous frame of this workspace built (same camera and shape)."""
        cfg = self.ds.config
        camc = camera_struct(cam)
        W, H = camc.width, camc.height
        lv = (ctypes.c_int32 * len(levels))(*[int(x) for x in levels])
        sst = self.ds.struct
        if dense is not None:
            plan, cc = dense
            s0 = self.ds.struct
            sst = N.SfScene(s0.num_gaussians, 1, cc, cc, s0.D, s0.positions, s0.rotations, s0.scales,
                            s0.opacities, s0.coeff_indices, s0.coeff_values, s0.ids, s0.codebooks)
            ws = self.workspace(W, H, 1, cc, cc)
        else:
            ws = self.workspace(W, H, len(levels))
        fr = N.SfFrame()
        fr.host_levels = ctypes.cast(lv, ctypes.c_void_p)
        fr.n_levels = len(levels)
        fr.early_exit = 1 if early_exit else 0
        fr.pair_capacity = self.pair_capacity
        fr.coeff_map = N.ptr(out.coeff_map)
        fr.final_t = N.ptr(out.final_t)
        fr.features = N.ptr(out.features)
        fr.relevancy_raw = N.ptr(out.relevancy_raw)
        fr.relevancy_filtered = N.ptr(out.relevancy_filtered)
        fr.mask = N.ptr(out.mask)
        fr.stats_i64 = N.ptr(out.stats_i64)
        fr.stats_f64 = N.ptr(out.stats_f64)
        if band is not None:
            fr.band_y0, fr.band_y1 = int(band[0]), int(band[1])
        fr.reuse_lists = 1 if reuse_lists else 0
        if dense is not None:
            fr.chan_by_row = N.ptr(dense[0])
        elif len(levels) * cfg.K <= 16:
            fr.chan_by_row = N.ptr(self.channel_plan(levels))
        if dense is None and out.features is not None:
            fr.dec_image = N.ptr(self.decode_image(levels))
        if timing:
            if self._events is None:
                lib = N.load()
                self._events = tuple(lib.sf_event_create() for _ in range(5))
            for i in range(5):
                fr.events[i] = self._events[i]
            out.events = self._events
        qs = None
        keep = None
        if query is not None:
            if qdev is None:
                # pinned staging + async copies: the launches need not wait for them
                hq = torch.from_numpy(np.ascontiguousarray(query.vector, dtype=np.float64)).pin_memory()
                hc = torch.from_numpy(np.ascontiguousarray(query.canonicals, dtype=np.float64)).pin_memory()
                qdev = (hq.to(self.ds.device, non_blocking=True), hc.to(self.ds.device, non_blocking=True), hq, hc)
            keep = qdev
            qs = N.SfQuery(N.ptr(qdev[0]), N.ptr(qdev[1]), int(query.canonicals.shape[0]),
                           int(query.window), int(query.fixed_level), float(query.threshold))
        lib = N.load()
        if prep_stream is None:
            rc = lib.sf_render_frame(ctypes.byref(sst), ctypes.byref(camc),
                                     ctypes.byref(qs) if qs is not None else None, ctypes.byref(fr),
                                     N.ptr(ws), ws.numel(), stream_ptr())
        else:
            if self._handoff is None:
                self._handoff = lib.sf_event_create()
            rc = lib.sf_render_frame_split(ctypes.byref(sst), ctypes.byref(camc),
                                           ctypes.byref(qs) if qs is not None else None, ctypes.byref(fr),
                                           N.ptr(ws), ws.numel(), ctypes.c_void_p(prep_stream.cuda_stream),
                                           stream_ptr(), self._handoff)
        N.check(rc)
        return keep

    def run(self, cam, levels, out: FrameOutputs, *, fetch_mask: bool = False, **kw) -> FrameOutputs:
        """Launch and synchronise once; grows the pair buffer and re-runs on overflow.

        The statistics (and with ``fetch_mask`` the mask) come back through
        pinned host buffers with asynchronous copies behind the frame."""
        with self._lock:
            for _ in range(4):
                keep = self.enqueue(cam, levels, out, **kw)
                hi = torch.empty(out.stats_i64.shape, dtype=out.stats_i64.dtype, pin_memory=True)
                hf = torch.empty(out.stats_f64.shape, dtype=out.stats_f64.dtype, pin_memory=True)
                hi.copy_(out.stats_i64, non_blocking=True)
                hf.copy_(out.stats_f64, non_blocking=True)
                if fetch_mask and out.mask is not None:
                    hm = torch.empty(out.mask.shape, dtype=out.mask.dtype, pin_memory=True)
                    hm.copy_(out.mask, non_blocking=True)
                    out.mask_host = hm
                torch.cuda.current_stream().synchronize()
                out._host = (hi.numpy(), hf.numpy())
                st = out._host[0]
                del keep
                if int(st[N.STAT_OVERFLOW]) == 0:
                    N.check_fixups(st, out.width, out.height)
                    return out
                self.pair_capacity = int(int(st[N.STAT_PAIRS]) * 1.25) + 1024
            raise SplatfieldError("pair buffer overflow persisted after growing")


    def tile_lists(self, W: int, H: int, n_levels: int, n_pairs: int):
        """The last frame's per-tile lists (offsets, scene rows) from its
        workspace, as host int64 arrays (parity checks of the frame binning)."""
        cfg = self.ds.config
        ws = self.workspace(W, H, n_levels)
        n_tiles = ((W + 15) // 16) * ((H + 15) // 16)
        offs = torch.empty(n_tiles + 1, dtype=torch.int32, device=self.ds.device)
        rows = torch.empty(max(1, n_pairs), dtype=torch.int32, device=self.ds.device)
        N.check(N.load().sf_frame_tile_lists(self.ds.num_gaussians, W, H, n_levels, cfg.L, cfg.K, cfg.D,
                                             self.pair_capacity, N.ptr(ws), ws.numel(), N.ptr(offs), N.ptr(rows),
                                             int(rows.numel()), stream_ptr()))
        o = offs.cpu().numpy().view(np.uint32).astype(np.int64)
        r = rows.cpu().numpy().view(np.uint32).astype(np.int64)[:int(o[-1])]
        return o, r

    def sweep(self, cam, levels, out: FrameOutputs, prompts: np.ndarray, canonicals: np.ndarray, *,
              window: int = 11, threshold: float = 0.5, band=None):
        """Render ``out.coeff_map`` once, then run the query post of every
        prompt over it (sf_query_sweep); returns device tensors
        (filtered (n, levels, H, W) fp64, masks (n, H, W) u8, stats_i64 (n, 16),
        stats_f64 (n, 8 + 2 levels)) and the host statistics, after one sync.
        ``band=(y0, y1)``: tile-band mode (only those rows are owned; the
        statistics cover them and the masks are written there)."""
        cfg = self.ds.config
        dev = self.ds.device
        n, nl = int(prompts.shape[0]), len(levels)
        W, H = int(cam.width), int(cam.height)
        hp = torch.from_numpy(np.ascontiguousarray(prompts, dtype=np.float64)).pin_memory()
        hc = torch.from_numpy(np.ascontiguousarray(canonicals, dtype=np.float64)).pin_memory()
        filt = torch.empty((n, nl, H, W), dtype=torch.float64, device=dev)
        raw = torch.empty((n, nl, H, W), dtype=torch.float64, device=dev)
        masks = torch.empty((n, H, W), dtype=torch.uint8, device=dev)
        si = torch.empty((max(n, 1), 16), dtype=torch.int64, device=dev)
        sf = torch.empty((max(n, 1), 8 + 2 * nl), dtype=torch.float64, device=dev)
        camc = camera_struct(cam)
        lv = (ctypes.c_int32 * nl)(*[int(x) for x in levels])
        lib = N.load()
        with self._lock:
            for _ in range(4):
                qd, cd = hp.to(dev, non_blocking=True), hc.to(dev, non_blocking=True)
                ws = self.workspace(W, H, nl)
                fr = N.SfFrame()
                fr.host_levels = ctypes.cast(lv, ctypes.c_void_p)
                fr.n_levels = nl
                fr.early_exit = 1
                fr.pair_capacity = self.pair_capacity
                fr.coeff_map = N.ptr(out.coeff_map)
                fr.final_t = N.ptr(out.final_t)
                fr.relevancy_raw = N.ptr(raw)
                fr.stats_i64 = N.ptr(out.stats_i64)
                fr.stats_f64 = N.ptr(out.stats_f64)
                if band is not None:
                    fr.band_y0, fr.band_y1 = int(band[0]), int(band[1])
                if nl * cfg.K <= 16:
                    fr.chan_by_row = N.ptr(self.channel_plan(levels))
                N.check(lib.sf_query_sweep(ctypes.byref(self.ds.struct), ctypes.byref(camc), ctypes.byref(fr),
                                           N.ptr(qd), n, N.ptr(cd), int(canonicals.shape[0]), int(window),
                                           float(threshold), N.ptr(filt), N.ptr(masks), N.ptr(si), N.ptr(sf),
                                           N.ptr(ws), ws.numel(), stream_ptr()))
                hsi = torch.empty(si.shape, dtype=si.dtype, pin_memory=True)
                hsf = torch.empty(sf.shape, dtype=sf.dtype, pin_memory=True)
                hsi.copy_(si, non_blocking=True)
                hsf.copy_(sf, non_blocking=True)
                fst = out.stats_i64.cpu().numpy()  # synchronises the stream
                if int(fst[N.STAT_OVERFLOW]) == 0:
                    N.check_fixups(fst, out.width, out.height)
                    out._host = (fst, out.stats_f64.cpu().numpy())
                    return filt, masks, hsi.numpy()[:n], hsf.numpy()[:n]
                self.pair_capacity = int(int(fst[N.STAT_PAIRS]) * 1.25) + 1024
            raise SplatfieldError("pair buffer overflow persisted after growing")


class FramePipeline:
    """Frames of one scene overlapped on the GPU: frame i's projection / sort /
    binning run on a shared prepare stream and its blend (+ decode) / post on
    render stream i % 2 (sf_render_frame_split), with two engines
    (workspaces) and two output sets used alternately.  So frame i+1's
    first half overlaps frame i's blend, and frame i+1's blend overlaps frame
    i's fixup / post tail.  Every frame does the complete work.

    begin() / end() join the pipeline's streams with the caller's stream."""

    def __init__(self, dscene: DeviceScene, W: int, H: int, levels, **alloc):
        # engines of their own: the scene's default engine may be in use on another stream
        self.engines = [FrameEngine(dscene), FrameEngine(dscene)]
        for e in self.engines:
            e.pair_capacity = dscene.engine.pair_capacity
            e._plans = dscene.engine._plans  # the cached scatter plans are read-only
        self.outs = [e.allocate(W, H, levels, **alloc) for e in self.engines]
        # the prepare stream is the frame's critical path after the splat kernel (which
        # holds every SM): at high priority its CTAs go first when the splat drains,
        # and the previous frame's fixup / post fill the SMs it leaves idle
        self.prep = torch.cuda.Stream(priority=-1)
        self.render = [torch.cuda.Stream(), torch.cuda.Stream()]
        self.k = 0

    def begin(self):
        cur = torch.cuda.current_stream()
        for st in (self.prep, *self.render):
            st.wait_stream(cur)

    def enqueue(self, cam, levels, **kw) -> FrameOutputs:
        i = self.k % 2
        self.k += 1
        rs = self.render[i]
        self.prep.wait_stream(rs)  # buffer i: the frame two back has finished with it
        out = self.outs[i]
        with torch.cuda.stream(rs):
            self.engines[i].enqueue(cam, levels, out, prep_stream=self.prep, **kw)
        return out

    def end(self):
        cur = torch.cuda.current_stream()
        for st in self.render:
            cur.wait_stream(st)
