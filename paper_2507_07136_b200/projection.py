"""Screen-space projection and tile binning (drop-in for splatfield/projection.py).

``project_scene`` (projection.py:311-315) and ``bin_projected``
(projection.py:379-450) run on the GPU (sf_project / sf_bin) and return
bitwise-identical fp64 records and byte-identical per-tile lists.  Results
are device-backed; numpy views materialise on first attribute access.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import ValidationError

DEFAULT_TILE_SIZE = 16   # projection.py:31
LOWPASS_FLOOR = 0.3      # projection.py:32
CUTOFF_MAHAL_SQ = 9.0    # projection.py:33
ALPHA_CLAMP = 0.99       # projection.py:34


@dataclass(frozen=True)
class Camera:
    """Pinhole camera (projection.py:37-103): x right, y down, z forward."""

    rotation: np.ndarray
    translation: np.ndarray
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    near: float = 0.01

    def __post_init__(self):
        object.__setattr__(self, "rotation", np.asarray(self.rotation, dtype=np.float64))
        object.__setattr__(self, "translation", np.asarray(self.translation, dtype=np.float64))
        if self.rotation.shape != (3, 3) or self.translation.shape != (3,):
            raise ValidationError("camera transform must be a 3x3 rotation and 3-vector")
        if self.fx <= 0 or self.fy <= 0:
            raise ValidationError("focal lengths must be > 0")
        if self.width < 1 or self.height < 1:
            raise ValidationError("image size must be >= 1 pixel")
        if self.near <= 0:
            raise ValidationError("near plane must be > 0")

    @classmethod
    def look_at(cls, position, target, up=(0.0, 1.0, 0.0), fov_y_deg: float = 50.0,
                width: int = 64, height: int = 64, near: float = 0.01) -> "Camera":
        """Camera at ``position`` looking at ``target`` (projection.py:67-103)."""
        position = np.asarray(position, dtype=np.float64)
        forward = np.asarray(target, dtype=np.float64) - position
        n = np.linalg.norm(forward)
        if n == 0:
            raise ValidationError("camera position and target coincide")
        z = forward / n
        right = np.cross(np.asarray(up, dtype=np.float64), z)
        rn = np.linalg.norm(right)
        if rn < 1e-12:
            raise ValidationError("up vector is parallel to the view direction")
        x = right / rn
        y = np.cross(z, x)
        rot = np.stack([x, y, z])
        fy = (height / 2.0) / np.tan(np.radians(fov_y_deg) / 2.0)
        return cls(rotation=rot, translation=-rot @ position, fx=fy, fy=fy, cx=width / 2.0,
                   cy=height / 2.0, width=width, height=height, near=near)


@dataclass(frozen=True)
class CameraPose:
    """Position + look-at + vertical FOV (projection.py:106-148)."""

    position: tuple
    look_at: tuple
    up: tuple = (0.0, 1.0, 0.0)
    fov_y_deg: float = 50.0
    width: int = 64
    height: int = 64
    near: float = 0.01

    def to_camera(self) -> Camera:
        return Camera.look_at(self.position, self.look_at, self.up, fov_y_deg=self.fov_y_deg,
                              width=self.width, height=self.height, near=self.near)

    def to_dict(self) -> dict:
        """JSON form (projection.py:124-133)."""
        return {"position": list(self.position), "look_at": list(self.look_at), "up": list(self.up),
                "fov_y_deg": self.fov_y_deg, "width": self.width, "height": self.height, "near": self.near}

    @classmethod
    def from_dict(cls, d: dict) -> "CameraPose":
        """projection.py:135-148; missing / malformed fields raise ValidationError."""
        try:
            vec = lambda v: tuple(float(x) for x in v)  # noqa: E731
            return cls(position=vec(d["position"]), look_at=vec(d["look_at"]),
                       up=vec(d.get("up", (0.0, 1.0, 0.0))), fov_y_deg=float(d.get("fov_y_deg", 50.0)),
                       width=int(d.get("width", 64)), height=int(d.get("height", 64)),
                       near=float(d.get("near", 0.01)))
        except (KeyError, TypeError, ValueError) as exc:
            raise ValidationError(f"bad camera pose: {exc}") from exc


@dataclass(frozen=True)
class ProjectedGaussian:
    """Screen-space record consumed by the rasterizer (projection.py:151-159)."""

    mean2d: np.ndarray
    inv_cov2d: np.ndarray
    depth: float
    opacity: float
    source_id: int


class ProjectedScene:
    """Surviving projected Gaussians (projection.py:162-188), device-backed.

    Arrays: means2d (N,2), inv_covs (N,2,2), depths (N,), opacities (N,) all
    float64; source_ids, rows (N,) int64.  ``dev`` holds the torch tensors.
    """

    _FIELDS = ("means2d", "inv_covs", "depths", "opacities", "source_ids", "rows")

    def __init__(self, means2d=None, inv_covs=None, depths=None, opacities=None, source_ids=None,
                 rows=None, *, dev=None):
        self.dev = dev  # dict of torch tensors or None
        self._host = {}
        if dev is None:
            n = np.asarray(means2d).shape[0]
            self._host = {
                "means2d": np.asarray(means2d, dtype=np.float64).reshape(n, 2),
                "inv_covs": np.asarray(inv_covs, dtype=np.float64).reshape(n, 2, 2),
                "depths": np.asarray(depths, dtype=np.float64).reshape(n),
                "opacities": np.asarray(opacities, dtype=np.float64).reshape(n),
                "source_ids": np.asarray(source_ids, dtype=np.int64).reshape(n),
                "rows": np.asarray(rows, dtype=np.int64).reshape(n),
            }

    def _get(self, name):
        if name not in self._host:
            self._host[name] = self.dev[name].cpu().numpy()
        return self._host[name]

    means2d = property(lambda self: self._get("means2d"))
    inv_covs = property(lambda self: self._get("inv_covs"))
    depths = property(lambda self: self._get("depths"))
    opacities = property(lambda self: self._get("opacities"))
    source_ids = property(lambda self: self._get("source_ids"))
    rows = property(lambda self: self._get("rows"))

    @property
    def count(self) -> int:
        if self.dev is not None:
            return int(self.dev["means2d"].shape[0])
        return int(self._host["means2d"].shape[0])

    def record(self, i: int) -> ProjectedGaussian:
        return ProjectedGaussian(mean2d=self.means2d[i], inv_cov2d=self.inv_covs[i],
                                 depth=float(self.depths[i]), opacity=float(self.opacities[i]),
                                 source_id=int(self.source_ids[i]))

    def device_arrays(self):
        """(means2d, inv_covs, depths, opacities, source_ids, rows) as CUDA tensors."""
        import torch

        from .device import require_cuda
        if self.dev is None:
            dev = require_cuda()
            self.dev = {k: torch.from_numpy(np.ascontiguousarray(self._host[k])).to(dev)
                        for k in self._FIELDS}
        return tuple(self.dev[k] for k in self._FIELDS)


def project_scene(scene, cam) -> ProjectedScene:
    """project_scene (projection.py:311-315) on the GPU: bitwise-equal fp64 records."""
    import torch

    from .device import camera_struct, device_scene, stream_ptr
    ds = device_scene(scene)
    g = ds.num_gaussians
    dev = ds.device
    lib = N.load()
    nbytes = ctypes.c_size_t(0)
    N.check(lib.sf_project_workspace_bytes(g, ctypes.byref(nbytes)))
    ws = torch.empty(nbytes.value, dtype=torch.uint8, device=dev)
    gp = max(g, 1)
    out = {
        "means2d": torch.empty((gp, 2), dtype=torch.float64, device=dev),
        "inv_covs": torch.empty((gp, 2, 2), dtype=torch.float64, device=dev),
        "depths": torch.empty(gp, dtype=torch.float64, device=dev),
        "opacities": torch.empty(gp, dtype=torch.float64, device=dev),
        "source_ids": torch.empty(gp, dtype=torch.int64, device=dev),
        "rows": torch.empty(gp, dtype=torch.int64, device=dev),
    }
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    camc = camera_struct(cam)
    N.check(lib.sf_project_rows(ctypes.byref(ds.struct), ctypes.byref(camc), N.ptr(ds.orig_rows),
                                *(N.ptr(out[k]) for k in ProjectedScene._FIELDS), N.ptr(count),
                                N.ptr(ws), ws.numel(), stream_ptr()))
    n = int(count.item())
    return ProjectedScene(dev={k: v[:n] for k, v in out.items()})


class TileBinning:
    """Per-tile depth/id-ordered lists (projection.py:342-376) in CSR form."""

    def __init__(self, tile_size, tiles_x, tiles_y, width, height, projected, tile_offsets,
                 tile_entries):
        self.tile_size = tile_size
        self.tiles_x = tiles_x
        self.tiles_y = tiles_y
        self.width = width
        self.height = height
        self.projected = projected        # canonical (depth, id) order
        self.tile_offsets = tile_offsets  # (n_tiles + 1,) int64 numpy
        self.tile_entries = tile_entries  # (pairs,) int64 numpy, indices into projected
        self._lists = None

    @property
    def tile_lists(self):
        if self._lists is None:
            o = self.tile_offsets
            self._lists = [self.tile_entries[o[t]:o[t + 1]] for t in range(len(o) - 1)]
        return self._lists

    def tile_index(self, tx: int, ty: int) -> int:
        return ty * self.tiles_x + tx

    def tile_records(self, tx: int, ty: int):
        return [self.projected.record(int(i)) for i in self.tile_lists[self.tile_index(tx, ty)]]

    def tile_pixel_bounds(self, tx: int, ty: int):
        x0 = tx * self.tile_size
        y0 = ty * self.tile_size
        return x0, min(x0 + self.tile_size, self.width), y0, min(y0 + self.tile_size, self.height)

    def canonical_bytes(self) -> bytes:
        """Deterministic serialisation (projection.py:370-376)."""
        parts = [np.int64(len(self.tile_offsets) - 1).tobytes()]
        sid = self.projected.source_ids
        o = self.tile_offsets
        for t in range(len(o) - 1):
            lst = self.tile_entries[o[t]:o[t + 1]]
            parts.append(np.int64(lst.size).tobytes())
            parts.append(sid[lst].tobytes())
        return b"".join(parts)


def bin_projected(proj: ProjectedScene, cam, tile_size: int = DEFAULT_TILE_SIZE) -> TileBinning:
    """bin_projected (projection.py:379-450) on the GPU (sf_bin)."""
    import torch

    from .device import require_cuda, stream_ptr
    if tile_size < 1:
        raise ValidationError("tile size must be >= 1")
    if tile_size != DEFAULT_TILE_SIZE:
        raise ValidationError("the sm_100a kernels are specialised for 16x16 tiles")
    W, H = int(cam.width), int(cam.height)
    tx = (W + tile_size - 1) // tile_size
    ty = (H + tile_size - 1) // tile_size
    n = proj.count
    dev = require_cuda()
    means, inv, depths, opac, sids, rows = proj.device_arrays()
    lib = N.load()
    cap = max(1 << 12, 8 * n)
    order = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    offsets = torch.empty(tx * ty + 1, dtype=torch.int64, device=dev)
    stats = torch.zeros(16, dtype=torch.int64, device=dev)
    for _ in range(4):
        nbytes = ctypes.c_size_t(0)
        N.check(lib.sf_bin_workspace_bytes(n, W, H, cap, ctypes.byref(nbytes)))
        ws = torch.empty(nbytes.value, dtype=torch.uint8, device=dev)
        entries = torch.empty(cap, dtype=torch.int32, device=dev)
        N.check(lib.sf_bin(n, N.ptr(means.contiguous()), N.ptr(inv.contiguous()),
                           N.ptr(depths.contiguous()), N.ptr(sids.contiguous()), W, H, cap,
                           N.ptr(order), N.ptr(offsets), N.ptr(entries), N.ptr(stats), N.ptr(ws),
                           ws.numel(), stream_ptr()))
        st = stats.cpu().numpy()
        if st[N.STAT_OVERFLOW] == 0:
            break
        cap = int(st[N.STAT_PAIRS]) + 1024
    pairs = int(st[N.STAT_PAIRS])
    o = order[:n]
    canon = ProjectedScene(dev={
        "means2d": means[o], "inv_covs": inv[o], "depths": depths[o], "opacities": opac[o],
        "source_ids": sids[o], "rows": rows[o]})
    return TileBinning(tile_size, tx, ty, W, H, canon, offsets.cpu().numpy(),
                       entries[:pairs].to(torch.int64).cpu().numpy())


def bin_tiles(projected, cam, tile_size: int = DEFAULT_TILE_SIZE) -> TileBinning:
    """Bin a list of ProjectedGaussian records (projection.py:453-466)."""
    n = len(projected)
    proj = ProjectedScene(
        means2d=np.array([p.mean2d for p in projected], dtype=np.float64).reshape(n, 2),
        inv_covs=np.array([p.inv_cov2d for p in projected], dtype=np.float64).reshape(n, 2, 2),
        depths=np.array([p.depth for p in projected], dtype=np.float64),
        opacities=np.array([p.opacity for p in projected], dtype=np.float64),
        source_ids=np.array([p.source_id for p in projected], dtype=np.int64),
        rows=np.arange(n, dtype=np.int64))
    return bin_projected(proj, cam, tile_size)


def eval_alpha(p: ProjectedGaussian, pixel) -> float:
    """Opacity-weighted Gaussian value clamped to [0, 0.99] (projection.py:335-339)."""
    d = np.asarray(pixel, dtype=np.float64) - np.asarray(p.mean2d, dtype=np.float64)
    q = float(d @ np.asarray(p.inv_cov2d, dtype=np.float64) @ d)
    return min(float(p.opacity) * float(np.exp(-0.5 * q)), ALPHA_CLAMP)
