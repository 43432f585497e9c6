"""CPU oracle for the splatfield hot path -- TEST INFRASTRUCTURE ONLY.

Thin ctypes driver over ``oracle/splat_oracle.c`` (the C restatement of the
reference algorithm) plus numpy for the trivial reductions.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg and
``--impl reference``) may import this module; the product package never
does.

Each function mirrors the reference function named in its docstring
(paths relative to /root/reference/pkg/src/splatfield) and takes the same
duck-typed arguments (anything with the ``Scene`` / ``Camera`` attributes).

Parity pinning: ``oracle/gen_golden.py`` runs the imported reference and
this oracle on the same inputs; the fixtures it writes under
``tests/golden/`` are checked by ``tests/test_oracle_golden.py`` (projection
and binning bitwise, blend/decode/query within 1e-12 relative).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

TILE = 16
CUTOFF = 9.0


class _OrCamera(ctypes.Structure):
    _fields_ = [
        ("R", ctypes.c_double * 9),
        ("t", ctypes.c_double * 3),
        ("fx", ctypes.c_double),
        ("fy", ctypes.c_double),
        ("cx", ctypes.c_double),
        ("cy", ctypes.c_double),
        ("near", ctypes.c_double),
        ("width", ctypes.c_int64),
        ("height", ctypes.c_int64),
    ]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no FMA contraction, OpenMP)."""
    src = os.path.join(_HERE, "splat_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(
            ["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math",
             "-fopenmp", "-o", _LIB_PATH, src, "-lm"]
        )
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        L.or_project.restype = i64
        L.or_project.argtypes = [i64, P, P, P, P, P, ctypes.POINTER(_OrCamera), P, P, P, P, P, P]
        L.or_canonical_order.restype = None
        L.or_canonical_order.argtypes = [i64, P, P, P]
        L.or_bin.restype = i64
        L.or_bin.argtypes = [i64, P, P, i64, i64, i64, P, P, i64]
        L.or_splat.restype = None
        L.or_splat.argtypes = [i64, i64, i64, i64, i64, P, P, P, P, P, P, i64, P, P, i64,
                               ctypes.c_int, P, P, i64, i64]
        L.or_decode.restype = None
        L.or_decode.argtypes = [i64, i64, i64, P, i64, P, P]
        L.or_relevancy.restype = None
        L.or_relevancy.argtypes = [i64, i64, P, P, i64, P, P]
        L.or_mean_filter.restype = None
        L.or_mean_filter.argtypes = [i64, i64, P, i64, P]
        L.or_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _cam(cam) -> _OrCamera:
    c = _OrCamera()
    R = np.ascontiguousarray(np.asarray(cam.rotation, dtype=np.float64)).ravel()
    t = np.asarray(cam.translation, dtype=np.float64).ravel()
    for i in range(9):
        c.R[i] = float(R[i])
    for i in range(3):
        c.t[i] = float(t[i])
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.near = float(cam.near)
    c.width, c.height = int(cam.width), int(cam.height)
    return c


@dataclass
class OracleProjection:
    """Mirror of ProjectedScene (projection.py:162-188)."""

    means2d: np.ndarray
    inv_covs: np.ndarray
    depths: np.ndarray
    opacities: np.ndarray
    source_ids: np.ndarray
    rows: np.ndarray

    @property
    def count(self) -> int:
        return int(self.means2d.shape[0])


def project_arrays(positions, rotations, scales, opacities, ids, cam) -> OracleProjection:
    """project_arrays, projection.py:240-308."""
    pos = np.ascontiguousarray(positions, dtype=np.float32)
    rot = np.ascontiguousarray(rotations, dtype=np.float32)
    scl = np.ascontiguousarray(scales, dtype=np.float32)
    opa = np.ascontiguousarray(opacities, dtype=np.float32)
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    g = pos.shape[0]
    means = np.empty((g, 2))
    inv = np.empty((g, 2, 2))
    depths = np.empty(g)
    op = np.empty(g)
    sid = np.empty(g, dtype=np.int64)
    rows = np.empty(g, dtype=np.int64)
    c = _cam(cam)
    n = lib().or_project(g, _p(pos), _p(rot), _p(scl), _p(opa), _p(ids), ctypes.byref(c),
                         _p(means), _p(inv), _p(depths), _p(op), _p(sid), _p(rows))
    return OracleProjection(means[:n].copy(), inv[:n].copy(), depths[:n].copy(), op[:n].copy(),
                            sid[:n].copy(), rows[:n].copy())


def project_scene(scene, cam) -> OracleProjection:
    """project_scene, projection.py:311-315."""
    return project_arrays(scene.positions, scene.rotations, scene.scales, scene.opacities,
                          scene.ids, cam)


@dataclass
class OracleBinning:
    """Mirror of TileBinning (projection.py:342-376) in CSR form."""

    tile_size: int
    tiles_x: int
    tiles_y: int
    width: int
    height: int
    projected: OracleProjection  # canonical (depth, id) order
    tile_offsets: np.ndarray  # (n_tiles + 1,) int64
    tile_entries: np.ndarray  # (pairs,) int64 indices into `projected`

    @property
    def tile_lists(self):
        o = self.tile_offsets
        return [self.tile_entries[o[t]:o[t + 1]] for t in range(len(o) - 1)]

    def canonical_bytes(self) -> bytes:
        """TileBinning.canonical_bytes, projection.py:370-376."""
        parts = [np.int64(len(self.tile_offsets) - 1).tobytes()]
        o = self.tile_offsets
        sid = self.projected.source_ids
        for t in range(len(o) - 1):
            lst = self.tile_entries[o[t]:o[t + 1]]
            parts.append(np.int64(lst.size).tobytes())
            parts.append(sid[lst].tobytes())
        return b"".join(parts)


def bin_projected(proj: OracleProjection, cam, tile_size: int = TILE) -> OracleBinning:
    """bin_projected, projection.py:379-450."""
    W, H = int(cam.width), int(cam.height)
    tx = (W + tile_size - 1) // tile_size
    ty = (H + tile_size - 1) // tile_size
    n = proj.count
    order = np.empty(n, dtype=np.int64)
    depths = np.ascontiguousarray(proj.depths)
    sids = np.ascontiguousarray(proj.source_ids)
    lib().or_canonical_order(n, _p(depths), _p(sids), _p(order))
    sp = OracleProjection(
        np.ascontiguousarray(proj.means2d[order]), np.ascontiguousarray(proj.inv_covs[order]),
        proj.depths[order].copy(), proj.opacities[order].copy(), proj.source_ids[order].copy(),
        proj.rows[order].copy())
    offsets = np.zeros(tx * ty + 1, dtype=np.int64)
    cap = max(16, 8 * n)
    while True:
        lists = np.empty(cap, dtype=np.int64)
        total = lib().or_bin(n, _p(sp.means2d), _p(sp.inv_covs), tile_size, W, H, _p(offsets),
                             _p(lists), cap)
        if total <= cap:
            break
        cap = int(total)
    return OracleBinning(tile_size, tx, ty, W, H, sp, offsets, lists[:total].copy())


@dataclass
class OracleCoefficientMap:
    data: np.ndarray  # (H, W, len(levels) * L) float64
    L: int
    K: int
    levels: tuple

    def level_view(self, level: int) -> np.ndarray:
        b = self.levels.index(level)
        return self.data[:, :, b * self.L:(b + 1) * self.L]


@dataclass
class OracleStats:
    final_transmittance: np.ndarray
    pairs_blended: int
    channels_per_gaussian: int
    workers: int


def splat_levels(scene, cam, levels, *, binning: OracleBinning | None = None, early_exit=True,
                 tile_range=None, with_stats=False):
    """_splat_levels, sparse_splat.py:103-170 (tile_blend_weights + scatter)."""
    cfg = scene.config
    levels = tuple(int(lv) for lv in levels)
    L = cfg.L
    cat_idx = np.ascontiguousarray(np.concatenate(
        [scene.coeff_indices[lv].astype(np.int64) + b * L for b, lv in enumerate(levels)], axis=1))
    cat_vals = np.ascontiguousarray(np.concatenate(
        [scene.coeff_values[lv].astype(np.float32) for lv in levels], axis=1))
    nch = len(levels) * L
    W, H = int(cam.width), int(cam.height)
    if binning is None:
        binning = bin_projected(project_scene(scene, cam), cam)
    out = np.zeros((H, W, nch))
    final_t = np.ones((H, W))
    sp = binning.projected
    n_tiles = binning.tiles_x * binning.tiles_y
    t0, t1 = (0, n_tiles) if tile_range is None else tile_range
    lib().or_splat(binning.tiles_x, binning.tiles_y, TILE, W, H, _p(binning.tile_offsets),
                   _p(binning.tile_entries), _p(sp.means2d), _p(sp.inv_covs),
                   _p(np.ascontiguousarray(sp.opacities)), _p(np.ascontiguousarray(sp.rows)),
                   cat_idx.shape[1], _p(cat_idx), _p(cat_vals), nch, 1 if early_exit else 0,
                   _p(out), _p(final_t), t0, t1)
    cmap = OracleCoefficientMap(out, L, cfg.K, levels)
    if not with_stats:
        return cmap
    return cmap, OracleStats(final_t, int(binning.tile_offsets[-1]), int(cat_idx.shape[1]), 1)


def splat_multilevel(scene, cam, **kw):
    """splat_multilevel, sparse_splat.py:178-180."""
    return splat_levels(scene, cam, range(scene.config.num_levels), **kw)


def splat_sparse(scene, cam, level, **kw):
    """splat_sparse, sparse_splat.py:173-175."""
    return splat_levels(scene, cam, [level], **kw)


def decode_level(w: np.ndarray, atoms: np.ndarray) -> np.ndarray:
    """One level of decode, sparse_splat.py:183-199: the reference's own
    operation, ``w.reshape(-1, L) @ atoms.astype(float64)`` (numpy / BLAS
    dgemm, as the reference computes it; or_decode is the plain-C twin)."""
    shp = w.shape
    L = shp[-1]
    w2 = np.ascontiguousarray(w.reshape(-1, L), dtype=np.float64)
    out = w2 @ np.asarray(atoms, dtype=np.float32).astype(np.float64)
    return out.reshape(shp[:-1] + (out.shape[1],))


def decode(cmap: OracleCoefficientMap, codebooks):
    """decode, sparse_splat.py:183-199."""
    codebooks = list(codebooks)
    return tuple(decode_level(cmap.level_view(lv), codebooks[lv].atoms) for lv in cmap.levels)


def relevancy_map(features: np.ndarray, q: np.ndarray, canonicals) -> np.ndarray:
    """relevancy_map, query.py:65-84 (raw dot products, two-branch sigmoid)."""
    f = np.ascontiguousarray(features, dtype=np.float64)
    h, w, d = f.shape
    qv = np.ascontiguousarray(q, dtype=np.float64)
    cn = np.ascontiguousarray(np.asarray(canonicals, dtype=np.float64).reshape(-1, d))
    out = np.empty((h, w))
    lib().or_relevancy(h * w, d, _p(f), _p(qv), cn.shape[0], _p(cn), _p(out))
    return out


def mean_filter(m: np.ndarray, window: int) -> np.ndarray:
    """mean_filter, query.py:87-108 (edge padding + integral image)."""
    m = np.ascontiguousarray(m, dtype=np.float64)
    if window == 1:
        return m.copy()
    out = np.empty_like(m)
    lib().or_mean_filter(m.shape[0], m.shape[1], _p(m), window, _p(out))
    return out


def select_level(maps) -> int:
    """select_level, query.py:111-118: first argmax of per-map maxima."""
    return int(np.argmax(np.array([float(m.max()) for m in maps])))


def localize(m: np.ndarray):
    """localize, query.py:121-126: first row-major argmax."""
    r, c = np.unravel_index(int(np.argmax(m)), m.shape)
    return int(r), int(c)


def segment(m: np.ndarray, threshold: float = 0.5):
    """segment, query.py:136-145 -> (mask, degenerate)."""
    lo, hi = float(m.min()), float(m.max())
    if hi <= lo:
        return np.zeros(m.shape, dtype=bool), True
    return (m - lo) / (hi - lo) > threshold, False


@dataclass
class OracleQuery:
    level_maps: tuple
    level: int
    point: tuple
    raw_maps: tuple
    cmap: OracleCoefficientMap
    features: tuple | None


def query_pipeline(scene, cam, qvec, canonicals, *, window=11, level=None, keep_features=True):
    """query_pipeline, sparse_splat.py:243-297."""
    cmap = splat_multilevel(scene, cam)
    raws, maps = [], []
    feats = []
    for b, lv in enumerate(cmap.levels):
        f = decode_level(cmap.level_view(lv), scene.codebooks[lv].atoms)
        raw = relevancy_map(f, qvec, canonicals)
        raws.append(raw)
        maps.append(mean_filter(raw, window))
        if keep_features:
            feats.append(f)
    if level is None:
        chosen = select_level(maps)
    else:
        chosen = cmap.levels.index(level)
    point = localize(maps[chosen])
    return OracleQuery(tuple(maps), cmap.levels[chosen], point, tuple(raws), cmap,
                       tuple(feats) if keep_features else None)


def num_threads() -> int:
    return int(lib().or_num_threads())
