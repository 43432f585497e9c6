"""Host value types and per-Gaussian helpers of the drop-in API
(splatfield/core.py:59-105, 133-256, 333-376; projection.py:318-332;
train.py:142-153).

These are small host-side objects (one Gaussian, one sparse coefficient
vector) that callers use to build or inspect scenes; none of them is on the
frame path.  ``project_gaussian`` projects through the same sm_100a kernel as
``project_scene`` (a one-Gaussian scene), so its numbers are the frame's.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import QUAT_NORM_TOL, SIMPLEX_SUM_TOL, Codebook, Scene, SceneConfig
from .errors import ValidationError


def _vec_f32(x, n: int, what: str) -> np.ndarray:
    v = np.asarray(x, dtype=np.float32)
    if v.shape != (n,):
        raise ValidationError(f"{what} must have shape ({n},), got {v.shape}")
    if not np.isfinite(v).all():
        raise ValidationError(f"{what} must be finite")
    return v


@dataclass(frozen=True, eq=False)
class SparseCoefficients:
    """K stored entries of an L-simplex vector: strictly increasing u16
    indices, non-negative f32 values summing to 1 (core.py:59-105)."""

    indices: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        idx = np.asarray(self.indices, dtype=np.uint16)
        val = np.asarray(self.values, dtype=np.float32)
        object.__setattr__(self, "indices", idx)
        object.__setattr__(self, "values", val)
        if idx.ndim != 1 or idx.shape != val.shape:
            raise ValidationError("indices and values must be 1-D arrays of equal length")
        if idx.size == 0:
            raise ValidationError("at least one stored entry is required")
        if np.any(np.diff(idx.astype(np.int64)) <= 0):
            raise ValidationError("indices must be strictly increasing")
        if (val < 0).any():
            raise ValidationError("values must be non-negative")
        total = float(val.astype(np.float64).sum())
        if abs(total - 1.0) > SIMPLEX_SUM_TOL:
            raise ValidationError(f"values must sum to 1 +- {SIMPLEX_SUM_TOL}, got {total}")

    @property
    def k(self) -> int:
        return int(self.indices.size)

    def validate_against(self, L: int) -> None:
        top = int(self.indices.max())
        if top >= L:
            raise ValidationError(f"coefficient index {top} >= codebook size {L}")

    def __eq__(self, other) -> bool:
        if not isinstance(other, SparseCoefficients):
            return NotImplemented
        return np.array_equal(self.indices, other.indices) and np.array_equal(self.values, other.values)


@dataclass(frozen=True)
class Gaussian:
    """One scene point (core.py:133-156): position, unit wxyz quaternion,
    per-axis sigma > 0, opacity in [0, 1], colour, one SparseCoefficients
    per level, id."""

    position: np.ndarray
    rotation: np.ndarray
    scale: np.ndarray
    opacity: float
    color: np.ndarray
    coeffs: tuple
    id: int = 0

    def __post_init__(self):
        object.__setattr__(self, "position", _vec_f32(self.position, 3, "position"))
        object.__setattr__(self, "rotation", _vec_f32(self.rotation, 4, "rotation"))
        object.__setattr__(self, "scale", _vec_f32(self.scale, 3, "scale"))
        object.__setattr__(self, "color", _vec_f32(self.color, 3, "color"))
        object.__setattr__(self, "coeffs", tuple(self.coeffs))
        norm = float(np.sqrt((self.rotation.astype(np.float64) ** 2).sum()))
        if abs(norm - 1.0) > QUAT_NORM_TOL:
            raise ValidationError(f"quaternion norm must be 1 +- {QUAT_NORM_TOL}, got {norm}")
        if (self.scale <= 0).any():
            raise ValidationError("scale components must be > 0")
        if not 0.0 <= float(self.opacity) <= 1.0:
            raise ValidationError(f"opacity must be in [0, 1], got {self.opacity}")


def quaternion_to_matrix(q) -> np.ndarray:
    """3x3 rotation of a scalar-first unit quaternion (core.py:159-168)."""
    w, x, y, z = (float(c) for c in np.asarray(q, dtype=np.float64))
    xx, yy, zz = x * x, y * y, z * z
    return np.array([[1 - 2 * (yy + zz), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (xx + zz), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (xx + yy)]])


def build_covariance(rotation, scale) -> np.ndarray:
    """R S S^T R^T of one Gaussian, symmetrised exactly (core.py:171-190)."""
    q = np.asarray(rotation, dtype=np.float64)
    s = np.asarray(scale, dtype=np.float64)
    if q.shape != (4,) or s.shape != (3,):
        raise ValidationError("rotation must be a quaternion, scale a 3-vector")
    if not (np.isfinite(q).all() and np.isfinite(s).all()):
        raise ValidationError("non-finite rotation or scale")
    if abs(float(np.linalg.norm(q)) - 1.0) > QUAT_NORM_TOL:
        raise ValidationError("quaternion must be unit norm")
    if (s <= 0).any():
        raise ValidationError("scale components must be > 0")
    rs = quaternion_to_matrix(q) * s[None, :]
    cov = rs @ rs.T
    return (cov + cov.T) * 0.5


def reconstruct_feature(coeffs: SparseCoefficients, codebook: Codebook) -> np.ndarray:
    """sum_k w_k atom_{i_k} in float64 (core.py:212-216)."""
    coeffs.validate_against(codebook.L)
    rows = codebook.atoms[coeffs.indices.astype(np.int64)].astype(np.float64)
    return coeffs.values.astype(np.float64) @ rows


def densify(coeffs: SparseCoefficients, L: int) -> np.ndarray:
    """Dense float64 L-vector of the stored entries (core.py:219-224)."""
    coeffs.validate_against(L)
    out = np.zeros(L)
    out[coeffs.indices.astype(np.int64)] = coeffs.values
    return out


def top_k_indices(values, k: int) -> np.ndarray:
    """The k largest entries' indices, ties to the lower index, ascending (core.py:227-234)."""
    v = np.asarray(values)
    if k < 1 or k > v.size:
        raise ValidationError(f"require 1 <= k <= {v.size}, got {k}")
    return np.sort(np.argsort(-v, kind="stable")[:k])


def compact(dense, k: int | None = None) -> SparseCoefficients:
    """Top-k (or, without k, the nonzero) entries of a dense vector (core.py:237-254)."""
    d = np.asarray(dense, dtype=np.float64)
    if d.ndim != 1:
        raise ValidationError("dense coefficient vector must be 1-D")
    if k is None:
        keep = np.flatnonzero(d)
        if keep.size == 0:
            raise ValidationError("cannot compact an all-zero vector without k")
    else:
        keep = top_k_indices(d, k)
    return SparseCoefficients(indices=keep.astype(np.uint16), values=d[keep].astype(np.float32))


def scene_gaussian(scene, i: int) -> Gaussian:
    """Row i of a scene as a Gaussian value (Scene.gaussian, core.py:333-347)."""
    levels = scene.config.num_levels
    return Gaussian(position=scene.positions[i], rotation=scene.rotations[i], scale=scene.scales[i],
                    opacity=float(scene.opacities[i]), color=scene.colors[i],
                    coeffs=tuple(SparseCoefficients(scene.coeff_indices[b, i], scene.coeff_values[b, i])
                                 for b in range(levels)),
                    id=int(scene.ids[i]))


def scene_from_gaussians(gaussians, codebooks, config: SceneConfig) -> Scene:
    """Scene.from_gaussians (core.py:349-376): stack the values, then validate."""
    gs = list(gaussians)
    g, levels, K = len(gs), config.num_levels, config.K

    def stack(attr, width, dtype):
        return np.array([getattr(p, attr) for p in gs], dtype=dtype).reshape((g,) + width)

    ci = np.array([[p.coeffs[b].indices for p in gs] for b in range(levels)], dtype=np.uint16)
    cv = np.array([[p.coeffs[b].values for p in gs] for b in range(levels)], dtype=np.float32)
    scene = Scene(positions=stack("position", (3,), np.float32), rotations=stack("rotation", (4,), np.float32),
                  scales=stack("scale", (3,), np.float32), opacities=stack("opacity", (), np.float32),
                  colors=stack("color", (3,), np.float32), coeff_indices=ci.reshape(levels, g, K),
                  coeff_values=cv.reshape(levels, g, K), codebooks=tuple(codebooks), config=config,
                  ids=np.array([p.id for p in gs], dtype=np.int64).reshape(g))
    scene.validate()
    return scene


Scene.gaussian = scene_gaussian
Scene.from_gaussians = classmethod(lambda cls, gaussians, codebooks, config: scene_from_gaussians(
    gaussians, codebooks, config))


def project_gaussian(g: Gaussian, cam):
    """One Gaussian projected by the frame's projection kernel; None when culled
    (projection.py:318-332)."""
    from .projection import project_scene
    if not (np.isfinite(g.position).all() and np.isfinite(g.opacity)):
        raise ValidationError("non-finite gaussian input")
    k = g.coeffs[0].k if g.coeffs else 1
    L = int(max((int(c.indices.max()) for c in g.coeffs), default=0)) + 1 if g.coeffs else 1
    levels = max(1, len(g.coeffs))
    cfg = SceneConfig(num_levels=levels, L=max(L, k), K=k, D=1)
    if g.coeffs:
        ci = np.stack([c.indices for c in g.coeffs]).reshape(levels, 1, k)
        cv = np.stack([c.values for c in g.coeffs]).reshape(levels, 1, k)
    else:
        ci = np.zeros((1, 1, 1), np.uint16)
        cv = np.ones((1, 1, 1), np.float32)
    one = Scene(positions=g.position.reshape(1, 3), rotations=g.rotation.reshape(1, 4),
                scales=g.scale.reshape(1, 3), opacities=np.array([g.opacity], np.float32),
                colors=g.color.reshape(1, 3), coeff_indices=ci, coeff_values=cv,
                codebooks=tuple(Codebook(np.zeros((cfg.L, 1), np.float32), level=b) for b in range(levels)),
                config=cfg, ids=np.array([g.id], np.int64))
    proj = project_scene(one, cam)
    if proj.count == 0:
        return None
    return proj.record(0)
