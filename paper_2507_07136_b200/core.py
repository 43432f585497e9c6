"""Scene container types of the drop-in API (splatfield/core.py:40-130, 256-408).

The hot path accepts these or any object exposing the same attributes (a
``splatfield.Scene`` works unchanged): positions (G,3) f32, rotations (G,4)
f32 wxyz, scales (G,3) f32, opacities (G,) f32, colors (G,3) f32,
coeff_indices (levels,G,K) u16, coeff_values (levels,G,K) f32, codebooks
(one (L,D) atoms matrix per level), config (num_levels, L, K, D), ids (G,)
i64.  Scenes are immutable by contract (the reference never mutates one);
the device copy is cached per object.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ValidationError

QUAT_NORM_TOL = 1e-6
SIMPLEX_SUM_TOL = 1e-6


@dataclass(frozen=True)
class SceneConfig:
    """Dimensions shared by every Gaussian (core.py:40-56)."""

    num_levels: int = 3
    L: int = 64
    K: int = 4
    D: int = 512

    def __post_init__(self):
        if self.K < 1 or self.K > self.L:
            raise ValidationError(f"require 1 <= K <= L, got K={self.K}, L={self.L}")
        if self.num_levels < 1:
            raise ValidationError("num_levels must be >= 1")
        if self.D < 1:
            raise ValidationError("D must be >= 1")


@dataclass(frozen=True)
class Codebook:
    """L basis vectors of dimension D for one semantic level (core.py:106-130)."""

    atoms: np.ndarray
    level: int = 0

    def __post_init__(self):
        atoms = np.asarray(self.atoms, dtype=np.float32)
        object.__setattr__(self, "atoms", atoms)
        if atoms.ndim != 2 or atoms.shape[0] < 1 or atoms.shape[1] < 1:
            raise ValidationError(f"atoms must be a non-empty 2-D matrix, got {atoms.shape}")
        if not np.all(np.isfinite(atoms)):
            raise ValidationError("codebook atoms must be finite")
        if self.level < 0:
            raise ValidationError("level must be >= 0")

    @property
    def L(self) -> int:
        return int(self.atoms.shape[0])

    @property
    def D(self) -> int:
        return int(self.atoms.shape[1])


@dataclass(eq=False)
class Scene:
    """Struct-of-arrays Gaussian scene plus per-level codebooks (core.py:256-331)."""

    positions: np.ndarray
    rotations: np.ndarray
    scales: np.ndarray
    opacities: np.ndarray
    colors: np.ndarray
    coeff_indices: np.ndarray
    coeff_values: np.ndarray
    codebooks: tuple
    config: SceneConfig
    ids: np.ndarray = field(default=None)

    def __post_init__(self):
        if self.ids is None:
            self.ids = np.arange(self.num_gaussians, dtype=np.int64)
        self.codebooks = tuple(self.codebooks)

    @property
    def num_gaussians(self) -> int:
        return int(self.positions.shape[0])

    def validate(self) -> None:
        g = self.num_gaussians
        cfg = self.config
        shapes = {
            "positions": (self.positions, (g, 3)),
            "rotations": (self.rotations, (g, 4)),
            "scales": (self.scales, (g, 3)),
            "opacities": (self.opacities, (g,)),
            "colors": (self.colors, (g, 3)),
            "coeff_indices": (self.coeff_indices, (cfg.num_levels, g, cfg.K)),
            "coeff_values": (self.coeff_values, (cfg.num_levels, g, cfg.K)),
        }
        for name, (arr, shape) in shapes.items():
            if arr.shape != shape:
                raise ValidationError(f"{name}: expected shape {shape}, got {arr.shape}")
        for name in ("positions", "rotations", "scales", "opacities", "colors", "coeff_values"):
            if not np.all(np.isfinite(getattr(self, name))):
                raise ValidationError(f"{name}: non-finite entries")
        if len(self.codebooks) != cfg.num_levels:
            raise ValidationError("one codebook per semantic level is required")
        for cb in self.codebooks:
            if cb.L != cfg.L or cb.D != cfg.D:
                raise ValidationError(
                    f"codebook {cb.atoms.shape} does not match config L={cfg.L}, D={cfg.D}")
        if g == 0:
            return
        norms = np.linalg.norm(self.rotations.astype(np.float64), axis=1)
        if np.any(np.abs(norms - 1.0) > QUAT_NORM_TOL):
            raise ValidationError("all quaternions must be unit norm")
        if np.any(self.scales <= 0):
            raise ValidationError("all scales must be > 0")
        if np.any((self.opacities < 0) | (self.opacities > 1)):
            raise ValidationError("opacities must be in [0, 1]")
        if np.any(self.coeff_indices >= cfg.L):
            raise ValidationError("coefficient index >= L")
        if cfg.K > 1 and not np.all(self.coeff_indices[:, :, 1:] > self.coeff_indices[:, :, :-1]):
            raise ValidationError("coefficient indices must be strictly increasing")
        if np.any(self.coeff_values < 0):
            raise ValidationError("coefficient values must be >= 0")
        sums = self.coeff_values.sum(axis=2, dtype=np.float64)
        if np.any(np.abs(sums - 1.0) > SIMPLEX_SUM_TOL):
            raise ValidationError("coefficient values must sum to 1 per level")
        if np.unique(self.ids).size != g:
            raise ValidationError("gaussian ids must be unique")

    def permuted(self, order: np.ndarray) -> "Scene":
        """Rows reordered, ids travelling with their rows (core.py:378-391)."""
        return Scene(
            positions=self.positions[order], rotations=self.rotations[order],
            scales=self.scales[order], opacities=self.opacities[order], colors=self.colors[order],
            coeff_indices=self.coeff_indices[:, order], coeff_values=self.coeff_values[:, order],
            codebooks=self.codebooks, config=self.config, ids=self.ids[order])

    def densified_coefficients(self, level: int) -> np.ndarray:
        """(G, L) float64 dense coefficient rows of one level (core.py:400-408)."""
        g, k = self.coeff_values[level].shape
        dense = np.zeros((g, self.config.L), dtype=np.float64)
        rows = np.repeat(np.arange(g), k)
        dense[rows, self.coeff_indices[level].astype(np.int64).ravel()] = \
            self.coeff_values[level].astype(np.float64).ravel()
        return dense

    def reconstructed_features(self, level: int) -> np.ndarray:
        """(G, D) float64 per-Gaussian features w @ atoms (core.py:393-398)."""
        atoms = self.codebooks[level].atoms.astype(np.float64)
        idx = self.coeff_indices[level].astype(np.int64)
        vals = self.coeff_values[level].astype(np.float64)
        return np.einsum("gk,gkd->gd", vals, atoms[idx])
