"""Deterministic synthetic scenes of SURVEY.md section 8(d) (test/bench fixtures).

The reference's ``conftest.random_scene`` distribution (tests/conftest.py:8-50),
vectorised and resolution-scaled: scales are multiplied by sqrt(1e4 / N) so
per-tile load and blend depth stay constant across configurations.  Draw
order is fixed (seed 1 for every config).
"""

from __future__ import annotations

import numpy as np

from .core import Codebook, Scene, SceneConfig
from .projection import Camera, CameraPose

CONFIGS = {
    # name: (num_gaussians, width, height)
    "A": (10_000, 256, 256),
    "B": (1_000_000, 988, 731),
    "C": (2_000_000, 1440, 1080),
    "E": (5_000_000, 1920, 1080),
}


def make_scene(num_gaussians: int, *, seed: int = 1, num_levels: int = 3, L: int = 64, K: int = 4,
               D: int = 512, chunk: int = 1 << 18) -> Scene:
    """Scene with the section 8(d) distribution (draw order is part of the spec)."""
    n = int(num_gaussians)
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    # argsort(random((levels, n, L)))[..., :K], sorted: drawn in row chunks so
    # memory stays bounded; the stream is consumed in the same C order.
    idx = np.empty((num_levels * n, K), dtype=np.uint16)
    for r0 in range(0, num_levels * n, chunk):
        r1 = min(num_levels * n, r0 + chunk)
        u = rng.random((r1 - r0, L))
        part = np.argpartition(u, K - 1, axis=1)[:, :K] if K < L else np.tile(np.arange(L), (r1 - r0, 1))
        idx[r0:r1] = np.sort(part, axis=1)
    idx = idx.reshape(num_levels, n, K)
    raw = rng.random((num_levels, n, K)) + 1e-3
    val = (raw / raw.sum(axis=2, keepdims=True)).astype(np.float32)
    pos = (rng.uniform(-1, 1, (n, 3)) * np.array([1.0, 1.0, 0.4])).astype(np.float32)
    scl = (rng.uniform(0.03, 0.15, (n, 3)) * np.sqrt(1e4 / max(n, 1))).astype(np.float32)
    opa = rng.uniform(0.2, 0.95, n).astype(np.float32)
    col = rng.uniform(0, 1, (n, 3)).astype(np.float32)
    cbs = tuple(Codebook(rng.standard_normal((L, D)).astype(np.float32), level=lv)
                for lv in range(num_levels))
    return Scene(positions=pos, rotations=q.astype(np.float32), scales=scl, opacities=opa,
                 colors=col, coeff_indices=idx, coeff_values=val, codebooks=cbs,
                 config=SceneConfig(num_levels=num_levels, L=L, K=K, D=D))


def make_camera(width: int, height: int) -> Camera:
    """Camera.look_at((0,0,-3), (0,0,0), fov 45) as in tests/conftest.py:53-60."""
    return Camera.look_at((0.0, 0.0, -3.0), (0.0, 0.0, 0.0), fov_y_deg=45.0, width=width,
                          height=height)


def make_query(D: int = 512, n_canonicals: int = 4, seed: int = 2):
    r = np.random.default_rng(seed)
    return r.standard_normal(D), r.standard_normal((n_canonicals, D))


def orbit_cameras(n: int, width: int = 1440, height: int = 1080):
    """Config D cameras: the orbit rule of io.py:390-405 (fov 42, distance 3.4)."""
    poses = []
    for j in range(n):
        a = 2.0 * np.pi * j / n + 0.35
        poses.append(CameraPose(position=(float(np.sin(a) * 0.55), float(np.cos(a) * 0.55), -3.4),
                                look_at=(0.0, 0.0, 0.0), fov_y_deg=42.0, width=width, height=height))
    return [p.to_camera() for p in poses]
