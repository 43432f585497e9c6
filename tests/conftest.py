"""Shared fixtures.  ``gpu`` marks tests that need a B200 (run with -m gpu)."""

import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")


from paper_2507_07136_b200.core import Codebook, Scene, SceneConfig  # noqa: E402
from paper_2507_07136_b200.projection import Camera  # noqa: E402


def golden_names(require_query=False, require_features=False):
    out = []
    for p in sorted(glob.glob(os.path.join(GOLDEN, "*.npz"))):
        name = os.path.basename(p)[:-4]
        if name.startswith(("config", "dense", "train")):
            continue
        with np.load(p) as z:
            if require_query and "q_filtered" not in z:
                continue
        out.append(name)
    return out


def load_golden(name):
    """(scene, camera, dict of reference outputs) of one fixture."""
    z = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    nl, L, K, D = (int(v) for v in z["config"])
    cfg = SceneConfig(num_levels=nl, L=L, K=K, D=D)
    scene = Scene(positions=z["positions"], rotations=z["rotations"], scales=z["scales"],
                  opacities=z["opacities"], colors=z["colors"], coeff_indices=z["coeff_indices"],
                  coeff_values=z["coeff_values"],
                  codebooks=tuple(Codebook(z["codebooks"][lv], level=lv) for lv in range(nl)),
                  config=cfg, ids=z["ids"])
    fx, fy, cx, cy, near = (float(v) for v in z["cam_intr"])
    w, h = (int(v) for v in z["cam_size"])
    cam = Camera(rotation=z["cam_R"], translation=z["cam_t"], fx=fx, fy=fy, cx=cx, cy=cy, width=w,
                 height=h, near=near)
    return scene, cam, z


def random_scene(rng, num_gaussians=50, num_levels=1, L=16, K=4, D=8, image_extent=1.0,
                 opacity_range=(0.2, 0.95)):
    """The reference tests' scene distribution (tests/conftest.py:8-50), vectorised draws."""
    cfg = SceneConfig(num_levels=num_levels, L=L, K=K, D=D)
    g = num_gaussians
    quats = rng.standard_normal((g, 4))
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    idx = np.sort(np.argsort(rng.random((num_levels, g, L)), axis=2)[:, :, :K], axis=2).astype(np.uint16)
    raw = rng.random((num_levels, g, K)) + 1e-3
    val = (raw / raw.sum(axis=2, keepdims=True)).astype(np.float32)
    cbs = tuple(Codebook(rng.standard_normal((L, D)).astype(np.float32), level=lv)
                for lv in range(num_levels))
    return Scene(
        positions=(rng.uniform(-image_extent, image_extent, (g, 3)) * np.array([1.0, 1.0, 0.4])).astype(np.float32),
        rotations=quats.astype(np.float32), scales=rng.uniform(0.03, 0.15, (g, 3)).astype(np.float32),
        opacities=rng.uniform(*opacity_range, g).astype(np.float32),
        colors=rng.uniform(0, 1, (g, 3)).astype(np.float32), coeff_indices=idx, coeff_values=val,
        codebooks=cbs, config=cfg)


def make_camera(width=32, height=32, fov=45.0):
    return Camera.look_at(position=(0.0, 0.0, -3.0), target=(0.0, 0.0, 0.0), fov_y_deg=fov,
                          width=width, height=height)


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


TIE_MARGIN = 1e-12


def assert_selection_matches(ref_maps, level, point, mask, ref_level, ref_point, ref_mask=None,
                             threshold=0.5):
    """level / point / mask identity, tie-aware.

    The reference filters with an integral image (query.py:96-104) whose
    rounding noise (~1e-15) decides between exactly tied maxima, although its
    own contract is "ties to the lowest level" / "smallest row, then column"
    (query.py:111-126).  We implement the contract on the exact filter.  So:
    a differing choice is accepted only if the reference's own values tie
    within TIE_MARGIN there (the margin is reported), and mask pixels are
    compared wherever the reference's normalised value is not within 1e-9 of
    the threshold.
    """
    maxima = np.array([m.max() for m in ref_maps])
    if level != ref_level:
        margin = maxima[ref_level] - maxima[level]
        assert margin <= TIE_MARGIN, f"level {level} != {ref_level}, reference margin {margin:.3g}"
    m = ref_maps[level]
    if tuple(point) != tuple(ref_point):
        margin = m.max() - m[tuple(point)]
        assert margin <= TIE_MARGIN, f"point {point} != {ref_point}, reference margin {margin:.3g}"
    if mask is not None:
        lo, hi = m.min(), m.max()
        if hi <= lo:
            assert not np.asarray(mask).any()
            return
        norm = (m - lo) / (hi - lo)
        want = norm > threshold
        decided = np.abs(norm - threshold) > 1e-9
        bad = (np.asarray(mask, dtype=bool) != want) & decided
        assert not bad.any(), f"{int(bad.sum())} mask pixels differ away from the threshold"
        if ref_mask is not None and level == ref_level:
            bad = (np.asarray(mask, dtype=bool) != np.asarray(ref_mask, dtype=bool)) & decided
            assert not bad.any()
