"""The frame path's per-tile depth sort over every list-size class.

k_tile_sort_depth (sf_binning.cu) sorts each tile's list with one of five
kernels chosen by the list length: <= 2048, (2048, 3072], (3072, 4096],
(4096, 8192] and > 8192 entries (split sort); the mid-size classes run on a
side stream concurrently with the <= 2048 class.  The reference orders each
tile list by (depth, id) (projection.py:396, 443-449); a wrong order changes
the blend.  This scene puts a chosen number of small Gaussians in each tile
of a 4 x 3 tile image so that every class is exercised in one frame, and the
frame's coefficient map, final transmittance and pair count must match the
oracle's (same tolerances as tests/test_gpu_parity.py).
"""

import numpy as np
import pytest

import paper_2507_07136_b200 as sf
from conftest import make_camera, random_scene
from oracle import oracle as O

pytestmark = pytest.mark.gpu

W_TOL = 2e-6
T_TOL = 1e-6
# per-tile Gaussian counts (row-major over the 4 x 3 tiles): every class, an empty tile
WANT = [1500, 2500, 2900, 3500, 4000, 6000, 9000, 500, 0, 100, 2200, 3100]
CLASSES = [(1, 2048), (2049, 3072), (3073, 4096), (4097, 8192), (8193, 1 << 30)]


def _class_scene(rng):
    W, H = 64, 48
    cam = make_camera(W, H)
    pool = random_scene(rng, num_gaussians=160_000, num_levels=1, L=16, K=4, D=8, image_extent=1.0,
                        opacity_range=(0.01, 0.06))
    pool.scales[:] = rng.uniform(0.004, 0.012, pool.scales.shape).astype(np.float32)
    p = O.project_scene(pool, cam)
    rows = np.asarray(p.rows)
    tx = np.floor(p.means2d[:, 0] / 16).astype(np.int64)
    ty = np.floor(p.means2d[:, 1] / 16).astype(np.int64)
    inside = (tx >= 0) & (tx < 4) & (ty >= 0) & (ty < 3)
    pick = []
    for t, n in enumerate(WANT):
        cand = rows[inside & (ty * 4 + tx == t)]
        assert cand.size >= n, (t, cand.size, n)
        pick.append(cand[:n])
    order = np.sort(np.concatenate(pick))
    return pool.permuted(order), cam


def test_tile_sort_every_list_class_vs_oracle():
    rng = np.random.default_rng(7)
    scene, cam = _class_scene(rng)
    ob = O.bin_projected(O.project_scene(scene, cam), cam)
    lens = np.diff(np.asarray(ob.tile_offsets))
    for lo, hi in CLASSES:
        assert ((lens >= lo) & (lens <= hi)).any(), (lo, hi, lens.tolist())
    cm, st = sf.splat_multilevel(scene, cam, with_stats=True)
    ocm, ost = O.splat_multilevel(scene, cam, binning=ob, with_stats=True)
    assert st.pairs_blended == ost.pairs_blended
    assert np.abs(cm.data - ocm.data).max() <= W_TOL
    assert np.abs(st.final_transmittance - ost.final_transmittance).max() <= T_TOL
    # the frame is deterministic: a second render gives the same bytes
    again = sf.splat_multilevel(scene, cam).data
    assert again.tobytes() == cm.data.tobytes()
