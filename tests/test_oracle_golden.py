"""The CPU oracle (oracle/) against the reference's own outputs (tests/golden/).

Pins the oracle before it is trusted as the parity checker: projection and
binning bitwise, blend / decode / relevancy / filter to 1e-12 (the only
difference is exp() ulps and BLAS summation order), level / point / mask
identical.
"""

import numpy as np
import pytest

from conftest import golden_names, load_golden
from oracle import oracle as O


@pytest.mark.parametrize("name", golden_names())
def test_projection_bitwise(name):
    scene, cam, z = load_golden(name)
    p = O.project_scene(scene, cam)
    assert p.count == z["p_means2d"].shape[0]
    for f in ("means2d", "inv_covs", "depths", "opacities", "source_ids", "rows"):
        assert getattr(p, f).tobytes() == z["p_" + f].tobytes(), f


@pytest.mark.parametrize("name", golden_names())
def test_binning_bytes(name):
    scene, cam, z = load_golden(name)
    b = O.bin_projected(O.project_scene(scene, cam), cam)
    assert b.canonical_bytes() == z["b_canonical_bytes"].tobytes()
    np.testing.assert_array_equal(b.tile_offsets, z["b_offsets"])


@pytest.mark.parametrize("name", golden_names())
def test_splat_decode(name):
    scene, cam, z = load_golden(name)
    cmap, st = O.splat_multilevel(scene, cam, with_stats=True)
    assert np.abs(cmap.data - z["cmap"]).max(initial=0) <= 1e-12
    assert np.abs(st.final_transmittance - z["final_t"]).max(initial=0) <= 1e-12
    assert st.pairs_blended == int(z["pairs"])
    assert st.channels_per_gaussian == int(z["channels"])
    feats = O.decode(cmap, scene.codebooks)
    for b in range(len(feats)):
        assert np.abs(feats[b] - z["features"][b]).max(initial=0) <= 1e-12


@pytest.mark.parametrize("name", golden_names(require_query=True))
def test_query(name):
    scene, cam, z = load_golden(name)
    if scene.num_gaussians == 0:
        pytest.skip("constant maps: covered by the GPU empty-scene test")
    res = O.query_pipeline(scene, cam, z["q_vector"], z["q_canon"], window=int(z["q_window"]))
    for b in range(len(res.raw_maps)):
        assert np.abs(res.raw_maps[b] - z["q_raw"][b]).max() <= 1e-12
        assert np.abs(res.level_maps[b] - z["q_filtered"][b]).max() <= 1e-12
    assert res.level == int(z["q_level"])
    assert res.point == tuple(int(v) for v in z["q_point"])
    mask, deg = O.segment(res.level_maps[res.level])
    assert deg == bool(z["q_degenerate"])
    np.testing.assert_array_equal(mask, z["q_mask"])


def test_config_a_binning():
    """10k Gaussians, 256x256 -- 175,770 pairs, byte-identical lists."""
    import os
    from conftest import GOLDEN
    from paper_2507_07136_b200 import synthetic
    z = np.load(os.path.join(GOLDEN, "configA_binning.npz"))
    scene = synthetic.make_scene(10_000)
    cam = synthetic.make_camera(256, 256)
    p = O.project_scene(scene, cam)
    assert p.means2d.tobytes() == z["p_means2d"].tobytes()
    assert p.inv_covs.tobytes() == z["p_inv_covs"].tobytes()
    b = O.bin_projected(p, cam)
    np.testing.assert_array_equal(b.tile_offsets, z["b_offsets"])
    np.testing.assert_array_equal(b.projected.source_ids[b.tile_entries], z["b_source_ids"])
    assert int(b.tile_offsets[-1]) == 175_770 == int(z["pairs"])
    cm, st = O.splat_multilevel(scene, cam, binning=b, with_stats=True)
    assert np.abs(cm.data[[5, 130]] - z["cmap_rows"]).max() <= 1e-12
