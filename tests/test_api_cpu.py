"""Host-side logic of the drop-in API that runs without a GPU."""

import numpy as np
import pytest

from conftest import make_camera, random_scene
from paper_2507_07136_b200 import (Camera, CameraPose, Codebook, QueryEmbedding, RelevancyMap,
                                   ResourceLimitError, SceneConfig, ValidationError,
                                   check_render_budget, iou, synthetic)
from paper_2507_07136_b200.sparse_splat import StageTimings, timing_csv_row


def test_errors_hierarchy_matches_reference():
    from paper_2507_07136_b200 import errors as E
    assert issubclass(E.ValidationError, E.SplatfieldError)
    assert issubclass(E.TruncatedFileError, E.FormatError)
    assert issubclass(E.ResourceLimitError, E.SplatfieldError)


def test_camera_validation():
    with pytest.raises(ValidationError):
        Camera(rotation=np.eye(3), translation=np.zeros(3), fx=-1, fy=1, cx=0, cy=0, width=8, height=8)
    with pytest.raises(ValidationError):
        Camera.look_at((0, 0, 0), (0, 0, 0))
    pose = CameraPose(position=(1, 2, -3), look_at=(0, 0, 0), fov_y_deg=40)
    cam = pose.to_camera()
    assert cam.width == 64 and cam.fx > 0


def test_scene_config_and_codebook_validation():
    with pytest.raises(ValidationError):
        SceneConfig(K=5, L=4)
    with pytest.raises(ValidationError):
        Codebook(np.zeros((0, 3)))


def test_scene_validate(rng):
    s = random_scene(rng, num_gaussians=20, num_levels=2)
    s.validate()
    bad = s.permuted(np.arange(20))
    bad.coeff_indices = bad.coeff_indices.copy()
    bad.coeff_indices[0, 0, -1] = 40
    with pytest.raises(ValidationError):
        bad.validate()


def test_render_budget():
    check_render_budget(64, 64, 192, 1 << 27)
    with pytest.raises(ResourceLimitError):
        check_render_budget(1440, 1080, 192, 1 << 27)


def test_query_embedding_and_relevancy_map_types():
    with pytest.raises(ValidationError):
        QueryEmbedding("q", np.zeros((2, 2)))
    with pytest.raises(ValidationError):
        QueryEmbedding("q", np.array([np.inf]))
    with pytest.raises(ValidationError):
        RelevancyMap(np.zeros(3), "q", 0)
    m = RelevancyMap(np.ones((2, 3)), "q", 1)
    assert m.data.dtype == np.float64 and m.shape == (2, 3)


def test_iou_conventions():
    e = np.zeros((3, 3), dtype=bool)
    assert iou(e, e) == 1.0
    a = e.copy(); a[0, 0] = True
    assert iou(a, e) == 0.0


def test_timing_csv():
    t = StageTimings(render_ms=2.0, decode_ms=0.1, post_ms=0.5)
    row = timing_csv_row("scene0", 64, 64, 64, 4, 3, t)
    assert row.split(",")[:6] == ["scene0", "64", "64", "64", "4", "3"]
    assert t.total_ms == pytest.approx(2.6)


def test_synthetic_generator_matches_survey_statistics():
    """10k Gaussians -> 175,770 (tile, Gaussian) pairs."""
    from oracle import oracle as O
    s = synthetic.make_scene(10_000)
    cam = synthetic.make_camera(256, 256)
    b = O.bin_projected(O.project_scene(s, cam), cam)
    assert b.tiles_x * b.tiles_y == 256
    assert int(b.tile_offsets[-1]) == 175_770


def test_compute_paths_fail_loudly_without_cuda(rng):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2507_07136_b200 import SplatfieldError, splat_multilevel
    s = random_scene(rng, num_gaussians=5)
    with pytest.raises(SplatfieldError):
        splat_multilevel(s, make_camera())
