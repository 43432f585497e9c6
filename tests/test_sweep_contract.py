"""query_sweep's argument contract (raised before any device work, like
query_pipeline's, sparse_splat.py:243-297): runs without a GPU."""

import numpy as np
import pytest

import paper_2507_07136_b200 as sf
from conftest import make_camera, random_scene


def test_query_sweep_validates_before_work(rng):
    scene = random_scene(rng, 50, num_levels=2, L=16, K=4, D=8)
    cam = make_camera(32, 24)
    q = [sf.QueryEmbedding("a", rng.standard_normal(8)), sf.QueryEmbedding("b", rng.standard_normal(8))]
    canon = rng.standard_normal((3, 8))
    with pytest.raises(sf.ValidationError):
        sf.query_sweep(scene, cam, q, canon, window=4)           # even window
    with pytest.raises(sf.ValidationError):
        sf.query_sweep(scene, cam, q, np.zeros((0, 8)))          # no canonical
    with pytest.raises(sf.ValidationError):
        sf.query_sweep(scene, cam, q, rng.standard_normal((3, 7)))  # D mismatch
    with pytest.raises(sf.ValidationError):
        sf.query_sweep(scene, cam, [sf.QueryEmbedding("c", rng.standard_normal(5))], canon)
    with pytest.raises(sf.ValidationError):
        sf.query_sweep(scene, cam, q, canon, tile_size=8)        # kernels are 16x16-tile
    with pytest.raises(sf.ResourceLimitError):
        sf.query_sweep(scene, cam, q, canon, max_elements=10)    # render budget


def test_query_stream_validates_before_work(rng):
    scene = random_scene(rng, 50, num_levels=2, L=16, K=4, D=8)
    with pytest.raises(sf.ValidationError):
        sf.QueryStream(scene, 32, 24, np.zeros((0, 8)))
    with pytest.raises(sf.ValidationError):
        sf.QueryStream(scene, 32, 24, rng.standard_normal((2, 7)))
    with pytest.raises(sf.ValidationError):
        sf.QueryStream(scene, 32, 24, rng.standard_normal((2, 8)), window=6)
