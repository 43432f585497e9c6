"""Round-2 behaviour: scene cache invalidation, render_dense's reused tile lists
and zero-channel frames, the relevancy-fusion rule of the C ABI."""

import numpy as np
import pytest

from conftest import make_camera, random_scene


def test_relevancy_fused_rule():
    """sf_relevancy_fused (pure host query): fused for the tensor-core splat with 4
    canonicals and for shapes the legacy blend serves; from the map otherwise."""
    from paper_2507_07136_b200 import _native as N
    lib = N.load()
    assert lib.sf_relevancy_fused(3, 64, 4, 4) == 1
    assert lib.sf_relevancy_fused(3, 64, 4, 9) == 0     # tensor-core splat, 9 canonicals
    assert lib.sf_relevancy_fused(1, 16, 4, 3) == 1     # legacy blend (L != 64) fuses any count
    assert lib.sf_relevancy_fused(4, 64, 4, 4) == 0     # 256 channels span several CTAs


@pytest.mark.gpu
def test_scene_cache_reuploads_reassigned_arrays(rng):
    import paper_2507_07136_b200 as sf
    from paper_2507_07136_b200.device import device_scene, invalidate
    scene = random_scene(rng, 800, num_levels=3, L=64, K=4, D=64)
    cam = make_camera(64, 48)
    first = sf.splat_multilevel(scene, cam).data
    ds0 = device_scene(scene)
    assert device_scene(scene) is ds0                      # unchanged: cached
    scene.opacities = np.clip(scene.opacities * 0.5, 0.0, 1.0).astype(np.float32)  # reassigned array
    ds1 = device_scene(scene)
    assert ds1 is not ds0
    second = sf.splat_multilevel(scene, cam).data
    assert not np.array_equal(first, second)
    scene.opacities[:] = 0.0                               # in place: needs invalidate()
    invalidate(scene)
    assert np.abs(sf.splat_multilevel(scene, cam).data).max() == 0.0


@pytest.mark.gpu
def test_render_dense_reused_lists_equal_single_pass_renders(rng):
    """40 channels = 3 passes sharing the first pass's binning; each channel
    slice equals its own one-pass render bit for bit."""
    import paper_2507_07136_b200 as sf
    scene = random_scene(rng, 1500, num_levels=1, L=16, K=4, D=8)
    cam = make_camera(80, 56)
    vals = rng.random((scene.num_gaussians, 40))
    fb, stats = sf.render_dense(scene, cam, vals, with_stats=True)
    for c0, c1 in ((0, 16), (16, 32), (32, 40)):
        part, pst = sf.render_dense(scene, cam, vals[:, c0:c1], with_stats=True)
        np.testing.assert_array_equal(fb.data[:, :, c0:c1], part.data)
        np.testing.assert_array_equal(stats.final_transmittance, pst.final_transmittance)
        assert stats.pairs_blended == pst.pairs_blended


@pytest.mark.gpu
def test_render_dense_zero_channels_is_a_real_frame(rng):
    """C = 0 still projects, bins and blends: the transmittance and pair count
    are the frame's (equal to the sparse splat's), not placeholders."""
    import paper_2507_07136_b200 as sf
    scene = random_scene(rng, 1200, num_levels=1, L=16, K=4, D=8)
    cam = make_camera(72, 40)
    fb, stats = sf.render_dense(scene, cam, np.zeros((scene.num_gaussians, 0)), with_stats=True)
    assert fb.data.shape == (40, 72, 0)
    _, ref = sf.splat_multilevel(scene, cam, with_stats=True)
    assert stats.pairs_blended == ref.pairs_blended > 0
    np.testing.assert_allclose(stats.final_transmittance, ref.final_transmittance, atol=1e-6)
    assert stats.final_transmittance.min() < 1.0


@pytest.mark.gpu
def test_device_topk_and_adam_match_numpy():
    """materialize / normalize_coefficients (k_train_plan) and OptimState.step
    (k_train_adam) against numpy restatements of train.py:79-139."""
    import paper_2507_07136_b200 as sf
    from paper_2507_07136_b200 import train as T
    rng = np.random.default_rng(5)
    lg = rng.standard_normal((2, 300, 64)) * 3
    lg[0, 0, 9] = lg[0, 0, 5]  # an exact tie: the lower index first (stable argsort of -p)
    idx, vals = T._device_topk(lg, 4)
    p = np.exp(lg - lg.max(-1, keepdims=True))
    p /= p.sum(-1, keepdims=True)
    ref = np.sort(np.argsort(-p, axis=-1, kind="stable")[..., :4], axis=-1)
    assert np.array_equal(idx, ref)
    kept = np.take_along_axis(p, ref, -1)
    kept /= kept.sum(-1, keepdims=True)
    assert np.abs(vals - kept).max() <= 1e-6
    c = sf.normalize_coefficients(lg[1, 7], 4)
    assert np.array_equal(c.indices, ref[1, 7]) and np.abs(c.values - kept[1, 7]).max() <= 1e-6
    # Adam: two steps on both parameter groups
    fld = T.TrainableField(logits=lg.copy(), codebooks=rng.standard_normal((2, 64, 8)))
    opt = T.OptimState(0.05, 0.02, 0.9, 0.999, 1e-8)
    ref_p = [fld.logits.copy(), fld.codebooks.copy()]
    m = [np.zeros_like(x) for x in ref_p]
    v = [np.zeros_like(x) for x in ref_p]
    for t in (1, 2):
        g = T.Gradients(logits=rng.standard_normal(lg.shape), codebooks=rng.standard_normal((2, 64, 8)))
        opt.step(fld, g)
        for k, (gr, lr) in enumerate(((g.logits, 0.05), (g.codebooks, 0.02))):
            m[k] += (1 - 0.9) * (gr - m[k])
            v[k] += (1 - 0.999) * (gr * gr - v[k])
            ref_p[k] -= lr * (m[k] / (1 - 0.9 ** t)) / (np.sqrt(v[k] / (1 - 0.999 ** t)) + 1e-8)
    assert np.abs(fld.logits - ref_p[0]).max() <= 1e-12
    assert np.abs(fld.codebooks - ref_p[1]).max() <= 1e-12
