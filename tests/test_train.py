"""GPU training step (train.py) against the reference's forward_loss / backward
(tests/golden/train_s8.npz: validity mask + cosine term; train_s9: neither).

Tolerances: the coefficient map is blended in fp32 from fp32-rounded
coefficient values, so the loss matches to 1e-5 relative and the gradients to
1e-4 of their largest entry (the reference is fp64 throughout)."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["train_s8", "train_s9"])
def test_forward_backward_vs_reference(name):
    from paper_2507_07136_b200 import train as T
    scene, cam, z = load_golden(name)
    fld = T.TrainableField(logits=z["t_logits"].copy(), codebooks=z["t_codebooks"].copy())
    mask = z["t_mask"] if z["t_mask"].size else None
    batch = T.TrainingBatch(camera=cam, targets=z["t_targets"], mask=mask)
    cfg = T.TrainConfig(cosine_weight=float(z["t_cosine"]))
    loss, cache = T.forward_loss(fld, scene, batch, cfg)
    assert abs(loss - float(z["t_loss"])) <= 1e-5 * abs(float(z["t_loss"]))
    cm = cache.coeff_maps.cpu().numpy().reshape(z["t_coeff_maps"].shape)
    assert np.abs(cm - z["t_coeff_maps"]).max() <= 2e-6
    g = T.backward(cache)
    for got, ref in ((g.logits, z["t_grad_logits"]), (g.codebooks, z["t_grad_codebooks"])):
        assert got.shape == ref.shape
        assert np.abs(got - ref).max() <= 1e-4 * np.abs(ref).max()


def test_optimizer_step_lowers_the_loss():
    from paper_2507_07136_b200 import train as T
    scene, cam, z = load_golden("train_s9")
    fld = T.TrainableField(logits=z["t_logits"].copy(), codebooks=z["t_codebooks"].copy())
    batch = T.TrainingBatch(camera=cam, targets=z["t_targets"])
    cfg = T.TrainConfig(lr_logits=0.05, lr_codebook=0.02)
    opt = T.OptimState(cfg.lr_logits, cfg.lr_codebook, cfg.beta1, cfg.beta2, cfg.eps)
    first, _ = T.forward_loss(fld, scene, batch, cfg)
    for _ in range(20):
        loss, cache = T.forward_loss(fld, scene, batch, cfg)
        opt.step(fld, T.backward(cache))
    assert loss < first


def test_train_field_vs_reference(tmp_path):
    """init_field (k-means seeding with the reference's draws, distances and
    means on the device) and train_field (6 Adam iterations over two batches,
    cosine term, a validity mask, a holdout) against the reference's
    (tests/golden/train_field_s10.npz)."""
    import paper_2507_07136_b200 as sf
    from paper_2507_07136_b200 import train as T
    from paper_2507_07136_b200.errors import ValidationError
    scene, _, z = load_golden("train_field_s10")
    cams = [sf.Camera.look_at(position=tuple(p), target=(0.0, 0.0, 0.0), fov_y_deg=45.0, width=40, height=32)
            for p in z["cams_pos"]]
    assert np.array_equal(cams[0].rotation, z["cam_R"]) and np.array_equal(cams[0].translation, z["cam_t"])
    batches = [T.TrainingBatch(camera=c, targets=z["t_targets"][i], mask=z["t_mask1"] if i == 1 else None)
               for i, c in enumerate(cams)]
    init = T.init_field(scene, batches[:2], seed=3)
    assert np.array_equal(init.logits, z["i_logits"])
    assert np.abs(init.codebooks - z["i_codebooks"]).max() <= 1e-12 * np.abs(z["i_codebooks"]).max()
    rnd = T.init_field(scene, batches[:2], seed=4, codebook_init="random")
    assert np.array_equal(rnd.codebooks, z["r_codebooks"])

    cfg = T.TrainConfig(lr_logits=0.05, lr_codebook=0.02, cosine_weight=0.25)
    res = T.train_field(scene, batches[:2], 6, cfg, seed=3, holdout=batches[2])
    curve, ref = np.array(res.loss_curve), z["f_curve"]
    assert curve.shape == ref.shape and np.array_equal(curve[:, 0], ref[:, 0])
    assert np.abs(curve[:, 1] - ref[:, 1]).max() <= 1e-5 * ref[:, 1].max()
    assert np.abs(curve[:, 2] - ref[:, 2]).max() <= 1e-4 * ref[:, 2].max()
    assert np.abs(np.array([res.holdout_initial, res.holdout_final]) - z["f_holdout"]).max() <= 1e-5 * z["f_holdout"].max()
    assert res.initial_loss == curve[0, 1] and res.final_loss == curve[-1, 1]
    assert np.abs(res.field.codebooks - z["f_codebooks"]).max() <= 1e-4 * np.abs(z["f_codebooks"]).max()
    assert np.abs(res.field.logits - z["f_logits"]).max() <= 1e-4 * np.abs(z["f_logits"]).max()
    # the materialised scene: top-K sets (a near-tie may flip) and renormalised values
    same = res.scene.coeff_indices == z["f_coeff_indices"]
    assert same.mean() >= 0.999
    both = same.all(axis=2)
    assert np.abs(res.scene.coeff_values[both] - z["f_coeff_values"][both]).max() <= 1e-4
    assert res.scene.positions is scene.positions  # geometry shared, never touched
    T.write_loss_curve(tmp_path / "curve.csv", res.loss_curve)
    lines = (tmp_path / "curve.csv").read_text().splitlines()
    assert lines[0] == "iter,loss,grad_norm" and len(lines) == 7
    # contract: iters=0 returns the input scene; no batches is an error
    assert T.train_field(scene, batches[:1], 0).scene is scene
    with pytest.raises(ValidationError):
        T.train_field(scene, [], 3)
