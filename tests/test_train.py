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
