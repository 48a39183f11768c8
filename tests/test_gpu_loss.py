"""Fused SSIM + L1 loss kernel (csrc/loss.cu) against the float64 NumPy
restatement of the reference loss (oracle/ref_dense.py loss_and_dimg, which
follows render.py:433-509) and the reference's known answers
(test_render.py:186-238 restated)."""

import dataclasses

import numpy as np
import pytest
import torch

from oracle import ref_dense
from paper_2509_07021_b200.loss import image_loss
from paper_2509_07021_b200.render import LossConfig

pytestmark = pytest.mark.gpu


def _oracle(img, tgt, cfg):
    return ref_dense.loss_and_dimg(img, tgt, cfg.lambda_ssim, cfg.window, cfg.sigma, cfg.c1, cfg.c2)


@pytest.mark.parametrize("shape", [(16, 16), (37, 45), (8, 33), (1, 1), (130, 71)])
@pytest.mark.parametrize("lam", [0.0, 0.2, 1.0])
def test_loss_f64_matches_oracle(shape, lam):
    rng = np.random.default_rng(hash(shape) % 1000 + int(lam * 10))
    img = rng.uniform(0, 1, shape + (3,))
    tgt = rng.uniform(0, 1, shape + (3,))
    tgt[: shape[0] // 2] = img[: shape[0] // 2]  # a flat-difference region (sign(0) = 0)
    cfg = LossConfig(lambda_ssim=lam)
    out, d, _ = image_loss(torch.from_numpy(img).cuda(), torch.from_numpy(tgt).cuda(), cfg, grad="f64")
    val, grad = _oracle(img, tgt, cfg)
    assert float(out[0]) == pytest.approx(val, rel=1e-12, abs=1e-15)
    np.testing.assert_allclose(d.cpu().numpy(), grad, rtol=1e-9, atol=1e-15)


def test_loss_f32_inputs_and_grad():
    rng = np.random.default_rng(7)
    img = rng.uniform(0, 1, (72, 128, 3)).astype(np.float32)
    tgt = rng.uniform(0, 1, (72, 128, 3)).astype(np.float32)
    cfg = LossConfig()
    out, d, _ = image_loss(torch.from_numpy(img).cuda(), torch.from_numpy(tgt).cuda(), cfg, grad="f32")
    val, grad = _oracle(img.astype(np.float64), tgt.astype(np.float64), cfg)
    assert float(out[0]) == pytest.approx(val, rel=1e-12)
    assert d.dtype == torch.float32
    np.testing.assert_allclose(d.cpu().numpy(), grad, rtol=1e-6, atol=1e-12)


def test_custom_window_and_constants():
    rng = np.random.default_rng(3)
    img = rng.uniform(0, 1, (40, 50, 3))
    tgt = np.clip(img + rng.normal(0, 0.05, img.shape), 0, 1)
    cfg = LossConfig(lambda_ssim=0.5, window=7, sigma=1.0, c1=1e-3, c2=2e-3)
    out, d, _ = image_loss(torch.from_numpy(img).cuda(), torch.from_numpy(tgt).cuda(), cfg, grad="f64")
    val, grad = _oracle(img, tgt, cfg)
    assert float(out[0]) == pytest.approx(val, rel=1e-12)
    np.testing.assert_allclose(d.cpu().numpy(), grad, rtol=1e-9, atol=1e-15)


def test_known_answers_and_fd():
    """test_render.py:186-238: loss(x, x) = 0, SSIM(x, x) = 1, L1 of a constant
    offset, and the SSIM gradient against central differences."""
    from paper_2509_07021_b200 import render as R
    rng = np.random.default_rng(11)
    img = rng.uniform(0, 1, (12, 12, 3))
    assert R.loss(img, img) == pytest.approx(0.0, abs=1e-12)
    assert R.ssim(img, img) == pytest.approx(1.0, abs=1e-12)
    assert R.loss(np.full((12, 12, 3), 0.4), np.full((12, 12, 3), 0.5),
                  R.LossConfig(lambda_ssim=0.0)) == pytest.approx(0.1)
    a = rng.uniform(0, 1, (10, 11, 3))
    b = rng.uniform(0, 1, (10, 11, 3))
    g, smap = R._ssim_grad(a, b, R.LossConfig())
    assert smap.shape == a.shape and float(smap.mean()) == pytest.approx(R.ssim(a, b), rel=1e-12)
    h = 1e-6
    for idx in [(0, 0, 0), (5, 5, 1), (9, 10, 2), (3, 7, 0)]:
        up, dn = a.copy(), a.copy()
        up[idx] += h
        dn[idx] -= h
        fd = (R.ssim(up, b) - R.ssim(dn, b)) / (2 * h)
        assert g[idx] == pytest.approx(fd, rel=1e-5, abs=1e-9)
    with pytest.raises(ValueError):
        R.loss(np.zeros((4, 4, 3)), np.zeros((5, 4, 3)))


def test_ssim_map_matches_oracle_terms():
    rng = np.random.default_rng(5)
    img = rng.uniform(0, 1, (33, 20, 3))
    tgt = rng.uniform(0, 1, (33, 20, 3))
    cfg = dataclasses.replace(LossConfig(), lambda_ssim=1.0)
    out, _, smap = image_loss(torch.from_numpy(img).cuda(), torch.from_numpy(tgt).cuda(), cfg,
                              grad=None, ssim_map=True)
    val, _ = _oracle(img, tgt, cfg)
    assert float(out[2]) == pytest.approx(1.0 - val, rel=1e-12)
    assert float(smap.mean()) == pytest.approx(float(out[2]), rel=1e-12)
    assert float(out[1]) == pytest.approx(np.abs(img - tgt).mean(), rel=1e-12)
