"""CPU: pin the oracles to the reference.

- oracle/ref_dense.py (float64 restatement of the reference algorithm) must
  reproduce the fixtures the reference produced (tests/golden/) to float64
  round-off;
- oracle/sgs_tiled.cpp (the bit-exact authority for tile keys / order /
  ranges) must reproduce the reference images within 1e-4 and gradients
  within the composite criterion -- the same bar the GPU is held to.
"""

from pathlib import Path

import numpy as np
import pytest

from helpers import composite_ok, crop_fixture, golden, golden_camera, golden_scene
from oracle import ref_dense, tiled
from paper_2509_07021_b200 import scenes


def test_dense_matches_reference_crop_grads():
    d = golden("cfg0_crop_grads")
    s, cam = golden_scene(d), golden_camera(d)
    img = ref_dense.render(s, cam)
    np.testing.assert_allclose(img, d["img"], rtol=0, atol=1e-12)
    for lam in (0.0, 0.2):
        val, g, _ = ref_dense.loss_and_grads(s, cam, d["target"], lambda_ssim=lam)
        assert val == pytest.approx(float(d[f"loss_{lam}"]), rel=1e-12)
        for f in ("position", "quat", "log_scale", "opacity", "diffuse", "axis_raw", "sharpness",
                  "amplitude"):
            np.testing.assert_allclose(g[f], d[f"g{lam}_{f}"], rtol=1e-7, atol=1e-14)


def test_dense_matches_reference_acceptance_scenes():
    d = golden("accept_grads")
    cam = golden_camera(d)
    for seed in range(5):
        s = type("P", (), {})()
        for f in ("position", "quat", "log_scale", "opacity", "diffuse", "axis_raw", "sharpness",
                  "amplitude"):
            setattr(s, f, d[f"s{seed}_{f}"])
        s.lobe_mask = np.ones(d[f"s{seed}_sharpness"].shape)
        s.prim_mask = None
        img = ref_dense.render(s, cam)
        np.testing.assert_allclose(img, d[f"s{seed}_img"], atol=1e-12)
        val, g, _ = ref_dense.loss_and_grads(s, cam, d[f"s{seed}_target"])
        assert val == pytest.approx(float(d[f"s{seed}_loss"]), rel=1e-12)
        for f in ("position", "quat", "opacity", "axis_raw"):
            np.testing.assert_allclose(g[f], d[f"s{seed}_g_{f}"], rtol=1e-7, atol=1e-14)


def test_dense_mask_gradients_match_reference_fd():
    d = golden("masks_grads")
    s, cam = golden_scene(d), golden_camera(d)
    val, g, img = ref_dense.loss_and_grads(s, cam, d["target"])
    np.testing.assert_allclose(img, d["img"], atol=1e-12)
    # the reference saw opacity * prim_mask as its opacity: dL/do = m_p dL/do_eff
    np.testing.assert_allclose(g["opacity"], d["prim_mask"] * d["g_opacity"], rtol=1e-6, atol=1e-14)
    pick = d["pick"]
    np.testing.assert_allclose(g["prim_mask"][pick], d["fd_prim_mask"], rtol=2e-4, atol=1e-9)
    np.testing.assert_allclose(g["lobe_mask"][pick], d["fd_lobe_mask"], rtol=2e-4, atol=1e-9)


def test_dense_vram_model_matches_reference():
    d = golden("vram_model")
    cam = golden_camera(d)
    for k in range(4):
        q = d[f"k{k}_quat"].astype(np.float64)
        p = type("P", (), {})()
        p.position = d[f"k{k}_position"]
        p.quat = q
        p.log_scale = np.log(d[f"k{k}_scale"].astype(np.float64))
        p.opacity = d[f"k{k}_opacity"]
        p.diffuse = np.zeros_like(p.position)
        p.axis_raw = np.tile([0.0, 0.0, 1.0], (len(q), 1, 1))
        p.sharpness = np.zeros((len(q), 1))
        p.amplitude = np.zeros((len(q), 1, 3))
        p.lobe_mask = np.zeros((len(q), 1))
        for tile in (8, 16):
            vis, ent = ref_dense.vram_model_counts(p, cam, tile)
            assert 40 * vis + 12 * ent == int(d[f"k{k}_t{tile}"][1])


def test_tiled_oracle_full_frame_config0():
    d = golden("cfg0_full")
    s, cam = golden_scene(d), golden_camera(d)
    r = tiled.render(s, cam)
    err = np.abs(r.img - d["img"])
    assert err.max() <= 1e-4, err.max()
    assert r.n_visible == 10_000


@pytest.mark.parametrize("name", ["cfg1_crop", "cfg2_crop", "cfg3_crop", "cfg4_crop"])
def test_tiled_oracle_crops(name):
    scene, cam, ref_img = crop_fixture(name)
    r = tiled.render(scene, cam)
    assert np.abs(r.img - ref_img).max() <= 1e-4


@pytest.mark.parametrize("lam", [0.0, 0.2])
def test_tiled_oracle_gradients_match_reference(lam):
    d = golden("cfg0_crop_grads")
    s, cam = golden_scene(d), golden_camera(d)
    r = tiled.render(s, cam)
    _, dimg = ref_dense.loss_and_dimg(r.img.astype(np.float64), d["target"], lam)
    tiled.raster_backward(r, dimg)
    g = tiled.preprocess_backward(r)
    for f in ("position", "quat", "log_scale", "opacity", "diffuse", "axis_raw", "sharpness",
              "amplitude"):
        ok = composite_ok(g[f], d[f"g{lam}_{f}"])
        assert ok.all(), f"{f}: {np.count_nonzero(~ok)} elements"


def test_tiled_oracle_mask_gradients():
    d = golden("masks_grads")
    s, cam = golden_scene(d), golden_camera(d)
    r = tiled.render(s, cam)
    _, dimg = ref_dense.loss_and_dimg(r.img.astype(np.float64), d["target"])
    tiled.raster_backward(r, dimg)
    g = tiled.preprocess_backward(r)
    pick = d["pick"]
    assert composite_ok(g["prim_mask"][pick], d["fd_prim_mask"], rel=2e-3).all()
    assert composite_ok(g["lobe_mask"][pick], d["fd_lobe_mask"], rel=2e-3).all()
    assert composite_ok(g["opacity"], d["prim_mask"] * d["g_opacity"]).all()


def test_polynomial_exp_log_accuracy():
    xs = np.concatenate([np.linspace(-100, 80, 2001), [-1e-3, 0.0, 1e-7, 0.6931472]]).astype(np.float32)
    for x in xs:
        got, want = np.float32(tiled.expf(float(x))), np.exp(np.float64(x))
        if want > 1e-37:
            assert abs(got - want) <= 4 * np.spacing(np.float32(want)), x
    for x in np.geomspace(1e-30, 1e10, 1500).astype(np.float32):
        got, want = np.float32(tiled.logf(float(x))), np.log(np.float64(x))
        assert abs(got - want) <= 4 * np.spacing(np.float32(abs(want)) + np.float32(1e-30)), x
    assert tiled.logf(0.0) == -np.inf


def test_tiled_bins_are_a_stable_key_sort():
    d = golden("cfg0_full")
    s, cam = golden_scene(d), golden_camera(d)
    r = tiled.preprocess(s, cam)
    tiled.bin(r)
    k = r.keys
    assert np.all(k[1:] >= k[:-1])
    # ties in the 64-bit key resolve by lower primitive index
    tie = k[1:] == k[:-1]
    assert np.all(r.vals[1:][tie] > r.vals[:-1][tie])
    # ranges partition [0, E)
    nz = r.ranges[:, 1] > r.ranges[:, 0]
    assert r.ranges[nz, 1].sum() - r.ranges[nz, 0].sum() == r.n_entries
    assert np.all((k >> np.uint64(32)).astype(np.int64)[r.ranges[nz, 0]] == np.flatnonzero(nz))


@pytest.mark.parametrize("cfg", [1, 3])
def test_float32_key_order_inverts_pairs_and_the_residual_order_does_not(cfg):
    """SURVEY App. B depth-swap bound on the CPU restatement (bit-identical to
    the GPU preprocess): the float32 depth key alone inverts hundreds of
    pairs relative to the reference's float64 argsort (render.py:307); the
    build's order (ties by the float64 residual) inverts none."""
    import sys
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from swap_bound import f64_depth, swap_bound
    scene, cams = scenes.CONFIGS[cfg]()
    cam = cams[0]
    r = tiled.preprocess(scene, cam)
    z = f64_depth(scene.position, cam)
    args = (z, r.depth_bits, r.rect, r.tiles_touched, r.records, cam.width, cam.height)
    f32 = swap_bound(*args, floor=1.0)   # counts only
    exact = swap_bound(*args, floor=1.0, depth_res=r.depth_res)
    assert f32["inverted_pairs"] > 100 and f32["overlapping_pairs"] > 10
    assert exact["inverted_pairs"] == 0
