"""Device ADMM step (admm.py) -- SURVEY.md §8(f) row 3.

Known answers restated from the reference's test_prune.py:42-160 (top-k
projection, ties, operators, slot masks, dual update), the split-step
update order (test_prune.py:212-257) against a hand-stepped transcription
on our own gradients, and the whole run_state schedule against the
reference's own run (tests/golden/admm.npz, made by make_golden.py)."""

from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2509_07021_b200 import admm as A
from paper_2509_07021_b200.camera import Camera
from paper_2509_07021_b200.render import loss_and_grads_device
from paper_2509_07021_b200.rasterizer import GRAD_FIELDS

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


def cfg(ko, ks, **kw):
    return A.PrunerConfig(kappa=11 * ko + 7 * ks, kappa_o=ko, kappa_s=ks, **kw)


def np_(t):
    return t.detach().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("n", [1, 7, 1000, 70_001])
def test_topk_mask_matches_stable_argsort(n):
    rng = np.random.default_rng(n)
    s = np.round(rng.normal(size=n), 2)
    s[rng.integers(0, n, size=n // 5 + 1)] = 0.0
    s[rng.integers(0, n, size=n // 7 + 1)] = -0.0
    s[rng.integers(0, n, size=n // 11 + 1)] = -np.inf
    for k in sorted({0, 1, n // 3, n // 2, n - 1, n}):
        want = np.zeros(n, bool)
        want[np.argsort(-s, kind="stable")[:k]] = True
        got = A.topk_mask(torch.from_numpy(s), k).cpu().numpy()
        assert np.array_equal(got, want), (n, k)


def test_prox_known_answers():
    o, s = A.prox_project(np.array([0.9, 0.1, 0.5]), np.zeros(3), cfg(2, 0))
    assert np.array_equal(np_(o), np.array([0.9, 0.0, 0.5], np.float32).astype(np.float64))
    assert np.array_equal(np_(s), np.zeros(3))
    o, _ = A.prox_project(np.array([0.5, 0.5, 0.5, 0.5]), np.zeros(1), cfg(2, 0))
    assert np.array_equal(np_(o), [0.5, 0.5, 0.0, 0.0])            # ties keep lower index
    o, _ = A.prox_project(np.array([0.9, 0.8, 0.7]), np.zeros(1), cfg(2, 0, opacity_operator="importance"),
                          importance=np.array([0.0, 5.0, 9.0]))
    assert np.allclose(np_(o), [0.0, 0.8, 0.7])
    _, s = A.prox_project(np.zeros(1), np.array([5.0, 4.0]), cfg(0, 1, sharpness_operator="range"),
                          range_sharpness=np.array([5.0, 4.0]),
                          range_amplitude=np.array([[0.1, 0, 0], [9.0, 0, 0]]))
    assert np.array_equal(np_(s), [0.0, 4.0])
    _, s = A.prox_project(np.zeros(1), np.array([[0.5, 9.0]]), cfg(0, 1), slot_mask=np.array([[True, False]]))
    assert np.array_equal(np_(s), [[0.5, 0.0]])
    with pytest.raises(A.ConfigError):
        A.prox_project(np.zeros(3), np.zeros(3), cfg(4, 0))
    with pytest.raises(A.ConfigError):
        A.prox_project(np.zeros(3), np.zeros(3), cfg(0, 4))
    with pytest.raises(A.ConfigError):
        A.prox_project(np.ones(3), np.zeros(1), cfg(1, 0, opacity_operator="importance"))


def test_prox_exhaustive_idempotent_and_golden():
    rng = np.random.default_rng(0)
    for _ in range(10):
        n = int(rng.integers(1, 10))
        x = rng.normal(size=n).astype(np.float32).astype(np.float64)
        for k in range(n + 1):
            o, _ = A.prox_project(x, np.zeros(1), cfg(k, 0))
            want = np.zeros(n, bool)
            want[np.argsort(-np.abs(x), kind="stable")[:k]] = True
            assert np.array_equal(np_(o), np.where(want, x, 0.0))
            o2, _ = A.prox_project(o, np.zeros(1), cfg(k, 0))
            assert torch.equal(o, o2)
    d = np.load(GOLDEN / "admm.npz")
    o, s = A.prox_project(d["prox_o_in"], d["prox_s_in"], cfg(137, 611))
    assert np.array_equal(np_(o), d["prox_o"].astype(np.float32).astype(np.float64))
    assert np.array_equal(np_(s), d["prox_s"].astype(np.float32).astype(np.float64))


def _state(n=6):
    rng = np.random.default_rng(2)

    class P:
        pass
    p = P()
    p.position = rng.normal(size=(n, 3))
    p.quat = rng.normal(size=(n, 4))
    p.log_scale = rng.normal(-2, 0.3, size=(n, 3))
    p.opacity = rng.uniform(size=n)
    p.diffuse = rng.uniform(size=(n, 3))
    p.axis_raw = rng.normal(size=(n, 2, 3))
    p.sharpness = rng.uniform(1, 5, size=(n, 2))
    p.amplitude = rng.normal(size=(n, 2, 3))
    p.lobe_mask = np.ones((n, 2))
    return A.DevicePrunerState.init(p), rng


def test_dual_update_matches_script():
    st, rng = _state()
    st.proxy_o = torch.from_numpy(rng.normal(size=6).astype(np.float32)).cuda()
    st.proxy_s = torch.from_numpy(rng.normal(size=(6, 2)).astype(np.float32)).cuda()
    st.dual_o = torch.from_numpy(rng.normal(size=6).astype(np.float32)).cuda()
    st.dual_s = torch.from_numpy(rng.normal(size=(6, 2)).astype(np.float32)).cuda()
    want_o = st.dual_o + (st.params["opacity"] - st.proxy_o)
    want_s = st.dual_s + (st.params["sharpness"] - st.proxy_s)
    A.dual_update(st)
    assert torch.equal(st.dual_o, want_o) and torch.equal(st.dual_s, want_s)
    st.proxy_o = st.params["opacity"].clone()
    st.dual_o.zero_()
    A.dual_update(st)
    assert float(st.dual_o.abs().max()) == 0.0


def _golden_views(d):
    views = []
    for k in range(3):
        R, t = d[f"v{k}_cam_R"], d[f"v{k}_cam_t"]
        fx, fy, cx, cy, near = d[f"v{k}_cam_intr"]
        w, h = (int(v) for v in d[f"v{k}_cam_size"])
        views.append((Camera(rotation=R, translation=t, fx=fx, fy=fy, cx=cx, cy=cy, width=w, height=h,
                             near=near), d[f"v{k}_target"]))
    return views


def _golden_state(d):
    class P:
        pass
    p = P()
    for f in GRAD_FIELDS:
        setattr(p, f, d[f])
    p.lobe_mask = d["lobe_mask"]
    return A.DevicePrunerState.init(p)


def test_split_step_matches_hand_stepped_update():
    """test_prune.py:212-257 restated on this build's gradients: the sharpness
    gradient is taken at the already-updated opacity."""
    d = np.load(GOLDEN / "admm.npz")
    views = _golden_views(d)
    c = A.PrunerConfig(kappa=10 ** 9, kappa_o=0, kappa_s=0, delta=2e-2, prox_every=None)
    r = c.group_rates
    st = _golden_state(d)
    rng = np.random.default_rng(99)
    st.proxy_o.zero_()
    st.proxy_s.zero_()
    st.dual_o = torch.from_numpy(rng.normal(scale=0.01, size=st.dual_o.shape).astype(np.float32)).cuda()
    st.dual_s = torch.from_numpy(rng.normal(scale=0.01, size=st.dual_s.shape).astype(np.float32)).cuda()
    w = {k: v.clone() for k, v in st.params.items()}
    cam, tgt = views[0]
    tgt_t = torch.from_numpy(tgt).cuda()
    ref = A.DevicePrunerState(w, st.lobe_mask)
    _, g1 = loss_and_grads_device(ref.gaussians(), cam, tgt_t, c.loss_cfg, sync=False)
    o_new = torch.clamp(w["opacity"] - c.eta * r.opacity * (g1["opacity"] + c.delta_o * (
        w["opacity"] - st.proxy_o + st.dual_o)), 0.0, 1.0)
    w2 = dict(w, opacity=o_new)
    _, g2 = loss_and_grads_device(A.DevicePrunerState(w2, st.lobe_mask).gaussians(), cam, tgt_t, c.loss_cfg,
                                  sync=False)
    s_new = torch.clamp(w["sharpness"] - c.eta * r.sharpness * (g2["sharpness"] + c.delta_s * (
        w["sharpness"] - st.proxy_s + st.dual_s)), min=0.0)
    A.gradient_step(st, views[0], c)
    np.testing.assert_allclose(np_(st.params["opacity"]), np_(o_new), atol=1e-6)
    np.testing.assert_allclose(np_(st.params["sharpness"]), np_(s_new), atol=1e-6)
    for name in ("position", "quat", "log_scale", "diffuse", "axis_raw", "amplitude"):
        want = w[name] - c.eta * getattr(r, name) * g1[name]
        np.testing.assert_allclose(np_(st.params[name]), np_(want), atol=1e-6)


@pytest.mark.parametrize("op", ["sharpness", "range"])
def test_run_state_matches_reference_run(op):
    """The whole schedule against the reference's own prune.run_state."""
    d = np.load(GOLDEN / "admm.npz")
    views = _golden_views(d)
    kappa, ko, ks = (int(v) for v in d[f"{op}_kappa"])
    c = A.PrunerConfig(kappa=kappa, kappa_o=ko, kappa_s=ks, delta=5e-3, iters=8, prox_every=3,
                       sharpness_operator=op, seed=1)
    st = _golden_state(d)
    trace = A.run_state(st, views, c)
    want = d[f"{op}_trace"]
    got = np.array([[t.iteration, t.loss, t.residual_o, t.residual_s, t.active_primitives,
                     t.active_lobes, t.budget_units] for t in trace])
    assert np.array_equal(got[:, [0, 4, 5, 6]], want[:, [0, 4, 5, 6]])   # schedule, budget exact
    np.testing.assert_allclose(got[:, 1:4], want[:, 1:4], rtol=2e-4, atol=1e-6)
    # kept supports identical, values within float32 training tolerance
    assert np.array_equal(np_(st.proxy_o) != 0, d[f"{op}_proxy_o"] != 0)
    assert np.array_equal(np_(st.proxy_s) != 0, d[f"{op}_proxy_s"] != 0)
    for f in GRAD_FIELDS:
        np.testing.assert_allclose(np_(st.params[f]), d[f"{op}_{f}"], rtol=1e-4, atol=2e-5, err_msg=f)
    np.testing.assert_allclose(np_(st.dual_o), d[f"{op}_dual_o"], rtol=1e-4, atol=2e-5)
    np.testing.assert_allclose(np_(st.dual_s), d[f"{op}_dual_s"], rtol=1e-4, atol=2e-5)


def test_budget_holds_and_reproducible():
    """Two runs of the importance-operator schedule are BITWISE identical:
    the importance scores are exact fixed-point sums (render.py:406-407 ->
    top-k ties by index, prune.py:204) and the gradient steps use the
    deterministic backward (order-independent fixed-point raster sums)."""
    d = np.load(GOLDEN / "admm.npz")
    views = _golden_views(d)
    c = A.PrunerConfig(kappa=11 * 50 + 7 * 200, kappa_o=50, kappa_s=200, iters=6, prox_every=2, seed=3,
                       opacity_operator="importance")
    runs = []
    for _ in range(2):
        st = _golden_state(d)
        trace = A.run_state(st, views, c)
        assert all(t.budget_units <= c.kappa for t in trace)
        assert int(torch.count_nonzero(st.params["opacity"])) <= 50
        runs.append((trace, st.to_numpy(), np_(st.proxy_o), np_(st.dual_o), np_(st.dual_s)))
    assert [t.loss for t in runs[0][0]] == [t.loss for t in runs[1][0]]
    assert [(t.residual_o, t.residual_s, t.active_primitives, t.active_lobes) for t in runs[0][0]] == \
        [(t.residual_o, t.residual_s, t.active_primitives, t.active_lobes) for t in runs[1][0]]
    for f in GRAD_FIELDS:
        assert np.array_equal(runs[0][1][f], runs[1][1][f]), f
    for a, b in zip(runs[0][2:], runs[1][2:]):
        assert np.array_equal(a, b)


def test_importance_is_bitwise_reproducible_across_streams():
    """The multi-view importance (views on 4 streams, atomics in any order)
    gives the same bits every time, and equals the one-stream result."""
    from paper_2509_07021_b200 import render as R
    from paper_2509_07021_b200 import scenes
    scene, cams = scenes.config0(n=4000)
    views = [cams[0].crop(0, 0, 128, 128), cams[0].crop(64, 32, 160, 96), cams[0].crop(10, 150, 200, 80),
             cams[0].crop(0, 0, 256, 256)]
    p = R.SceneParams(**{f: getattr(scene, f).astype(np.float64) for f in GRAD_FIELDS},
                      lobe_mask=scene.lobe_mask)
    a = R.accumulate_importance_params(p, views, streams=4)
    b = R.accumulate_importance_params(p, views, streams=4)
    c = R.accumulate_importance_params(p, views, streams=1)
    assert np.array_equal(a, b) and np.array_equal(a, c)
    assert np.count_nonzero(a) > 100


def test_deterministic_backward_is_bitwise_and_matches_default():
    from paper_2509_07021_b200 import scenes
    from paper_2509_07021_b200.rasterizer import GaussianTensors, Rasterizer
    from paper_2509_07021_b200.loss import image_loss
    scene, cams = scenes.config1(n=50_000)
    cam = cams[0].crop(320, 180, 640, 360)
    rast = Rasterizer()
    g = GaussianTensors.from_arrays(scene)
    fr = rast.forward(g, cam)
    tgt = torch.from_numpy(scenes.target_image(1, cam.height, cam.width)).cuda()
    _, dimg, _ = image_loss(fr.img, tgt, A.LossConfig(), grad="f32")
    d1 = rast.backward_raster(g, fr, dimg, deterministic=True)
    d2 = rast.backward_raster(g, fr, dimg, deterministic=True)
    f = rast.backward_raster(g, fr, dimg)
    assert torch.equal(d1, d2)
    ref = f.double()
    err = (d1.double() - ref).abs()
    assert bool((err <= 1e-5 * ref.abs() + 1e-6 * ref.abs().max()).all())


def test_nonfinite_gradient_is_reported_after_the_sync_free_steps():
    """prune.py:151-159: the first bad primitive is named; the state keeps the
    values it had when the bad gradient appeared (updates masked off)."""
    d = np.load(GOLDEN / "admm.npz")
    views = _golden_views(d)
    st = _golden_state(d)
    st.params["position"][7, 0] = float("nan")
    before = {f: t.clone() for f, t in st.params.items()}
    c = A.PrunerConfig(kappa=10 ** 9, kappa_o=0, kappa_s=0, iters=4, prox_every=2, seed=0)
    with pytest.raises(A.NumericalFailure) as e:
        A.run_state(st, views, c)
    assert e.value.index == 7
    for f in GRAD_FIELDS:
        if f not in ("opacity", "sharpness"):   # clamps still run (no-ops on unchanged values)
            assert torch.equal(torch.nan_to_num(st.params[f]), torch.nan_to_num(before[f])), f
