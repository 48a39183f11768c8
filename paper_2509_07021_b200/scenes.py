"""Seeded synthetic scenes and cameras for BASELINE.json configs[0..4].

The reference measures the product on real datasets that are not available
here; these generators restate the configs' distributions exactly
 with a FIXED draw order -- means, log-scales, quaternions,
opacity logits, base RGB, lobe axes, sharpness, amplitudes, masks -- from
``numpy.random.default_rng(seed)``, and everything is rounded to float32
(the oracle receives the float32 values upcast to float64).  Targets come
from the separate stream ``default_rng([seed, 1])``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .camera import Camera

L_LOBES = 3


@dataclass
class SceneArrays:
    """float32 SoA in the reference SceneParams layout (render.py:90-108),
    plus float soft masks: lobe_mask (N,L) and prim_mask (N)."""

    position: np.ndarray
    quat: np.ndarray
    log_scale: np.ndarray
    opacity: np.ndarray
    diffuse: np.ndarray
    axis_raw: np.ndarray
    sharpness: np.ndarray
    amplitude: np.ndarray
    lobe_mask: np.ndarray
    prim_mask: np.ndarray | None = None
    extra: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.position.shape[0])

    @property
    def n_lobes(self) -> int:
        return int(self.axis_raw.shape[1])

    def subset(self, idx) -> "SceneArrays":
        def s(a):
            return None if a is None else np.ascontiguousarray(a[idx])
        return SceneArrays(*(s(getattr(self, f)) for f in FIELDS),
                           lobe_mask=s(self.lobe_mask), prim_mask=s(self.prim_mask))


FIELDS = ("position", "quat", "log_scale", "opacity", "diffuse", "axis_raw", "sharpness",
          "amplitude")


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def _unit_rows(v):
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def _common_tail(rng, n, means, log_scales):
    quat = _unit_rows(rng.normal(size=(n, 4)))
    opacity = _sigmoid(rng.normal(size=n))
    diffuse = rng.uniform(0.0, 1.0, size=(n, 3))
    axes = _unit_rows(rng.normal(size=(n, L_LOBES, 3)))
    sharp = np.exp(rng.uniform(np.log(1.0), np.log(50.0), size=(n, L_LOBES)))
    amp = rng.normal(0.0, 0.3, size=(n, L_LOBES, 3))
    return SceneArrays(position=_f32(means), quat=_f32(quat), log_scale=_f32(log_scales),
                       opacity=_f32(opacity), diffuse=_f32(diffuse), axis_raw=_f32(axes),
                       sharpness=_f32(sharp), amplitude=_f32(amp),
                       lobe_mask=np.ones((n, L_LOBES), np.float32), prim_mask=None)


def orbit_camera(radius, azimuth, elevation, width, height, fov_deg, target=(0.0, 0.0, 0.0)):
    """Orbit camera in the viewer convention (frontend camera.ts:91-101):
    vertical FoV, fx = fy = (H/2)/tan(FoV/2), looking at the target, +z up."""
    t = np.asarray(target, dtype=np.float64)
    eye = t + radius * np.array([np.cos(elevation) * np.cos(azimuth),
                                 np.cos(elevation) * np.sin(azimuth), np.sin(elevation)])
    f = 0.5 * height / np.tan(np.radians(fov_deg) / 2.0)
    return Camera.look_at(eye, t, up=(0.0, 0.0, 1.0), fx=f, fy=f, width=width, height=height)


def config0(seed: int = 0, n: int = 10_000):
    """CPU-ref plumbing scene (configs[0]): 10k, 256x256, FoV 60, eye (3,0,0)."""
    rng = np.random.default_rng(seed)
    means = rng.uniform(-1.0, 1.0, size=(n, 3))
    ls = rng.normal(-3.5, 0.5, size=(n, 3))
    scene = _common_tail(rng, n, means, ls)
    f = 0.5 * 256 / np.tan(np.radians(60.0) / 2.0)
    cam = Camera.look_at((3.0, 0.0, 0.0), (0.0, 0.0, 0.0), up=(0.0, 0.0, 1.0), fx=f, fy=f,
                         width=256, height=256)
    return scene, [cam]


def config1(seed: int = 0, n: int = 200_000):
    """Forward-only pruned scene (configs[1]): prim mask Bernoulli(0.6), K~U{0..3} lobes."""
    rng = np.random.default_rng(seed)
    means = rng.uniform(-1.0, 1.0, size=(n, 3))
    ls = rng.normal(-3.5, 0.5, size=(n, 3))
    scene = _common_tail(rng, n, means, ls)
    scene.prim_mask = _f32(rng.uniform(size=n) < 0.6)
    k = rng.integers(0, L_LOBES + 1, size=n)
    scene.lobe_mask = _f32(np.arange(L_LOBES)[None, :] < k[:, None])
    cam = orbit_camera(3.0, -np.pi / 2, 0.25, 1280, 720, 50.0)
    return scene, [cam]


def config2(seed: int = 0, n: int = 1_000_000, n_cams: int = 64):
    """Multi-view forward batch (configs[2], the headline): 1M Gaussians in 64
    clusters (sigma 0.15), log-scales N(-4, 0.6); 64 cameras at radius 3.5,
    1920x1080, FoV 60, elevations 0.2 + 0.3 sin(2 pi 3k/64)."""
    rng = np.random.default_rng(seed)
    centres = rng.uniform(-1.0, 1.0, size=(64, 3))
    label = rng.integers(0, 64, size=n)
    means = centres[label] + rng.normal(0.0, 0.15, size=(n, 3))
    ls = rng.normal(-4.0, 0.6, size=(n, 3))
    scene = _common_tail(rng, n, means, ls)
    cams = [orbit_camera(3.5, 2 * np.pi * k / 64, 0.2 + 0.3 * np.sin(2 * np.pi * 3 * k / 64),
                         1920, 1080, 60.0) for k in range(n_cams)]
    return scene, cams


def config3(seed: int = 0, n: int = 500_000, n_views: int = 8):
    """Multi-view training step with soft pruning (configs[3]): cfg0 distributions,
    mask logits N(2,1) (returned in scene.extra), 8 views 1280x720 FoV 50."""
    rng = np.random.default_rng(seed)
    means = rng.uniform(-1.0, 1.0, size=(n, 3))
    ls = rng.normal(-3.5, 0.5, size=(n, 3))
    scene = _common_tail(rng, n, means, ls)
    prim_logit = rng.normal(2.0, 1.0, size=n)
    lobe_logit = rng.normal(2.0, 1.0, size=(n, L_LOBES))
    scene.extra["prim_logit"] = _f32(prim_logit)
    scene.extra["lobe_logit"] = _f32(lobe_logit)
    scene.prim_mask = _f32(_sigmoid(scene.extra["prim_logit"]))
    scene.lobe_mask = _f32(_sigmoid(scene.extra["lobe_logit"]))
    cams = [orbit_camera(3.0, 2 * np.pi * k / n_views, 0.25, 1280, 720, 50.0)
            for k in range(n_views)]
    return scene, cams


def config4(seed: int = 0, n: int = 5_000_000):
    """Stress frame (configs[4]): 70% N(0, 0.3^2 I), 30% U[-2,2]^3; one axis
    log-scale N(-2.5, 0.5), two N(-5, 0.5); 3840x2160 FoV 60, radius 2.5."""
    rng = np.random.default_rng(seed)
    n_c = int(round(0.7 * n))
    means = np.concatenate([rng.normal(0.0, 0.3, size=(n_c, 3)),
                            rng.uniform(-2.0, 2.0, size=(n - n_c, 3))])
    ls = rng.normal(-5.0, 0.5, size=(n, 3))
    big_axis = rng.integers(0, 3, size=n)
    ls[np.arange(n), big_axis] = rng.normal(-2.5, 0.5, size=n)
    scene = _common_tail(rng, n, means, ls)
    cam = orbit_camera(2.5, 0.0, 0.2, 3840, 2160, 60.0)
    return scene, [cam]


def target_image(seed: int, height: int, width: int, view: int = 0) -> np.ndarray:
    """U(0,1) target from the separate stream default_rng([seed, 1, view])."""
    rng = np.random.default_rng([seed, 1, view])
    return rng.uniform(0.0, 1.0, size=(height, width, 3)).astype(np.float32)


CONFIGS = {0: config0, 1: config1, 2: config2, 3: config3, 4: config4}
