"""Drop-in replacement for the reference renderer module ``sgsplat.render``
(/root/reference/pkg/src/sgsplat/render.py), running on the B200.

Same names, signatures, argument meaning, return types and errors as the
reference; the work runs in libsgs.so (hand-written sm_100a CUDA) through the
C ABI, the L1/SSIM loss runs in the fused CUDA loss kernel (float64 statistics).  Inputs are the
reference's float64 numpy arrays; they are rounded to float32 at the
boundary (the GPU computes in fp32) and results come back as float64.

  render / _render_params          render.py:393-413
  accumulate_importance(_params)   render.py:416-428
  loss / ssim / psnr               render.py:464-496, 689-696
  _loss_and_dimg / _ssim_grad      render.py:469-509
  loss_and_grads / render_backward render.py:645-686
  _prepare / project               render.py:259-330
  Camera / SceneParams / GradientSet / LossConfig / Splat2D / quat_to_rot

Semantic difference, documented in DESIGN.md: pairs outside the
opacity-aware support (o G < 1e-7) are skipped; SURVEY.md §0.4 measures the
resulting image difference at 2.1e-7 (tolerance 1e-4).  ``_PIXEL_CHUNK`` is
accepted for compatibility and ignored (the tiled renderer has no chunks).
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass

import numpy as np
import torch

from . import _ffi
from .camera import Camera, to_sgs
from .loss import image_loss
from .rasterizer import GRAD_FIELDS, GaussianTensors, Rasterizer, device_to_host_f64

ALPHA_MAX = 0.99
T_CUTOFF = 1e-4
LOWPASS_FLOOR = 0.3
_PIXEL_CHUNK = 4096
# Gradient renders bin every primitive with at least this opacity's support:
# the reference blends every primitive into every pixel, so a primitive at
# opacity 0 (the pruning loop clamps there, prune.py:185) still has
# dL/do = sum G dL/dalpha (render.py:538-560) and can recover.  The support
# q <= 2 ln(1e-3 / 1e-7) (4.3 sigma) holds all but ~1e-4 of that sum.
GRAD_OPACITY_FLOOR = 1e-3
_CACHE_ELEMENTS = 32_000_000

__all__ = ["Camera", "Splat2D", "SceneParams", "GradientSet", "LossConfig", "ColorModelError",
           "quat_to_rot", "render", "_render_params", "accumulate_importance",
           "accumulate_importance_params", "loss", "ssim", "psnr", "_loss_and_dimg", "_ssim_grad",
           "loss_and_grads", "render_backward", "_prepare", "project"]


class ColorModelError(Exception):
    """Operation applied to a scene with the wrong color model (scene.py:52-53)."""


@dataclass
class Splat2D:
    """One projected primitive, ready for alpha blending (render.py:79-87)."""

    mean2d: np.ndarray
    cov2d: np.ndarray
    depth: float
    color: np.ndarray
    opacity: float


_PARAM_FIELDS = GRAD_FIELDS


@dataclass
class SceneParams:
    """Packed optimizer-space arrays (render.py:90-108): opacity and sharpness
    activated, scales log, quaternions / lobe axes free vectors normalized on
    use, ``lobe_mask`` marks real lobe slots (bool, or float soft masks)."""

    position: np.ndarray
    quat: np.ndarray
    log_scale: np.ndarray
    opacity: np.ndarray
    diffuse: np.ndarray
    axis_raw: np.ndarray
    sharpness: np.ndarray
    amplitude: np.ndarray
    lobe_mask: np.ndarray

    @property
    def n(self) -> int:
        return self.position.shape[0]

    @property
    def max_lobes(self) -> int:
        return self.axis_raw.shape[1]

    def copy(self) -> "SceneParams":
        return SceneParams(*(getattr(self, f).copy() for f in _PARAM_FIELDS),
                           lobe_mask=self.lobe_mask.copy())

    @staticmethod
    def from_scene(scene) -> "SceneParams":
        """Vectorised packing of an SG scene (any object with the reference
        Scene / GaussianPrimitive / SGLobe attributes)."""
        _require_sg(scene, "parameter packing")
        prims = list(scene.primitives)
        n = len(prims)
        lmax = int(scene.color_model.max_lobes)
        p = SceneParams(
            position=np.zeros((n, 3)), quat=np.zeros((n, 4)), log_scale=np.zeros((n, 3)),
            opacity=np.zeros(n), diffuse=np.zeros((n, 3)), axis_raw=np.zeros((n, lmax, 3)),
            sharpness=np.zeros((n, lmax)), amplitude=np.zeros((n, lmax, 3)),
            lobe_mask=np.zeros((n, lmax), dtype=bool))
        p.axis_raw[:, :, 2] = 1.0
        if n == 0:
            return p
        p.position[:] = np.stack([np.asarray(q.position, np.float32) for q in prims])
        p.quat[:] = np.stack([np.asarray(q.rotation, np.float32) for q in prims])
        p.log_scale[:] = np.log(np.stack([np.asarray(q.scale, np.float32) for q in prims])
                                .astype(np.float64))
        p.opacity[:] = [float(q.opacity) for q in prims]
        p.diffuse[:] = np.stack([np.asarray(q.diffuse, np.float32) for q in prims])
        for i, q in enumerate(prims):
            for j, lobe in enumerate(q.lobes):
                p.axis_raw[i, j] = lobe.axis
                p.sharpness[i, j] = lobe.sharpness
                p.amplitude[i, j] = lobe.amplitude
                p.lobe_mask[i, j] = True
        return p


@dataclass
class GradientSet:
    """Partials of the scalar loss, shaped like SceneParams (render.py:179-194)."""

    position: np.ndarray
    quat: np.ndarray
    log_scale: np.ndarray
    opacity: np.ndarray
    diffuse: np.ndarray
    axis_raw: np.ndarray
    sharpness: np.ndarray
    amplitude: np.ndarray

    @staticmethod
    def zeros_like(p) -> "GradientSet":
        return GradientSet(*(np.zeros_like(np.asarray(getattr(p, f), dtype=np.float64))
                             for f in _PARAM_FIELDS))


@dataclass(frozen=True)
class LossConfig:
    """(1-lambda)*L1 + lambda*(1-SSIM); SSIM uses an 11x11 Gaussian window."""

    lambda_ssim: float = 0.2
    window: int = 11
    sigma: float = 1.5
    c1: float = 0.01 ** 2
    c2: float = 0.03 ** 2


def _require_sg(scene, what: str):
    cm = getattr(scene, "color_model", None)
    if cm is None or getattr(cm, "kind", "sg") != "sg":
        raise ColorModelError(f"{what} requires an SG-tagged scene, got "
                              f"{getattr(cm, 'kind', None)!r}")


def quat_to_rot(q: np.ndarray) -> np.ndarray:
    """Rotation matrices from unit quaternions (w, x, y, z), batched."""
    q = np.asarray(q, dtype=np.float64)
    w, x, y, z = (q[..., k] for k in range(4))
    out = np.empty(q.shape[:-1] + (3, 3))
    out[..., 0, :] = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1)
    out[..., 1, :] = np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1)
    out[..., 2, :] = np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1)
    return out


# ------------------------------------------------------------------ context
_RAST: Rasterizer | None = None


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2509_07021_b200.render needs a CUDA device (B200); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def rasterizer() -> Rasterizer:
    """The module's shared render context (workspace cache) on the current device."""
    global _RAST
    dev = _device()
    if _RAST is None or _RAST.device != dev:
        _RAST = Rasterizer(device=dev)
    return _RAST


def _bg(background) -> tuple:
    return tuple(float(v) for v in np.asarray(background, dtype=np.float64).reshape(3))


def _upload(p) -> GaussianTensors:
    return GaussianTensors.from_arrays(p, device=_device())


def _to_np64(t: torch.Tensor) -> np.ndarray:
    return device_to_host_f64(t)


# ------------------------------------------------------------------ forward
def _render_params(p, cam, background, weight_sums: np.ndarray | None = None) -> np.ndarray:
    """(H, W, 3) float64 image; ``weight_sums`` (N) is accumulated in place
    with the composited blending weights (render.py:393-408)."""
    rast = rasterizer()
    g = _upload(p)
    fx = None
    if weight_sums is not None:
        fx = torch.zeros(g.n, dtype=torch.int64, device=rast.device)
    frame = rast.forward(g, cam, _bg(background), weight_fx=fx, track=False)
    img = _to_np64(frame.img)
    if weight_sums is not None:
        weight_sums += _fx_to_np64(fx)
    return img


def _fx_to_np64(fx: torch.Tensor) -> np.ndarray:
    """Exact integer weight sums (2^-32 units) -> float64, as the reference
    accumulates its weights in float64 (render.py:406-407)."""
    return (fx.to(torch.float64) * 2.0 ** -_ffi.WEIGHT_FRAC_BITS).cpu().numpy()


def render(scene, cam, background=(0.0, 0.0, 0.0)) -> np.ndarray:
    """Render an (H, W, 3) float image, front-to-back alpha blending."""
    return _render_params(SceneParams.from_scene(scene), cam, background)


def accumulate_importance(scene, cams, background=(0.0, 0.0, 0.0)) -> np.ndarray:
    """Per-primitive sum of blending weights actually composited."""
    return accumulate_importance_params(SceneParams.from_scene(scene), cams, background)


_SIDE_STREAMS: dict = {}


def _side_streams(device, n: int) -> list:
    key = str(device)
    have = _SIDE_STREAMS.setdefault(key, [])
    while len(have) < n:
        have.append(torch.cuda.Stream(device))
    return have[:n]


def accumulate_importance_params(p, cams, background=(0.0, 0.0, 0.0), streams: int = 4) -> np.ndarray:
    """render.py:416-428.  The views render concurrently on ``streams`` CUDA
    streams; their weights are added as exact 64-bit fixed point into one
    array (so the result does not depend on the order the views and tiles
    land in: bitwise reproducible, ties stay ties for the top-k of
    prune.py:204).  Tile-entry capacity is checked once for all views, and a
    pass in which any view outgrew its capacity is redone from zero with the
    capacity grown."""
    rast = rasterizer()
    g = _upload(p)
    bg = _bg(background)
    cams = list(cams)
    main = torch.cuda.current_stream(rast.device)
    side = _side_streams(rast.device, max(1, min(int(streams), len(cams))))
    while True:
        fx = torch.zeros(g.n, dtype=torch.int64, device=rast.device)
        ovf = torch.zeros((max(len(cams), 1), 2), dtype=torch.int64, device=rast.device)
        ready = torch.cuda.Event()
        ready.record(main)
        for j, cam in enumerate(cams):
            st = side[j % len(side)]
            st.wait_event(ready)
            with torch.cuda.stream(st):
                rast.forward(g, cam, bg, weight_fx=fx, track=False, check=False).record_overflow(ovf[j])
        for st in side:
            main.wait_stream(st)
        o = ovf.cpu().numpy()
        if not o[:, 0].any():
            return _fx_to_np64(fx)
        for j, cam in enumerate(cams):
            if o[j, 0]:
                rast.grow_capacity(g, cam, int(o[j, 1]))


# --------------------------------------------------------------------- loss
# All loss math runs in the fused SSIM + L1 kernel (csrc/loss.cu, loss.py):
# float64 statistics on the device, exact dL/dimg (render.py:469-509).
def _t64(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=_device(), dtype=torch.float64)
    return torch.as_tensor(np.asarray(a, dtype=np.float64), device=_device())


def _check_shapes(img, target):
    if tuple(np.shape(img)) != tuple(np.shape(target)):
        raise ValueError(f"image shape {tuple(np.shape(img))} != target {tuple(np.shape(target))}")


def _with_ssim(cfg: LossConfig) -> LossConfig:
    """The same window / constants with lambda = 1 (pure SSIM term)."""
    return dataclasses.replace(cfg, lambda_ssim=1.0)


def ssim(img, target, cfg: LossConfig = LossConfig()) -> float:
    _check_shapes(img, target)
    out, _, _ = image_loss(_t64(img), _t64(target), _with_ssim(cfg), grad=None)
    return float(out[2])


def loss(img, target, cfg: LossConfig = LossConfig()) -> float:
    _check_shapes(img, target)
    out, _, _ = image_loss(_t64(img), _t64(target), cfg, grad=None)
    return float(out[0])


def _loss_and_dimg(img, target, cfg: LossConfig):
    _check_shapes(img, target)
    out, d, _ = image_loss(_t64(img), _t64(target), cfg, grad="f64")
    return float(out[0]), _to_np64(d)


def _ssim_grad(img, target, cfg: LossConfig):
    """d(mean SSIM)/d(img) and the SSIM map (render.py:469-486)."""
    _check_shapes(img, target)
    # with lambda = 1 the kernel's dL/dimg is -d(mean SSIM)/dimg
    _, d, smap = image_loss(_t64(img), _t64(target), _with_ssim(cfg), grad="f64", ssim_map=True)
    return -_to_np64(d), _to_np64(smap)


def psnr(img: np.ndarray, target: np.ndarray) -> float:
    """Peak signal-to-noise ratio in dB, both images clipped to [0, 1]."""
    a = np.clip(img, 0.0, 1.0)
    b = np.clip(target, 0.0, 1.0)
    mse = float(((a - b) ** 2).mean())
    if mse == 0.0:
        return float("inf")
    return -10.0 * np.log10(mse)


# ----------------------------------------------------------------- backward
def _grads_to_set(gr: dict) -> GradientSet:
    return GradientSet(*(_to_np64(gr[f]) for f in _PARAM_FIELDS))


def loss_and_grads_device(g: GaussianTensors, cam, target: torch.Tensor, cfg: LossConfig = LossConfig(),
                          background=(0.0, 0.0, 0.0), rast: Rasterizer | None = None,
                          mask_grads: bool = False, sync: bool = True, overflow_out=None,
                          grads_out: dict | None = None, accumulate: bool = False, mask_logit: bool = False,
                          deterministic: bool = False, grad_floor: float = GRAD_OPACITY_FLOOR):
    """Device-resident variant: (loss, dict of float32 gradient tensors).  The
    loss is a float, or a 0-dim float64 device tensor with ``sync=False`` (no
    host round trip).  With ``overflow_out`` (int64 device tensor of 2) the
    tile-entry capacity is not checked here: the frame's (overflow, entries)
    counters land in it and the caller checks them later (Frame.record_overflow).
    ``grads_out`` / ``accumulate`` / ``mask_logit`` / ``deterministic``: see
    Rasterizer.backward (a training step sums its views straight into one
    gradient bucket; the ADMM loop asks for bitwise-reproducible sums)."""
    rast = rast or rasterizer()
    frame = rast.forward(g, cam, _bg(background), check=overflow_out is None, grad_floor=grad_floor)
    if overflow_out is not None:
        frame.record_overflow(overflow_out)
    out, dimg, _ = image_loss(frame.img, target, cfg, grad="f32")
    grads = rast.backward(g, frame, dimg, mask_grads=mask_grads, out=grads_out, accumulate=accumulate,
                          mask_logit=mask_logit, deterministic=deterministic)
    return (float(out[0]) if sync else out[0]), grads


def loss_and_grads(p, cam, target: np.ndarray, cfg: LossConfig = LossConfig(),
                   background=(0.0, 0.0, 0.0)):
    """Scalar loss and analytic gradients for one view, params-space."""
    if tuple(np.shape(target)) != (cam.height, cam.width, 3):
        raise ValueError(f"target shape {tuple(np.shape(target))} does not match "
                         f"camera {(cam.height, cam.width, 3)}")
    val, gr = loss_and_grads_device(_upload(p), cam, _t64(target), cfg, background)
    return val, _grads_to_set(gr)


def render_backward(scene, cam, target, cfg: LossConfig = LossConfig(), background=(0.0, 0.0, 0.0)):
    """Loss against a target view plus gradients for every parameter class."""
    return loss_and_grads(SceneParams.from_scene(scene), cam, target, cfg, background)


# ------------------------------------------------------------- projection
class Projection:
    """Visible primitives in stable front-to-back order (the per-primitive
    fields of the reference's _Projected, render.py:232-256)."""


def _project_records(p, cam, lowpass: float) -> np.ndarray:
    import ctypes as C
    g = _upload(p)
    out = torch.empty((max(g.n, 1), 16), dtype=torch.float32, device=g.device)
    _ffi.call("sgs_project_records", C.byref(g.c_params()), C.byref(to_sgs(cam, lowpass=lowpass)),
              out.data_ptr(), C.c_void_p(torch.cuda.current_stream(g.device).cuda_stream))
    return out[: g.n].cpu().numpy().astype(np.float64)


def _prepare(p, cam, lowpass: float = LOWPASS_FLOOR) -> Projection | None:
    rec = _project_records(p, cam, lowpass)
    vis = np.flatnonzero(rec[:, 0] > 0)
    if vis.size == 0:
        return None
    # the reference's order: stable argsort of its float64 z (render.py:262, 307)
    z64 = (np.asarray(p.position, dtype=np.float64)[vis] @ np.asarray(cam.rotation, dtype=np.float64).T
           + np.asarray(cam.translation, dtype=np.float64))[:, 2]
    order = vis[np.argsort(z64, kind="stable")]
    r = rec[order]
    pr = Projection()
    pr.orig_idx = order
    pr.depth = z64[np.argsort(z64, kind="stable")]
    pr.mean2d = r[:, 2:4].copy()
    pr.cov2d = np.stack([np.stack([r[:, 4], r[:, 5]], -1), np.stack([r[:, 5], r[:, 6]], -1)], 1)
    pr.conic = np.stack([np.stack([r[:, 7], r[:, 8]], -1), np.stack([r[:, 8], r[:, 9]], -1)], 1)
    pr.color_pre = r[:, 10:13].copy()
    pr.color = r[:, 13:16].copy()
    pr.opacity = np.asarray(p.opacity, dtype=np.float64)[order]
    return pr


def project(prim, cam, lowpass: float = LOWPASS_FLOOR) -> Splat2D | None:
    """Project one primitive; None when its center is behind the near plane."""

    class _Model:
        kind = "sg"
        max_lobes = max(len(prim.lobes), 1)

    class _Scene:
        primitives = [prim]
        color_model = _Model()

    proj = _prepare(SceneParams.from_scene(_Scene()), cam, lowpass=lowpass)
    if proj is None:
        return None
    return Splat2D(mean2d=proj.mean2d[0], cov2d=proj.cov2d[0], depth=float(proj.depth[0]),
                   color=proj.color[0], opacity=float(proj.opacity[0]))
