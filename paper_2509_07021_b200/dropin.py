"""Patch an installed reference package (``sgsplat``) so its callers run on
the B200 renderer.

The reference imports the hot-path functions by name into several modules
(prune.py:20-21, postprocess.py:17, toy.py:15, cli.py:29), and its package
``__init__`` re-exports ``render`` over the submodule attribute
(__init__.py:12-14), so patching must go through ``sys.modules`` and every
importing namespace.  Reference dataclasses (SceneParams, Camera, Scene ...)
are consumed by duck typing; results are returned in the reference's own
GradientSet / VramEstimate types when those exist.
"""

from __future__ import annotations

import importlib
import sys

from . import postprocess as _post
from . import render as _r

_PATCHED: dict = {}


def _wrap_grads(ref_mod, gs):
    cls = getattr(ref_mod, "GradientSet", None)
    if cls is None:
        return gs
    return cls(*(getattr(gs, f) for f in _r._PARAM_FIELDS))


def install(package: str = "sgsplat") -> list[str]:
    """Route sgsplat's render hot path through libsgs.so; returns what was patched."""
    __import__(package)
    # every module that binds a hot-path name (prune.py:20, postprocess.py:17,
    # toy.py:15, cli.py:29); the package __init__ imports all but cli
    for sub in ("render", "prune", "postprocess", "toy", "cli"):
        try:
            importlib.import_module(f"{package}.{sub}")
        except ImportError:  # pragma: no cover - optional entry points (cli needs pillow)
            pass
    ref_render = sys.modules[f"{package}.render"]
    patched = []

    def loss_and_grads(p, cam, target, cfg=None, background=(0.0, 0.0, 0.0)):
        cfg = cfg if cfg is not None else ref_render.LossConfig()
        val, gs = _r.loss_and_grads(p, cam, target, _r.LossConfig(
            cfg.lambda_ssim, cfg.window, cfg.sigma, cfg.c1, cfg.c2), background)
        return val, _wrap_grads(ref_render, gs)

    def render_backward(scene, cam, target, cfg=None, background=(0.0, 0.0, 0.0)):
        return loss_and_grads(ref_render.SceneParams.from_scene(scene), cam, target, cfg, background)

    def estimate_vram(scene, cam, tile_px=16):
        est = _post.estimate_vram(scene, cam, tile_px)
        cls = getattr(sys.modules.get(f"{package}.postprocess"), "VramEstimate", None)
        return cls(est.static_bytes, est.dynamic_bytes) if cls else est

    table = {
        "render": _r.render,
        "_render_params": _r._render_params,
        "accumulate_importance": _r.accumulate_importance,
        "accumulate_importance_params": _r.accumulate_importance_params,
        "loss_and_grads": loss_and_grads,
        "render_backward": render_backward,
        "estimate_vram": estimate_vram,
    }
    for mod_name in (f"{package}.render", f"{package}.prune", f"{package}.postprocess",
                     f"{package}.toy", f"{package}.cli", package):
        mod = sys.modules.get(mod_name)
        if mod is None:
            continue
        for name, fn in table.items():
            if hasattr(mod, name):
                _PATCHED.setdefault((mod_name, name), getattr(mod, name))
                setattr(mod, name, fn)
                patched.append(f"{mod_name}.{name}")
    return patched


def uninstall() -> None:
    for (mod_name, name), fn in _PATCHED.items():
        mod = sys.modules.get(mod_name)
        if mod is not None:
            setattr(mod, name, fn)
    _PATCHED.clear()
