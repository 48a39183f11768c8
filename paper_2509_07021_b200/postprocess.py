"""Drop-in for the reference's render-time memory model
(/root/reference/pkg/src/sgsplat/postprocess.py:24-29, 85-137), evaluated on
the GPU with the renderer's own projection, plus the measured counterpart.

``estimate_vram`` keeps the reference's declared model exactly: a primitive
is visible when its center clears the near plane and its 3-sigma box meets
the image; it costs a 40-byte projected record plus a 12-byte key/value entry
per overlapped tile (floor/clip tile rectangle).  ``measured_render_vram``
reports what this renderer actually allocates for one frame.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _ffi
from .camera import to_sgs
from .render import SceneParams, _require_sg, _upload, rasterizer

SPLAT2D_RECORD_BYTES = 10 * 4
TILE_ENTRY_BYTES = 12
STATIC_FLOATS_PER_PRIMITIVE = 14
PARAMS_PER_LOBE = 7


@dataclass(frozen=True)
class VramEstimate:
    """Analytic peak-memory model: loaded floats + per-view intermediates."""

    static_bytes: int
    dynamic_bytes: int

    @property
    def peak_bytes(self) -> int:
        return self.static_bytes + self.dynamic_bytes


def static_bytes(scene) -> int:
    """budget_report(scene).static_bytes (scene.py:202-216): 4 B x (14 per
    primitive + 7 per lobe)."""
    n = len(scene.primitives)
    lobes = sum(len(p.lobes) for p in scene.primitives)
    return 4 * (STATIC_FLOATS_PER_PRIMITIVE * n + PARAMS_PER_LOBE * lobes)


def vram_counts(p, cam, tile_px: int = 16) -> tuple[int, int]:
    """(visible, tile entries) of the reference 3-sigma model on the GPU."""
    if tile_px < 1:
        raise ValueError("tile_px must be >= 1")
    rast = rasterizer()
    g = _upload(p)
    ws = rast.workspace(g, cam, private=True, capacity=1)
    _ffi.call("sgs_vram_model", C.byref(g.c_params()), C.byref(to_sgs(cam)), int(tile_px),
              C.byref(ws.desc), C.c_void_p(torch.cuda.current_stream(g.device).cuda_stream))
    st = ws.stats()
    return st["vram3s_visible"], st["vram3s_entries"]


def estimate_vram(scene, cam, tile_px: int = 16) -> VramEstimate:
    """Static bytes plus projected-splat records and tile key-value entries."""
    _require_sg(scene, "estimate_vram")
    if tile_px < 1:
        raise ValueError("tile_px must be >= 1")
    static = static_bytes(scene)
    if len(scene.primitives) == 0:
        return VramEstimate(static_bytes=static, dynamic_bytes=0)
    vis, entries = vram_counts(SceneParams.from_scene(scene), cam, tile_px)
    return VramEstimate(static_bytes=static,
                        dynamic_bytes=vis * SPLAT2D_RECORD_BYTES + entries * TILE_ENTRY_BYTES)


def measured_render_vram(p, cam, rast=None) -> dict:
    """Bytes this renderer allocates for one frame of `p` through `cam`: the
    workspace (projected records, depth-sort and tile-sort buffers, key/value
    entries, ranges) plus the output image / transmittance / contributor
    buffers, and the peak torch allocation seen while rendering."""
    from .rasterizer import GaussianTensors
    rast = rast or rasterizer()
    g = p if isinstance(p, GaussianTensors) else _upload(p)
    dev = g.device
    torch.cuda.synchronize(dev)
    base = torch.cuda.memory_allocated(dev)
    torch.cuda.reset_peak_memory_stats(dev)
    frame = rast.forward(g, cam, private=True)
    torch.cuda.synchronize(dev)
    st = frame.stats()
    outs = sum(t.numel() * t.element_size() for t in (frame.img, frame.final_T, frame.ncontrib))
    return {"workspace_bytes": frame.ws.nbytes, "output_bytes": outs,
            "peak_dynamic_bytes": torch.cuda.max_memory_allocated(dev) - base,
            "tile_entries": st["n_entries"], "visible": st["n_visible"],
            "emitting": st["n_emitting"]}
