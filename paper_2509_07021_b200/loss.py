"""Device image loss: the fused SSIM + L1 kernel of libsgs.so (csrc/loss.cu).

Replaces the reference's loss / ssim / _ssim_grad / _loss_and_dimg
(/root/reference/pkg/src/sgsplat/render.py:433-509):

  loss = (1 - lambda) mean|img - target| + lambda (1 - mean SSIM)

with the 11x11 (LossConfig.window) Gaussian window, zero padding, and the
exact gradient with respect to the image.  Images are (H, W, 3) CUDA tensors,
float32 or float64; statistics are accumulated in float64 on the device and
nothing synchronises -- the loss comes back as a device tensor.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _ffi

_WS: dict = {}


def _workspace(H: int, W: int, device) -> torch.Tensor:
    key = (H, W, str(device), torch.cuda.current_stream(device).cuda_stream)
    ws = _WS.get(key)
    if ws is None:
        nb = C.c_uint64()
        _ffi.call("sgs_loss_workspace_size", H, W, C.byref(nb))
        ws = torch.empty(int(nb.value), dtype=torch.uint8, device=device)
        _WS[key] = ws
    return ws


def loss_config(cfg) -> _ffi.SgsLossConfig:
    c = _ffi.SgsLossConfig()
    c.lambda_ssim = float(cfg.lambda_ssim)
    c.window = int(cfg.window)
    c.sigma = float(cfg.sigma)
    c.c1 = float(cfg.c1)
    c.c2 = float(cfg.c2)
    return c


def _as_input(t: torch.Tensor, device) -> torch.Tensor:
    if t.dtype not in (torch.float32, torch.float64):
        t = t.to(torch.float64)
    return t.to(device).contiguous()


def image_loss(img: torch.Tensor, target: torch.Tensor, cfg, grad: str | None = "f32",
               ssim_map: bool = False):
    """(out, dimg, smap): out = device float64 [loss, mean L1, mean SSIM];
    dimg = dL/dimg as float32 (grad="f32"), float64 (grad="f64") or None;
    smap = the (H, W, 3) float64 SSIM map when requested."""
    if tuple(img.shape) != tuple(target.shape):
        raise ValueError(f"image shape {tuple(img.shape)} != target {tuple(target.shape)}")
    if img.dim() != 3 or img.shape[2] != 3:
        raise ValueError(f"images must be (H, W, 3), got {tuple(img.shape)}")
    dev = img.device
    x = _as_input(img, dev)
    y = _as_input(target, dev)
    H, W = int(x.shape[0]), int(x.shape[1])
    out = torch.empty(5, dtype=torch.float64, device=dev)
    d32 = torch.empty_like(x, dtype=torch.float32) if grad == "f32" else None
    d64 = torch.empty_like(x, dtype=torch.float64) if grad == "f64" else None
    smap = torch.empty_like(x, dtype=torch.float64) if ssim_map else None
    ws = _workspace(H, W, dev)
    c = loss_config(cfg)

    def p(t):
        return None if t is None else t.data_ptr()

    _ffi.call("sgs_image_loss", x.data_ptr(), int(x.dtype == torch.float64), y.data_ptr(),
              int(y.dtype == torch.float64), H, W, C.byref(c), p(d32), p(d64), p(smap),
              out.data_ptr(), ws.data_ptr(), ws.numel(),
              C.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    return out[:3], (d32 if d32 is not None else d64), smap
