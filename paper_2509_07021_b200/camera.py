"""Pinhole camera with the reference's conventions.

Mirrors ``Camera`` / ``Camera.look_at`` of
/root/reference/pkg/src/sgsplat/render.py:30-76: world-to-camera rotation
whose rows are (right, down, forward), ``p_cam = R x + t``, pixel
``(fx x/z + cx, fy y/z + cy)``, default near plane 0.1, ``ValueError`` on
non-positive focal lengths or an empty image.  Any object exposing the same
attributes (e.g. the reference's own Camera) is accepted by this package.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _ffi


@dataclass(frozen=True)
class Camera:
    rotation: np.ndarray
    translation: np.ndarray
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    near: float = 0.1

    def __post_init__(self):
        object.__setattr__(self, "rotation",
                           np.asarray(self.rotation, dtype=np.float64).reshape(3, 3))
        object.__setattr__(self, "translation",
                           np.asarray(self.translation, dtype=np.float64).reshape(3))
        if self.fx <= 0 or self.fy <= 0:
            raise ValueError("focal lengths must be positive")
        if self.width < 1 or self.height < 1:
            raise ValueError("image size must be at least 1x1")

    @property
    def center(self) -> np.ndarray:
        """Camera position in world coordinates, -R^T t."""
        return -self.rotation.T @ self.translation

    @staticmethod
    def look_at(eye, target, up=(0.0, 0.0, 1.0), fx=None, fy=None, width=64, height=64,
                near=0.1) -> "Camera":
        eye = np.asarray(eye, dtype=np.float64)
        forward = np.asarray(target, dtype=np.float64) - eye
        forward /= np.linalg.norm(forward)
        right = np.cross(forward, np.asarray(up, dtype=np.float64))
        right /= np.linalg.norm(right)
        down = np.cross(forward, right)
        rot = np.stack([right, down, forward])
        fx = 1.2 * width if fx is None else fx
        fy = fx if fy is None else fy
        return Camera(rotation=rot, translation=-rot @ eye, fx=fx, fy=fy, cx=width / 2.0,
                      cy=height / 2.0, width=width, height=height, near=near)

    def crop(self, x0: int, y0: int, w: int, h: int) -> "Camera":
        """Camera rendering exactly the pixels [y0, y0+h) x [x0, x0+w) of this
        one (same R, t, f; principal point shifted)."""
        return Camera(rotation=self.rotation, translation=self.translation, fx=self.fx,
                      fy=self.fy, cx=self.cx - x0, cy=self.cy - y0, width=w, height=h,
                      near=self.near)


def to_sgs(cam, tile_rows: tuple[int, int] | None = None, lowpass: float = 0.3,
           grad_floor: float = 0.0) -> _ffi.SgsCamera:
    """Duck-typed camera -> C struct (float32, as the GPU computes)."""
    c = _ffi.SgsCamera()
    rot = np.asarray(cam.rotation, dtype=np.float64).reshape(9).astype(np.float32)
    tr = np.asarray(cam.translation, dtype=np.float64).reshape(3).astype(np.float32)
    for i in range(9):
        c.rotation[i] = float(rot[i])
    for i in range(3):
        c.translation[i] = float(tr[i])
    c.fx, c.fy, c.cx, c.cy = (float(np.float32(v)) for v in (cam.fx, cam.fy, cam.cx, cam.cy))
    c.near_z = float(np.float32(getattr(cam, "near", 0.1)))
    c.width, c.height = int(cam.width), int(cam.height)
    if tile_rows is None:
        c.tile_y0, c.tile_y1 = 0, 0
    else:
        c.tile_y0, c.tile_y1 = int(tile_rows[0]), int(tile_rows[1])
    c.lowpass = float(np.float32(lowpass))
    # float64 depth row (render.py:262): z = p . R[2] + t[2] in the caller's doubles
    r64 = np.asarray(cam.rotation, dtype=np.float64).reshape(3, 3)
    t64 = np.asarray(cam.translation, dtype=np.float64).reshape(3)
    for k in range(3):
        c.depth_row[k] = float(r64[2, k])
    c.depth_row[3] = float(t64[2])
    c.near_z64 = float(getattr(cam, "near", 0.1))
    c.grad_floor = float(np.float32(grad_floor))
    return c
