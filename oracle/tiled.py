"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper of the CPU tiled restatement
(oracle/sgs_tiled.cpp).  Imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg; never by the product package.
"""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

ORACLE_DIR = Path(__file__).resolve().parent
LIB = ORACLE_DIR / "_build" / "libsgs_oracle.so"

_lib = None


def build() -> Path:
    srcs = [ORACLE_DIR / "sgs_tiled.cpp",
            ORACLE_DIR.parent / "paper_2509_07021_b200" / "csrc" / "sgs_geom.h"]
    if not LIB.exists() or any(s.stat().st_mtime > LIB.stat().st_mtime for s in srcs):
        subprocess.run(["make", "-s", "-C", str(ORACLE_DIR)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        _lib = C.CDLL(str(LIB))
        _lib.oracle_count_entries.restype = C.c_int64
        _lib.oracle_sgs_expf.restype = C.c_float
        _lib.oracle_sgs_expf.argtypes = [C.c_float]
        _lib.oracle_sgs_logf.restype = C.c_float
        _lib.oracle_sgs_logf.argtypes = [C.c_float]
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def cam_arrays(cam, tile_rows=(0, 0), lowpass=0.3):
    f = np.zeros(18, np.float32)
    f[:9] = np.asarray(cam.rotation, dtype=np.float64).reshape(9)
    f[9:12] = np.asarray(cam.translation, dtype=np.float64).reshape(3)
    f[12:18] = [cam.fx, cam.fy, cam.cx, cam.cy, getattr(cam, "near", 0.1), lowpass]
    i = np.array([cam.width, cam.height, tile_rows[0], tile_rows[1]], np.int32)
    return f, i


def cam_f64(cam, grad_floor: float = 0.0):
    """(w0, w1, w2, t_z, near) in float64: the depth row (sgs_camera.depth_row)."""
    r = np.asarray(cam.rotation, dtype=np.float64).reshape(3, 3)
    t = np.asarray(cam.translation, dtype=np.float64).reshape(3)
    return np.array([r[2, 0], r[2, 1], r[2, 2], t[2], float(getattr(cam, "near", 0.1)),
                     float(np.float32(grad_floor))], np.float64)


def _arrays(s):
    f32 = lambda a: np.ascontiguousarray(np.asarray(a), dtype=np.float32)  # noqa: E731
    out = {k: f32(getattr(s, k)) for k in ("position", "quat", "log_scale", "opacity", "diffuse",
                                           "axis_raw", "sharpness", "amplitude", "lobe_mask")}
    pm = getattr(s, "prim_mask", None)
    out["prim_mask"] = None if pm is None else f32(pm)
    return out


class TiledResult:
    pass


def preprocess(scene, cam, tile_rows=(0, 0), lowpass=0.3, grad_floor=0.0):
    a = _arrays(scene)
    n, L = a["position"].shape[0], a["axis_raw"].shape[1]
    cf, ci = cam_arrays(cam, tile_rows, lowpass)
    r = TiledResult()
    r.depth_bits = np.zeros(n, np.uint32)
    r.depth_res = np.zeros(n, np.float32)
    r.rect = np.zeros((n, 2), np.uint32)
    r.tiles_touched = np.zeros(n, np.uint32)
    r.records = np.zeros((n, 16), np.float32)
    counts = np.zeros(2, np.int64)
    lib().oracle_preprocess(C.c_int64(n), C.c_int(L), _p(a["position"]), _p(a["quat"]),
                            _p(a["log_scale"]), _p(a["opacity"]), _p(a["diffuse"]),
                            _p(a["axis_raw"]), _p(a["sharpness"]), _p(a["amplitude"]),
                            _p(a["lobe_mask"]), _p(a["prim_mask"]), _p(cf), _p(ci), _p(cam_f64(cam, grad_floor)),
                            _p(r.depth_bits), _p(r.depth_res), _p(r.rect), _p(r.tiles_touched), _p(r.records),
                            _p(counts))
    r.n_visible, r.n_emitting = int(counts[0]), int(counts[1])
    r.cam_f, r.cam_i, r.n, r.arrays = cf, ci, n, a
    return r


def bin(r):  # noqa: A001 - mirrors sgs_bin
    E = int(lib().oracle_count_entries(C.c_int64(r.n), _p(r.tiles_touched)))
    tiles = ((int(r.cam_i[0]) + 15) // 16) * ((int(r.cam_i[1]) + 15) // 16)
    r.keys = np.zeros(max(E, 1), np.uint64)
    r.vals = np.zeros(max(E, 1), np.uint32)
    r.ranges = np.zeros((tiles, 2), np.uint32)
    lib().oracle_bin(C.c_int64(r.n), _p(r.depth_bits), _p(r.depth_res), _p(r.rect), _p(r.tiles_touched),
                     _p(r.records), _p(r.cam_f), _p(r.cam_i), _p(r.keys), _p(r.vals),
                     _p(r.ranges))
    r.keys, r.vals, r.n_entries = r.keys[:E], r.vals[:E], E
    return r


def raster_forward(r, background=(0.0, 0.0, 0.0), importance=False):
    W, H = int(r.cam_i[0]), int(r.cam_i[1])
    bg = np.asarray(background, np.float32).reshape(3)
    r.img = np.zeros((H, W, 3), np.float32)
    r.T = np.ones((H, W), np.float32)
    r.nc = np.zeros((H, W), np.uint32)
    r.weight_sums = np.zeros(r.n, np.float64) if importance else None
    vals = r.vals if r.n_entries else np.zeros(1, np.uint32)
    lib().oracle_raster_forward(_p(r.ranges), _p(vals), _p(r.records), _p(r.cam_f), _p(r.cam_i),
                                _p(bg), _p(r.img), _p(r.T), _p(r.nc), _p(r.weight_sums))
    r.bg = bg
    return r


def raster_backward(r, dimg):
    dimg = np.ascontiguousarray(dimg, dtype=np.float32)
    r.grad2d = np.zeros((r.n, 9), np.float64)
    vals = r.vals if r.n_entries else np.zeros(1, np.uint32)
    lib().oracle_raster_backward(_p(r.ranges), _p(vals), _p(r.records), _p(r.cam_f), _p(r.cam_i),
                                 _p(r.bg), _p(dimg), _p(r.grad2d))
    return r


def preprocess_backward(r, grad2d=None):
    a = r.arrays
    n, L = r.n, a["axis_raw"].shape[1]
    g2 = np.ascontiguousarray(r.grad2d if grad2d is None else grad2d, dtype=np.float64)
    out = {"position": np.zeros((n, 3)), "quat": np.zeros((n, 4)), "log_scale": np.zeros((n, 3)),
           "opacity": np.zeros(n), "diffuse": np.zeros((n, 3)), "axis_raw": np.zeros((n, L, 3)),
           "sharpness": np.zeros((n, L)), "amplitude": np.zeros((n, L, 3)),
           "lobe_mask": np.zeros((n, L)), "prim_mask": np.zeros(n)}
    lib().oracle_preprocess_backward(
        C.c_int64(n), C.c_int(L), _p(a["position"]), _p(a["quat"]), _p(a["log_scale"]),
        _p(a["opacity"]), _p(a["diffuse"]), _p(a["axis_raw"]), _p(a["sharpness"]),
        _p(a["amplitude"]), _p(a["lobe_mask"]), _p(a["prim_mask"]), _p(r.cam_f), _p(g2),
        *[_p(out[k]) for k in ("position", "quat", "log_scale", "opacity", "diffuse", "axis_raw",
                               "sharpness", "amplitude", "lobe_mask", "prim_mask")])
    r.grads = out
    return out


def render(scene, cam, background=(0.0, 0.0, 0.0), tile_rows=(0, 0), importance=False, grad_floor=0.0):
    r = preprocess(scene, cam, tile_rows, grad_floor=grad_floor)
    bin(r)
    return raster_forward(r, background, importance)


def expf(x: float) -> float:
    return float(lib().oracle_sgs_expf(float(x)))


def logf(x: float) -> float:
    return float(lib().oracle_sgs_logf(float(x)))
