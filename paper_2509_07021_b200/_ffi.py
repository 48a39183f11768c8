"""ctypes binding of libsgs.so (include/sgs.h).

The ABI takes plain device pointers; PyTorch only allocates them.  Loading
fails loudly: there is no CPU fallback anywhere in this package.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

from ._build import LIB_PATH

SGS_OK = 0
SGS_E_ARG = -1
SGS_E_CUDA = -2
SGS_E_WORKSPACE = -3
SGS_E_CAPACITY = -4
SGS_E_FORMAT = -5
SGS_E_TRUNCATED = -6
SORT_DEPTH_FIRST = 0
SORT_KEY64 = 1


class SgsCamera(C.Structure):
    _fields_ = [("rotation", C.c_float * 9), ("translation", C.c_float * 3),
                ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("near_z", C.c_float), ("width", C.c_int32), ("height", C.c_int32),
                ("tile_y0", C.c_int32), ("tile_y1", C.c_int32), ("lowpass", C.c_float),
                ("depth_row", C.c_double * 4), ("near_z64", C.c_double), ("grad_floor", C.c_float)]


class SgsParams(C.Structure):
    _fields_ = [("position", C.c_void_p), ("quat", C.c_void_p), ("log_scale", C.c_void_p),
                ("opacity", C.c_void_p), ("diffuse", C.c_void_p), ("axis_raw", C.c_void_p),
                ("sharpness", C.c_void_p), ("amplitude", C.c_void_p), ("lobe_mask", C.c_void_p),
                ("prim_mask", C.c_void_p), ("n", C.c_int64), ("n_lobes", C.c_int32)]


class SgsGrads(C.Structure):
    _fields_ = [("position", C.c_void_p), ("quat", C.c_void_p), ("log_scale", C.c_void_p),
                ("opacity", C.c_void_p), ("diffuse", C.c_void_p), ("axis_raw", C.c_void_p),
                ("sharpness", C.c_void_p), ("amplitude", C.c_void_p), ("lobe_mask", C.c_void_p),
                ("prim_mask", C.c_void_p), ("flags", C.c_int32)]


WEIGHT_FRAC_BITS = 32  # sgs_raster_forward's weight_sums_fx fixed point
GRADS_ACCUMULATE = 1   # SGS_GRADS_ACCUMULATE
GRADS_MASK_LOGIT = 2   # SGS_GRADS_MASK_LOGIT


class SgsWorkspace(C.Structure):
    _fields_ = [("base", C.c_void_p), ("bytes", C.c_uint64), ("n", C.c_int64),
                ("n_lobes", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
                ("sort_mode", C.c_int32), ("entry_capacity", C.c_int64)]


class SgsStats(C.Structure):
    _fields_ = [("n_visible", C.c_uint64), ("n_emitting", C.c_uint64), ("n_entries", C.c_uint64),
                ("capacity", C.c_uint64), ("overflow", C.c_uint64),
                ("vram3s_visible", C.c_uint64), ("vram3s_entries", C.c_uint64),
                ("n_bin_entries", C.c_uint64)]


class SgsSceneSoa(C.Structure):
    _fields_ = [(f, C.c_void_p) for f in ("position", "quat", "log_scale", "opacity", "diffuse",
                                           "axis_raw", "sharpness", "amplitude", "lobe_mask")]


class SgsAdmmFields(C.Structure):
    _fields_ = [(f, C.c_void_p) for f in ("position", "quat", "log_scale", "opacity", "diffuse", "axis_raw",
                                           "sharpness", "amplitude")]


class SgsAdmmRates(C.Structure):
    _fields_ = [(f, C.c_float) for f in ("position", "quat", "log_scale", "opacity", "diffuse", "axis_raw",
                                         "sharpness", "amplitude", "eta", "delta_o", "delta_s")]


class SgsLossConfig(C.Structure):
    _fields_ = [("lambda_ssim", C.c_double), ("window", C.c_int32), ("sigma", C.c_double),
                ("c1", C.c_double), ("c2", C.c_double)]


# every exported symbol and its signature (tests check the .so exports all of them)
_P = C.POINTER
SIGNATURES = {
    "sgs_version": (C.c_int32, []),
    "sgs_abi_sizes": (C.c_int, [_P(C.c_uint64)]),
    "sgs_admm_update": (C.c_int, [C.c_int64, C.c_int32, C.c_int32, C.c_int32, _P(SgsAdmmFields), _P(SgsAdmmFields),
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, _P(SgsAdmmRates),
                                  C.c_void_p, C.c_void_p]),
    "sgs_last_error": (C.c_char_p, []),
    "sgs_workspace_size": (C.c_int, [_P(SgsWorkspace), _P(C.c_uint64)]),
    "sgs_preprocess": (C.c_int, [_P(SgsParams), _P(SgsCamera), _P(SgsWorkspace), C.c_void_p]),
    "sgs_bin": (C.c_int, [_P(SgsCamera), _P(SgsWorkspace), C.c_void_p]),
    "sgs_raster_forward": (C.c_int, [_P(SgsCamera), _P(C.c_float), _P(SgsWorkspace), C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sgs_render_forward": (C.c_int, [_P(SgsParams), _P(SgsCamera), _P(C.c_float), _P(SgsWorkspace),
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p]),
    "sgs_raster_backward": (C.c_int, [_P(SgsCamera), _P(C.c_float), _P(SgsWorkspace), C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sgs_raster_backward_det_scratch_bytes": (C.c_uint64, [C.c_int64]),
    "sgs_raster_backward_det": (C.c_int, [_P(SgsCamera), _P(C.c_float), _P(SgsWorkspace), C.c_void_p,
                                          C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_uint64, C.c_void_p]),
    "sgs_fixed_to_float": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p]),
    "sgs_preprocess_backward": (C.c_int, [_P(SgsParams), _P(SgsCamera), C.c_void_p, _P(SgsGrads),
                                          C.c_void_p]),
    "sgs_preprocess_backward_views": (C.c_int, [_P(SgsParams), _P(SgsCamera), C.c_int, _P(C.c_void_p),
                                                _P(SgsGrads), C.c_void_p]),
    "sgs_project_records": (C.c_int, [_P(SgsParams), _P(SgsCamera), C.c_void_p, C.c_void_p]),
    "sgs_get_stats": (C.c_int, [_P(SgsWorkspace), _P(SgsStats), C.c_void_p]),
    "sgs_vram_model": (C.c_int, [_P(SgsParams), _P(SgsCamera), C.c_int32, _P(SgsWorkspace),
                                 C.c_void_p]),
    "sgs_export_bins": (C.c_int, [_P(SgsWorkspace), _P(SgsCamera), C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_void_p]),
    "sgs_export_projected": (C.c_int, [_P(SgsWorkspace), C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p]),
    "sgs_debug_buffer": (C.c_int, [_P(SgsWorkspace), C.c_int32, _P(C.c_void_p), _P(C.c_uint64)]),
    "sgs_sort_temp_size": (C.c_int, [C.c_int64, C.c_int32, _P(C.c_uint64)]),
    "sgs_sort_pairs_u64": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p,
                                     C.c_uint64, C.c_void_p]),
    "sgs_loss_workspace_size": (C.c_int, [C.c_int32, C.c_int32, _P(C.c_uint64)]),
    "sgs_topk_mask_temp_size": (C.c_int, [C.c_int64, _P(C.c_uint64)]),
    "sgs_compact_header": (C.c_int, [C.c_char_p, C.c_uint64, _P(C.c_int64)]),
    "sgs_compact_index": (C.c_int, [C.c_char_p, C.c_uint64, C.c_void_p, C.c_int64, _P(C.c_int32)]),
    "sgs_compact_decode": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, _P(SgsSceneSoa),
                                     C.c_void_p]),
    "sgs_topk_mask": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_uint64,
                                C.c_void_p]),
    "sgs_image_loss": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                 _P(SgsLossConfig), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_uint64, C.c_void_p]),
}


class SgsError(RuntimeError):
    """A libsgs.so call returned a non-zero status."""

    def __init__(self, func: str, code: int, message: str):
        super().__init__(f"{func} failed ({code}): {message}")
        self.code = code


class CapacityError(SgsError):
    pass


_lib = None


def load(path: Path | None = None) -> C.CDLL:
    """Load libsgs.so (building it first if the sources are newer)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    import os
    p = Path(path) if path is not None else Path(os.environ.get("SGS_LIB", LIB_PATH))
    if not p.exists():
        from ._build import build_lib
        build_lib()
    lib = C.CDLL(str(p))
    # SGS_ALLOW_MISSING=1: bind what an older build exports (A/B timing of
    # earlier revisions, profiles/variant.py); the product never sets it
    allow_missing = os.environ.get("SGS_ALLOW_MISSING") == "1"
    for name, (res, args) in SIGNATURES.items():
        if allow_missing and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def check(func: str, rc: int) -> None:
    if rc != SGS_OK:
        msg = load().sgs_last_error().decode(errors="replace")
        if rc == SGS_E_CAPACITY:
            raise CapacityError(func, rc, msg)
        if rc == SGS_E_ARG:
            raise ValueError(f"{func}: {msg}")
        raise SgsError(func, rc, msg)


def call(func: str, *args) -> None:
    check(func, getattr(load(), func)(*args))
