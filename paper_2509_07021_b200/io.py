"""MEGS2 compact scene files -> device SoA.

The reference reads the compact format (/root/reference/pkg/src/sgsplat/
io.py:1-15 layout, 173-214 read_compact) into one Python object per
primitive and then packs SceneParams in a Python loop (render.py:135-145).
Here the record offsets are walked once by libsgs.so on the host (one byte
read per record, with the reference's format checks) and one GPU thread per
primitive decodes its record from the uploaded bytes straight into the
renderer's float32 SoA (sgs_compact_decode) -- the same arrays
SceneParams.from_scene builds.  ``write_compact`` is the vectorised writer
(byte-identical to the reference's write_compact).
"""

from __future__ import annotations

import ctypes as C
import struct
from pathlib import Path

import numpy as np
import torch

from . import _ffi
from .rasterizer import GaussianTensors

MAGIC = b"MEGS2\x00"
FORMAT_VERSION = 1
DEFAULT_MAX_LOBES = 3   # scene.py:28


class SceneFormatError(ValueError):
    """Malformed input file (scene.py SceneFormatError)."""


class TruncatedFileError(SceneFormatError):
    """Payload shorter than the header promises (scene.py TruncatedFileError)."""

    def __init__(self, message: str, offset: int = 0):
        super().__init__(message)
        self.offset = offset


def _raise(func: str, rc: int):
    if rc == _ffi.SGS_OK:
        return
    msg = _ffi.load().sgs_last_error().decode(errors="replace")
    if rc == _ffi.SGS_E_TRUNCATED:
        raise TruncatedFileError(msg)
    if rc == _ffi.SGS_E_FORMAT:
        raise SceneFormatError(msg)
    _ffi.check(func, rc)


def _bytes(data) -> bytes:
    if isinstance(data, (bytes, bytearray, memoryview)):
        return bytes(data)
    return Path(data).read_bytes()


def compact_index(data) -> tuple[np.ndarray, int]:
    """(count + 1 record offsets, largest lobe count) of a compact file."""
    raw = _bytes(data)
    lib = _ffi.load()
    n = C.c_int64()
    _raise("sgs_compact_header", lib.sgs_compact_header(raw, len(raw), C.byref(n)))
    offs = np.empty(int(n.value) + 1, dtype=np.uint64)
    ml = C.c_int32()
    _raise("sgs_compact_index", lib.sgs_compact_index(raw, len(raw), offs.ctypes.data, offs.size,
                                                      C.byref(ml)))
    return offs, int(ml.value)


def load_compact(data, device="cuda", min_lobes: int = DEFAULT_MAX_LOBES) -> GaussianTensors:
    """Read a compact file (bytes or path) into device tensors: the file's
    bytes go up once (pinned), the records are decoded on the GPU.  Lobe
    slots = max(largest lobe count, min_lobes), as read_compact's
    ColorModel.sg(max(max_lobes, DEFAULT_MAX_LOBES))."""
    raw = _bytes(data)
    offs, ml = compact_index(raw)
    n = offs.size - 1
    L = max(ml, int(min_lobes))
    dev = torch.device(device)
    host = torch.empty(max(len(raw), 1), dtype=torch.uint8, pin_memory=True)
    host.numpy()[: len(raw)] = np.frombuffer(raw, np.uint8)
    d_raw = host.to(dev, non_blocking=True)
    d_off = torch.from_numpy(offs.view(np.int64)).to(dev, non_blocking=True)
    f32 = dict(dtype=torch.float32, device=dev)
    arr = dict(position=torch.empty((n, 3), **f32), quat=torch.empty((n, 4), **f32),
               log_scale=torch.empty((n, 3), **f32), opacity=torch.empty((n,), **f32),
               diffuse=torch.empty((n, 3), **f32), axis_raw=torch.empty((n, L, 3), **f32),
               sharpness=torch.empty((n, L), **f32), amplitude=torch.empty((n, L, 3), **f32))
    lobe_mask = torch.empty((n, L), **f32)
    soa = _ffi.SgsSceneSoa()
    for k, t in arr.items():
        setattr(soa, k, t.data_ptr())
    soa.lobe_mask = lobe_mask.data_ptr()
    _ffi.call("sgs_compact_decode", d_raw.data_ptr(), d_off.data_ptr(), n, L, C.byref(soa),
              C.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    torch.cuda.current_stream(dev).synchronize()  # host staging buffer may be freed after return
    return GaussianTensors(**arr, lobe_mask=lobe_mask)


def write_compact(position, quat, scale, opacity, diffuse, axis, sharpness, amplitude, n_lobes) -> bytes:
    """Vectorised compact writer (io.py:157-170): per primitive 14 f32, a u8
    lobe count and 7 f32 per present lobe (the first n_lobes[i] slots)."""
    pos = np.asarray(position, np.float32).reshape(-1, 3)
    n = pos.shape[0]
    nl = np.asarray(n_lobes, np.int64).reshape(n)
    if np.any(nl < 0) or np.any(nl > 255):
        raise ValueError("lobe counts must be in [0, 255]")
    base = np.concatenate([pos, np.asarray(quat, np.float32).reshape(n, 4),
                           np.asarray(scale, np.float32).reshape(n, 3),
                           np.asarray(opacity, np.float32).reshape(n, 1),
                           np.asarray(diffuse, np.float32).reshape(n, 3)], axis=1).astype("<f4")
    L = int(np.asarray(sharpness).reshape(n, -1).shape[1]) if n else 0
    lob = np.concatenate([np.asarray(axis, np.float32).reshape(n, L, 3),
                          np.asarray(sharpness, np.float32).reshape(n, L, 1),
                          np.asarray(amplitude, np.float32).reshape(n, L, 3)], axis=2).astype("<f4")
    sizes = 57 + 28 * nl
    offs = np.zeros(n + 1, np.int64)
    np.cumsum(sizes, out=offs[1:])
    out = np.empty(12 + int(offs[-1]), np.uint8)
    out[:12] = np.frombuffer(MAGIC + struct.pack("<HI", FORMAT_VERSION, n), np.uint8)
    body = out[12:]
    body[(offs[:-1, None] + np.arange(56)[None, :]).reshape(-1)] = base.view(np.uint8).reshape(-1)
    body[offs[:-1] + 56] = nl.astype(np.uint8)
    if n and L:
        lb = lob.view(np.uint8).reshape(n, L, 28)
        slot = np.arange(L)[None, :] < nl[:, None]
        ii, ll = np.nonzero(slot)
        idx = (offs[ii] + 57 + 28 * ll)[:, None] + np.arange(28)[None, :]
        body[idx.reshape(-1)] = lb[ii, ll].reshape(-1)
    return out.tobytes()
