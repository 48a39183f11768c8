"""Device-side render pipeline: PyTorch owns memory and streams, libsgs.so
does every computation.

``Rasterizer.forward`` = preprocess (K1) -> bin (K2-K4) -> raster (K5) and
``Rasterizer.backward`` = raster backward (K6) -> preprocess backward (K7),
all enqueued on the current torch stream through the C ABI.  There is no
CPU fallback: a missing or unloadable libsgs.so raises.

Workspaces are single torch byte tensors carved by the library, so
``torch.cuda.max_memory_allocated`` sees all render VRAM (the paper's VRAM
protocol).  The tile-entry capacity grows geometrically on
overflow; overflow is detected from the device counters (one 56-byte D2H
read) when ``check=True`` or by ``Frame.ensure_ok()``.
"""

from __future__ import annotations

import collections
import ctypes as C
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _ffi
from .camera import to_sgs

GRAD_FIELDS = ("position", "quat", "log_scale", "opacity", "diffuse", "axis_raw", "sharpness",
               "amplitude")


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def _dev_f32(a, device) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.detach().to(device=device, dtype=torch.float32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float32))).to(device)


class _PinnedArena:
    """One growing page-locked float32 host buffer.  Host arrays (the drop-in
    API's float64 SceneParams, bool lobe masks, ...) are narrowed into it by
    torch's multithreaded copy and cross the link at the full pinned
    bandwidth, each array's copy issued as soon as it is narrowed so the
    transfers overlap the narrowing of the next arrays; numpy's
    single-threaded astype plus a pageable copy took 1.6x as long for
    configs[2] (1M Gaussians)."""

    def __init__(self):
        self.buf = None
        self.lock = threading.Lock()
        self.stream = None

    @staticmethod
    def _host(a) -> np.ndarray:
        a = np.ascontiguousarray(np.asarray(a))
        if not a.dtype.isnative or a.dtype.kind not in "fbiu":  # torch.from_numpy needs native numbers
            a = np.ascontiguousarray(a, dtype=np.float32)
        return a

    def upload(self, arrays, device) -> list:
        arrays = [self._host(a) for a in arrays]
        sizes = [a.size for a in arrays]
        # each array starts on a 256-byte boundary (the kernels' float4 loads
        # need 16, coalescing likes 256)
        offs = np.concatenate([[0], np.cumsum([(n + 63) // 64 * 64 for n in sizes])]).astype(np.int64)
        total = max(64, int(offs[-1]))
        with self.lock:
            if self.buf is None or self.buf.numel() < total:
                self.buf = None
                self.buf = torch.empty(total + total // 4, dtype=torch.float32, pin_memory=True)
            if self.stream is None or self.stream.device != device:
                self.stream = torch.cuda.Stream(device)
            cur = torch.cuda.current_stream(device)
            dev = torch.empty(total, dtype=torch.float32, device=device)
            self.stream.wait_stream(cur)  # dev is allocated on the current stream
            for a, n, o, o1 in zip(arrays, sizes, offs[:-1], offs[1:]):
                if n:
                    self.buf[o:o + n].view(a.shape).copy_(torch.from_numpy(a))
                with torch.cuda.stream(self.stream):  # this array crosses while the next narrows
                    dev[o:o1].copy_(self.buf[o:o1], non_blocking=True)
            self.stream.synchronize()  # the arena is free again on return
            cur.wait_stream(self.stream)
        return [dev[o:o + n].view(a.shape) for a, n, o in zip(arrays, sizes, offs)]

    def download64(self, t: torch.Tensor) -> np.ndarray:
        """float64 host copy of a device float32 tensor: one pinned D2H copy,
        then a multithreaded widening into the new array."""
        n = t.numel()
        with self.lock:
            if self.buf is None or self.buf.numel() < n:
                self.buf = None
                self.buf = torch.empty(n + n // 4, dtype=torch.float32, pin_memory=True)
            h = self.buf[:n].view(t.shape)
            h.copy_(t)
            out = np.empty(tuple(t.shape), dtype=np.float64)
            torch.from_numpy(out).copy_(h)
        return out


_UPLOAD = _PinnedArena()
_DOWNLOAD = _PinnedArena()


def host_to_device_f32(arrays, device) -> list:
    """float32 device copies of host arrays (see _PinnedArena)."""
    device = torch.device(device)
    if device.type != "cuda" or not torch.cuda.is_available():
        return [_dev_f32(a, device) for a in arrays]
    if device.index is None:
        device = torch.device("cuda", torch.cuda.current_device())
    return _UPLOAD.upload(arrays, device)


def device_to_host_f64(t: torch.Tensor) -> np.ndarray:
    """float64 numpy copy of a tensor (the drop-in API returns float64)."""
    t = t.detach()
    if t.is_cuda and t.dtype == torch.float32 and t.is_contiguous() and t.numel() >= (1 << 16):
        return _DOWNLOAD.download64(t)
    return t.to(torch.float64).cpu().numpy()


class GaussianTensors:
    """Device float32 SoA of one scene (SceneParams layout + soft masks)."""

    def __init__(self, position, quat, log_scale, opacity, diffuse, axis_raw, sharpness, amplitude,
                 lobe_mask=None, prim_mask=None):
        self.position = position
        self.quat = quat
        self.log_scale = log_scale
        self.opacity = opacity
        self.diffuse = diffuse
        self.axis_raw = axis_raw
        self.sharpness = sharpness
        self.amplitude = amplitude
        n, L = position.shape[0], axis_raw.shape[1] if axis_raw.dim() == 3 else 0
        if lobe_mask is None:
            lobe_mask = torch.ones((n, L), dtype=torch.float32, device=position.device)
        self.lobe_mask = lobe_mask
        self.prim_mask = prim_mask
        self._check()

    def _check(self):
        n = self.position.shape[0]
        L = self.n_lobes
        shapes = {"position": (n, 3), "quat": (n, 4), "log_scale": (n, 3), "opacity": (n,),
                  "diffuse": (n, 3), "axis_raw": (n, L, 3), "sharpness": (n, L),
                  "amplitude": (n, L, 3), "lobe_mask": (n, L)}
        for k, shp in shapes.items():
            t = getattr(self, k)
            if tuple(t.shape) != shp:
                raise ValueError(f"{k} has shape {tuple(t.shape)}, expected {shp}")
            if t.dtype != torch.float32 or not t.is_contiguous() or not t.is_cuda:
                raise ValueError(f"{k} must be a contiguous float32 CUDA tensor")
        if self.prim_mask is not None and tuple(self.prim_mask.shape) != (n,):
            raise ValueError("prim_mask must have shape (N,)")

    @property
    def n(self) -> int:
        return int(self.position.shape[0])

    @property
    def n_lobes(self) -> int:
        return int(self.axis_raw.shape[1])

    @property
    def device(self):
        return self.position.device

    @classmethod
    def from_arrays(cls, p, device="cuda", prim_mask=None) -> "GaussianTensors":
        """From any object with SceneParams attributes (numpy or torch; the
        reference's f64 SceneParams, this package's SceneArrays, ...).  A bool
        lobe_mask becomes 0/1 floats; ``prim_mask`` falls back to
        ``p.prim_mask`` when present."""
        lm = getattr(p, "lobe_mask", None)
        pm = prim_mask if prim_mask is not None else getattr(p, "prim_mask", None)
        src = {f: getattr(p, f) for f in GRAD_FIELDS}
        src["lobe_mask"], src["prim_mask"] = lm, pm
        names = [f for f, a in src.items() if a is not None]
        if any(isinstance(src[f], torch.Tensor) for f in names):
            kw = {f: (None if src[f] is None else _dev_f32(src[f], device)) for f in src}
        else:  # host arrays: one staged copy (host_to_device_f32)
            kw = dict.fromkeys(src)
            kw.update(zip(names, host_to_device_f32([src[f] for f in names], device)))
        return cls(**kw)

    def c_params(self) -> _ffi.SgsParams:
        s = _ffi.SgsParams()
        for f in GRAD_FIELDS + ("lobe_mask",):
            setattr(s, f, _ptr(getattr(self, f)))
        s.prim_mask = _ptr(self.prim_mask)
        s.n = self.n
        s.n_lobes = self.n_lobes
        return s


class Workspace:
    """One device byte buffer carved by libsgs.so for (N, L, W, H, capacity)."""

    def __init__(self, n, n_lobes, width, height, capacity, sort_mode, device):
        self.desc = _ffi.SgsWorkspace()
        self.desc.n, self.desc.n_lobes = int(n), int(n_lobes)
        self.desc.width, self.desc.height = int(width), int(height)
        self.desc.sort_mode = int(sort_mode)
        self.desc.entry_capacity = int(capacity)
        nbytes = C.c_uint64()
        _ffi.call("sgs_workspace_size", C.byref(self.desc), C.byref(nbytes))
        self.buf = torch.empty(int(nbytes.value), dtype=torch.uint8, device=device)
        self.desc.base = self.buf.data_ptr()
        self.desc.bytes = int(nbytes.value)

    @property
    def capacity(self) -> int:
        return int(self.desc.entry_capacity)

    @property
    def nbytes(self) -> int:
        return int(self.desc.bytes)

    def stats(self) -> dict:
        s = _ffi.SgsStats()
        _ffi.call("sgs_get_stats", C.byref(self.desc), C.byref(s), C.c_void_p(_stream_ptr()))
        return {k: int(getattr(s, k)) for k, _ in _ffi.SgsStats._fields_}


@dataclass
class Frame:
    """Outputs of one forward render plus what the backward needs."""

    img: torch.Tensor          # (H, W, 3) float32
    final_T: torch.Tensor      # (H, W) float32
    ncontrib: torch.Tensor | None  # (H, W) int32 (uint32 on the device); None if not tracked
    ws: Workspace
    cam: _ffi.SgsCamera
    bg: tuple

    def stats(self) -> dict:
        return self.ws.stats()

    def record_overflow(self, dst: torch.Tensor) -> None:
        """Copy this frame's (overflow, binned entries) counters into the int64
        device tensor ``dst`` (2 elements) without a host round trip, so a
        caller can check many frames with one read (Counters layout,
        common.cuh: overflow at u64 slot 4, n_bin at slot 7)."""
        c = self.ws.buf[:64].view(torch.int64)
        dst[0].copy_(c[4])
        dst[1].copy_(c[7])


MAX_CAPACITY = (1 << 30) - 1


@dataclass
class _GraphEntry:
    """A captured image-only forward and everything its raw pointers refer to."""

    graph: "torch.cuda.CUDAGraph"
    ws: Workspace
    key: tuple                 # (n, lobes, W, H): the capacity-hint key
    ovf: torch.Tensor          # int64 (overflow, binned entries), written by each replay
    keep: tuple                # scene and output tensors the graph reads / writes


class Rasterizer:
    """Reusable render context (workspace cache + capacity policy)."""

    def __init__(self, sort_mode: int = _ffi.SORT_DEPTH_FIRST, device="cuda", headroom=1.25,
                 initial_capacity: int | None = None, max_graphs: int = 256):
        _ffi.load()
        self.sort_mode = sort_mode
        self.device = torch.device(device)
        self.headroom = headroom
        self.initial_capacity = initial_capacity
        self._cap_hint: dict = {}
        # captured view graphs kept (each holds its scene, output and
        # workspace buffers alive); the least recently replayed go first
        self.max_graphs = int(max_graphs)
        self._shared: dict = {}

    # --------------------------------------------------------------- workspace
    def _key(self, g, cam):
        return (g.n, g.n_lobes, int(cam.width), int(cam.height))

    def _capacity(self, key, g) -> int:
        if key in self._cap_hint:
            return self._cap_hint[key]
        if self.initial_capacity is not None:
            return self.initial_capacity
        return int(min(MAX_CAPACITY, max(1 << 16, 4 * g.n)))

    def workspace(self, g, cam, private=False, capacity=None) -> Workspace:
        """The shared workspace for this (scene size, image size) on the
        current stream (one per stream, so views on different streams render
        concurrently), or a private one.  A shared workspace that is too small
        is replaced; CUDA graphs captured against it are dropped first (they
        hold its raw pointers), see _retire."""
        key = self._key(g, cam)
        cap = capacity if capacity is not None else self._capacity(key, g)
        if private:
            return Workspace(*key[:4], cap, self.sort_mode, self.device)
        skey = key + (_stream_ptr(),)
        ws = self._shared.get(skey)
        if ws is None or ws.capacity < cap:
            if ws is not None:
                self._retire(ws)
            self._shared.pop(skey, None)
            ws = Workspace(*key[:4], cap, self.sort_mode, self.device)
            self._shared[skey] = ws
        return ws

    def _retire(self, ws: Workspace) -> None:
        """Drop every captured graph bound to ``ws`` before the workspace can
        be freed.  Graph workspaces are allocated on a capture stream but
        replayed on the caller's, so the device is synchronised first: no
        replay may still be writing into the buffer the allocator is about
        to hand out again."""
        graphs = self.__dict__.get("_graphs", {})
        dead = [k for k, e in graphs.items() if e.ws is ws]
        if dead:
            torch.cuda.synchronize(self.device)
            for k in dead:
                del graphs[k]

    def _set_hint(self, key, need: int) -> None:
        """Raise (never lower) the capacity hint for ``key``; captured graphs
        whose workspace is now too small are dropped and recaptured on their
        next use."""
        cap = max(self._cap_hint.get(key, 0), min(MAX_CAPACITY, int(need)))
        self._cap_hint[key] = cap
        graphs = self.__dict__.get("_graphs", {})
        small = [k for k, e in graphs.items() if e.key == key and e.ws.capacity < cap]
        if small:
            torch.cuda.synchronize(self.device)
            for k in small:
                del graphs[k]

    def grow_capacity(self, g, cam, n_entries: int) -> None:
        """Size the tile-entry capacity for ``n_entries`` binned entries (the
        deferred form of forward(check=True)'s retry).  The hint only grows:
        several views overflowing in one pass keep the largest need."""
        if n_entries > MAX_CAPACITY:
            raise _ffi.CapacityError("sgs_bin", _ffi.SGS_E_CAPACITY,
                                     f"{n_entries} entries exceed one bin call's limit {MAX_CAPACITY}")
        self._set_hint(self._key(g, cam), int(n_entries * self.headroom) + 1024)

    def release(self):
        self.release_graphs()
        self._shared.clear()

    # ------------------------------------------------------------------ forward
    def forward(self, g: GaussianTensors, cam, background=(0.0, 0.0, 0.0), weight_sums=None,
                check=True, private=False, tile_rows=None, out=None, pair_count=None,
                track=True, weight_fx=None, grad_floor: float = 0.0, _events=None) -> Frame:
        # _events (timing hooks): (raster start, raster end[, preprocess start,
        # preprocess end]) CUDA events recorded on the current stream
        """Render one view.  ``weight_sums`` (N float32 device tensor) is
        accumulated in place (render.py:406-407); ``weight_fx`` (N int64,
        fixed point in 2^-32 units) instead accumulates the exact integer
        sums, for several views to be added order-independently and
        converted once (``fixed_to_float``).  ``out`` may supply
        preallocated (img, T, nc) tensors.  ``track=False`` renders the image
        (and T) only, skipping the per-pixel contributor counts the backward
        needs (an image-only render, render.py:411).  ``grad_floor``: bin
        every primitive with at least this opacity's support (gradient
        renders: primitives at o_eff = 0 still get dL/do, see sgs.h)."""
        c_cam = to_sgs(cam, tile_rows, grad_floor=grad_floor)
        bg = tuple(float(v) for v in np.asarray(background, dtype=np.float64).reshape(3))
        c_bg = (C.c_float * 3)(*bg)
        H, W = int(cam.height), int(cam.width)
        if out is None:
            img = torch.empty((H, W, 3), dtype=torch.float32, device=self.device)
            T = torch.empty((H, W), dtype=torch.float32, device=self.device)
            nc = torch.empty((H, W), dtype=torch.int32, device=self.device) if track else None
        else:
            img, T, nc = out
            if not track:
                nc = None
        if weight_sums is not None:
            if weight_sums.dtype != torch.float32 or tuple(weight_sums.shape) != (g.n,):
                raise ValueError("weight_sums must be a float32 (N,) tensor")
            if weight_fx is not None:
                raise ValueError("pass weight_sums or weight_fx, not both")
            weight_fx = torch.zeros(g.n, dtype=torch.int64, device=self.device)
            to_float = weight_sums
        else:
            to_float = None
        if weight_fx is not None and (weight_fx.dtype != torch.int64 or tuple(weight_fx.shape) != (g.n,)):
            raise ValueError("weight_fx must be an int64 (N,) tensor")
        params = g.c_params()
        stream = C.c_void_p(_stream_ptr())
        key = self._key(g, cam)
        while True:
            ws = self.workspace(g, cam, private=private)
            if _events is not None and len(_events) > 2:
                _events[2].record()
            _ffi.call("sgs_preprocess", C.byref(params), C.byref(c_cam), C.byref(ws.desc), stream)
            if _events is not None and len(_events) > 2:
                _events[3].record()
            _ffi.call("sgs_bin", C.byref(c_cam), C.byref(ws.desc), stream)
            if check:
                st = ws.stats()
                if st["overflow"]:
                    need = int(st["n_bin_entries"] * self.headroom) + 1024
                    if st["n_bin_entries"] > MAX_CAPACITY:
                        raise _ffi.CapacityError(
                            "sgs_bin", _ffi.SGS_E_CAPACITY,
                            f"{st['n_bin_entries']} entries exceed one bin call's limit "
                            f"{MAX_CAPACITY}; render in tile-row strips")
                    self._set_hint(key, need)
                    continue
            break
        if _events is not None:
            _events[0].record()
        _ffi.call("sgs_raster_forward", C.byref(c_cam), c_bg, C.byref(ws.desc), _ptr(img), _ptr(T),
                  _ptr(nc), _ptr(weight_fx), _ptr(pair_count), stream)
        if _events is not None:
            _events[1].record()
        if to_float is not None:
            fixed_to_float(weight_fx, to_float, accumulate=True)
        return Frame(img=img, final_T=T, ncontrib=nc, ws=ws, cam=c_cam, bg=bg)

    def preprocess_only(self, g: GaussianTensors, cam, tile_rows=None):
        """K1 alone (no binning, no raster): per-primitive (depth bits, packed
        tile rectangle, tile count) device tensors, e.g. for strip planning
        (sharding.row_costs_from_rects).  Uses a private workspace of
        capacity 1."""
        c_cam = to_sgs(cam, tile_rows)
        ws = self.workspace(g, cam, private=True, capacity=1)
        _ffi.call("sgs_preprocess", C.byref(g.c_params()), C.byref(c_cam), C.byref(ws.desc),
                  C.c_void_p(_stream_ptr()))
        fr = Frame(img=None, final_T=None, ncontrib=None, ws=ws, cam=c_cam, bg=(0.0, 0.0, 0.0))
        depth, rect, tt, _ = self.export_projected(fr)
        return depth, rect, tt

    # ------------------------------------------------------- graph forward
    def graph_forward(self, g: GaussianTensors, cam, out, background=(0.0, 0.0, 0.0),
                      tile_rows=None) -> torch.Tensor:
        """Image-only forward of one view replayed from a CUDA graph on the
        current stream (one graph launch instead of ~20 kernel launches and
        ~3 FFI calls of host work per view).  The graph is captured on first
        use for this (scene buffers, camera, output buffers, stream) and
        re-reads the scene tensors at every replay, so in-place parameter
        updates are seen.  ``out`` = (img, T) device tensors.

        The entry keeps references to everything the graph writes or reads
        (workspace, scene and output tensors), so none of them can be freed
        and reused under it; a capacity growth drops the graphs bound to the
        smaller workspace (_retire / _set_hint).  Returns the entry's int64
        (overflow, binned entries) device pair, written by the replay: a
        frame denser than the capacity the graph was captured with sets it,
        and the caller must check it (BatchRenderer does, once per call)."""
        c = to_sgs(cam, tile_rows)
        stream = torch.cuda.current_stream(self.device)
        scene_t = tuple(getattr(g, f) for f in GRAD_FIELDS + ("lobe_mask",)) + (g.prim_mask,)
        key = (bytes(c), tuple(_ptr(t) for t in scene_t), g.n, g.n_lobes, out[0].data_ptr(),
               out[1].data_ptr(), stream.cuda_stream, tuple(float(v) for v in background))
        graphs = self.__dict__.setdefault("_graphs", collections.OrderedDict())
        e = graphs.get(key)
        if e is not None:
            graphs.move_to_end(key)
        else:
            if len(graphs) >= self.max_graphs:
                # least recently replayed first; its buffers may still be in
                # use by a replay in flight
                torch.cuda.synchronize(self.device)
                while len(graphs) >= self.max_graphs:
                    graphs.popitem(last=False)
            # capture on a private (non-default) stream paired with the caller's
            # stream; its workspace belongs to that pairing, so graphs replayed
            # concurrently on different streams never share scratch
            caps = self.__dict__.setdefault("_capture_streams", {})
            cap = caps.get(stream.cuda_stream)
            if cap is None:
                cap = torch.cuda.Stream(device=self.device)
                caps[stream.cuda_stream] = cap
            cap.wait_stream(stream)
            ovf = torch.zeros(2, dtype=torch.int64, device=self.device)
            with torch.cuda.stream(cap):
                self.forward(g, cam, background, check=True, tile_rows=tile_rows,
                             out=(out[0], out[1], None), track=False)
            cap.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=cap):
                fr = self.forward(g, cam, background, check=False, tile_rows=tile_rows,
                                  out=(out[0], out[1], None), track=False)
                fr.record_overflow(ovf)
            stream.wait_stream(cap)
            e = _GraphEntry(gr, fr.ws, self._key(g, cam), ovf, scene_t + tuple(out))
            graphs[key] = e
        e.graph.replay()
        return e.ovf

    def release_graphs(self):
        if self.__dict__.get("_graphs"):
            torch.cuda.synchronize(self.device)
        self.__dict__.pop("_graphs", None)

    # ----------------------------------------------------------------- backward
    def backward(self, g: GaussianTensors, frame: Frame, dimg: torch.Tensor,
                 mask_grads: bool = True, out: dict | None = None, accumulate: bool = False,
                 mask_logit: bool = False, deterministic: bool = False) -> dict:
        """dL/dparams for dL/dimg (H,W,3).  Returns a dict of float32 tensors
        shaped like the parameters (+ 'lobe_mask' / 'prim_mask' when
        ``mask_grads``) and 'grad2d' (N,9).  ``out`` supplies the output
        tensors (contiguous float32, parameter-shaped, 'quat' 16-byte
        aligned); with ``accumulate`` the gradients are added into them, and
        with ``mask_logit`` the mask gradients are taken with respect to the
        logits whose sigmoids are the masks (x m (1 - m)).  ``deterministic``:
        bitwise-reproducible raster sums (sgs_raster_backward_det, ~2x K6)."""
        grad2d = self.backward_raster(g, frame, dimg, deterministic=deterministic)
        out = self.backward_params(g, frame.cam, grad2d, mask_grads=mask_grads, out=out,
                                   accumulate=accumulate, mask_logit=mask_logit)
        out["grad2d"] = grad2d
        return out

    def backward_raster(self, g: GaussianTensors, frame: Frame, dimg: torch.Tensor,
                        deterministic: bool = False) -> torch.Tensor:
        """K6 alone: the (N, 9) per-primitive image-space partials for dL/dimg
        (``deterministic``: order-independent fixed-point sums)."""
        dimg = dimg.to(device=self.device, dtype=torch.float32).contiguous()
        if frame.ncontrib is None:
            raise ValueError("frame was rendered with track=False; the backward needs track=True")
        if tuple(dimg.shape) != tuple(frame.img.shape):
            raise ValueError(f"dimg shape {tuple(dimg.shape)} != image {tuple(frame.img.shape)}")
        c_bg = (C.c_float * 3)(*frame.bg)
        grad2d = torch.empty((g.n, 9), dtype=torch.float32, device=self.device)
        if deterministic:
            nb = int(_ffi.load().sgs_raster_backward_det_scratch_bytes(g.n))
            scratch = torch.empty(nb, dtype=torch.uint8, device=self.device)
            _ffi.call("sgs_raster_backward_det", C.byref(frame.cam), c_bg, C.byref(frame.ws.desc),
                      _ptr(frame.img), _ptr(frame.final_T), _ptr(frame.ncontrib), _ptr(dimg),
                      _ptr(grad2d), _ptr(scratch), nb, C.c_void_p(_stream_ptr()))
            return grad2d
        _ffi.call("sgs_raster_backward", C.byref(frame.cam), c_bg, C.byref(frame.ws.desc),
                  _ptr(frame.img), _ptr(frame.final_T), _ptr(frame.ncontrib), _ptr(dimg),
                  _ptr(grad2d), C.c_void_p(_stream_ptr()))
        return grad2d

    def backward_params(self, g: GaussianTensors, c_cam, grad2d: torch.Tensor, mask_grads: bool = True,
                        out: dict | None = None, accumulate: bool = False,
                        mask_logit: bool = False) -> dict:
        """K7 alone: parameter (and mask) gradients from K6's partials, on the
        current stream (``c_cam`` = the frame's sgs_camera)."""
        return self.backward_params_views(g, [c_cam], [grad2d], mask_grads, out, accumulate, mask_logit)

    def backward_params_views(self, g: GaussianTensors, c_cams, grad2ds, mask_grads: bool = True,
                              out: dict | None = None, accumulate: bool = False,
                              mask_logit: bool = False) -> dict:
        """K7 over several views (``c_cams`` / ``grad2ds``: their sgs_cameras and
        K6 partials): the sum of the per-view gradients in view order, with
        the parameters read and the gradient rows written once per 8 views
        (sgs_preprocess_backward_views)."""
        if len(c_cams) != len(grad2ds) or not c_cams:
            raise ValueError("one K6 partial buffer per camera, at least one view")
        for t in grad2ds:
            if t.dtype != torch.float32 or not t.is_contiguous() or t.numel() != g.n * 9:
                raise ValueError("K6 partials must be contiguous float32 (N, 9) tensors")
        if out is None:
            if accumulate:
                raise ValueError("accumulate=True needs the output tensors")
            out = {f: torch.empty_like(getattr(g, f)) for f in GRAD_FIELDS}
            if mask_grads:
                out["lobe_mask"] = torch.empty_like(g.lobe_mask)
                out["prim_mask"] = torch.empty((g.n,), dtype=torch.float32, device=self.device)
        else:
            out = dict(out)
            for f in GRAD_FIELDS + (("lobe_mask", "prim_mask") if mask_grads else ()):
                t = out.get(f)
                numel = g.n if f == "prim_mask" else getattr(g, f).numel()
                if t is None or t.dtype != torch.float32 or not t.is_contiguous() or t.numel() != numel:
                    raise ValueError(f"gradient output '{f}' must be a contiguous float32 tensor "
                                     f"of {numel} elements")
        cg = _ffi.SgsGrads()
        cg.flags = (_ffi.GRADS_ACCUMULATE if accumulate else 0) | (_ffi.GRADS_MASK_LOGIT if mask_logit else 0)
        for f in GRAD_FIELDS:
            setattr(cg, f, _ptr(out[f]))
        cg.lobe_mask = _ptr(out.get("lobe_mask")) if mask_grads else None
        cg.prim_mask = _ptr(out.get("prim_mask")) if mask_grads else None
        params = g.c_params()
        if len(c_cams) == 1:
            _ffi.call("sgs_preprocess_backward", C.byref(params), C.byref(c_cams[0]), _ptr(grad2ds[0]),
                      C.byref(cg), C.c_void_p(_stream_ptr()))
            return out
        cams = (_ffi.SgsCamera * len(c_cams))(*c_cams)
        ptrs = (C.c_void_p * len(grad2ds))(*[t.data_ptr() for t in grad2ds])
        _ffi.call("sgs_preprocess_backward_views", C.byref(params), cams, len(c_cams), ptrs, C.byref(cg),
                  C.c_void_p(_stream_ptr()))
        return out

    # ----------------------------------------------------------------- exports
    DEBUG_BUFFERS = ("counters", "rec_geo", "rec_con", "rec_col", "depth_key", "rect",
                     "tiles_touched", "dkey_alt", "dkey_tmp", "didx", "didx_alt", "offsets",
                     "scan_blocks", "ent_key", "ent_key_alt", "ent_val", "ent_val_alt", "ranges",
                     "hist", "status")

    @staticmethod
    def debug_view(frame: Frame, name: str, count: int, dtype=torch.int32) -> torch.Tensor:
        """Copy of `count` elements of an internal workspace buffer (debugging)."""
        ptr = C.c_void_p()
        off = C.c_uint64()
        _ffi.call("sgs_debug_buffer", C.byref(frame.ws.desc),
                  Rasterizer.DEBUG_BUFFERS.index(name), C.byref(ptr), C.byref(off))
        nbytes = count * torch.tensor([], dtype=dtype).element_size()
        return frame.ws.buf[off.value:off.value + nbytes].view(dtype).clone()

    def export_bins(self, frame: Frame):
        """(keys u64 as int64, values int32, ranges (T,2) int32) of the sorted tile list."""
        st = frame.ws.stats()
        n = int(st["n_entries"])
        keys = torch.empty(max(n, 1), dtype=torch.int64, device=self.device)
        vals = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        tiles = ((frame.cam.width + 15) // 16) * ((frame.cam.height + 15) // 16)
        ranges = torch.empty((tiles, 2), dtype=torch.int32, device=self.device)
        _ffi.call("sgs_export_bins", C.byref(frame.ws.desc), C.byref(frame.cam), _ptr(keys),
                  _ptr(vals), _ptr(ranges), C.c_void_p(_stream_ptr()))
        return keys[:n], vals[:n], ranges

    def export_projected(self, frame: Frame):
        n = int(frame.ws.desc.n)
        depth = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        rect = torch.empty((max(n, 1), 2), dtype=torch.int32, device=self.device)
        tt = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        rec = torch.empty((max(n, 1), 16), dtype=torch.float32, device=self.device)
        _ffi.call("sgs_export_projected", C.byref(frame.ws.desc), _ptr(depth), _ptr(rect),
                  _ptr(tt), _ptr(rec), C.c_void_p(_stream_ptr()))
        return depth[:n], rect[:n], tt[:n], rec[:n]


def fixed_to_float(fx: torch.Tensor, out: torch.Tensor, accumulate: bool = False,
                   frac_bits: int = _ffi.WEIGHT_FRAC_BITS) -> torch.Tensor:
    """out (+)= fx * 2^-frac_bits (int64 fixed point -> float32), on the device."""
    if fx.dtype != torch.int64 or out.dtype != torch.float32 or fx.numel() != out.numel():
        raise ValueError("fixed_to_float needs an int64 source and a float32 output of equal size")
    _ffi.call("sgs_fixed_to_float", _ptr(fx), fx.numel(), int(frac_bits), _ptr(out), int(accumulate),
              C.c_void_p(_stream_ptr()))
    return out


def sort_pairs_u64(keys: torch.Tensor, vals: torch.Tensor, key_bits: int) -> None:
    """In-place stable radix sort of int64-stored u64 keys with int32 values."""
    n = keys.numel()
    tb = C.c_uint64()
    _ffi.call("sgs_sort_temp_size", n, key_bits, C.byref(tb))
    tmp = torch.empty(int(tb.value), dtype=torch.uint8, device=keys.device)
    _ffi.call("sgs_sort_pairs_u64", _ptr(keys), _ptr(vals), n, key_bits, _ptr(tmp),
              int(tb.value), C.c_void_p(_stream_ptr()))


class RenderFunction(torch.autograd.Function):
    """Autograd wrapper: image = render(params) with the CUDA backward."""

    @staticmethod
    def forward(ctx, rast, cam, background, position, quat, log_scale, opacity, diffuse, axis_raw,
                sharpness, amplitude, lobe_mask, prim_mask):
        g = GaussianTensors(position.detach(), quat.detach(), log_scale.detach(),
                            opacity.detach(), diffuse.detach(), axis_raw.detach(),
                            sharpness.detach(), amplitude.detach(), lobe_mask.detach(),
                            None if prim_mask is None else prim_mask.detach())
        frame = rast.forward(g, cam, background, private=True)
        ctx.rast, ctx.g, ctx.frame = rast, g, frame
        ctx.has_pm = prim_mask is not None
        return frame.img

    @staticmethod
    def backward(ctx, dimg):
        gr = ctx.rast.backward(ctx.g, ctx.frame, dimg, mask_grads=True)
        ctx.frame = None
        return (None, None, None, *[gr[f] for f in GRAD_FIELDS], gr["lobe_mask"],
                gr["prim_mask"] if ctx.has_pm else None)


def render_torch(rast: Rasterizer, cam, background, position, quat, log_scale, opacity, diffuse,
                 axis_raw, sharpness, amplitude, lobe_mask, prim_mask=None) -> torch.Tensor:
    return RenderFunction.apply(rast, cam, background, position, quat, log_scale, opacity,
                                diffuse, axis_raw, sharpness, amplitude, lobe_mask, prim_mask)
