"""Host-buffer batch rendering: the end-to-end path a user of the reference's
``render(scene, cam)`` API takes for many views of one scene.

Per call: the scene's float32 SoA is copied host -> device once (from pinned
memory), every view is rendered on the compute stream, and each finished
image is copied device -> host on a side stream while the next view renders.
"""

from __future__ import annotations

import numpy as np
import torch

from .rasterizer import GRAD_FIELDS, GaussianTensors, Rasterizer

HOST_FIELDS = GRAD_FIELDS + ("lobe_mask",)


class PinnedScene:
    """Page-locked float32 copy of a scene's parameter arrays."""

    def __init__(self, p):
        self.arrays = {}
        for f in HOST_FIELDS:
            a = np.ascontiguousarray(np.asarray(getattr(p, f)), dtype=np.float32)
            t = torch.empty(a.shape, dtype=torch.float32, pin_memory=True)
            t.numpy()[...] = a
            self.arrays[f] = t
        pm = getattr(p, "prim_mask", None)
        self.prim_mask = None
        if pm is not None:
            a = np.ascontiguousarray(np.asarray(pm), dtype=np.float32)
            self.prim_mask = torch.empty(a.shape, dtype=torch.float32, pin_memory=True)
            self.prim_mask.numpy()[...] = a

    @property
    def nbytes(self) -> int:
        n = sum(t.numel() * 4 for t in self.arrays.values())
        return n + (0 if self.prim_mask is None else self.prim_mask.numel() * 4)

    def upload(self, device) -> GaussianTensors:
        dev = {f: t.to(device, non_blocking=True) for f, t in self.arrays.items()}
        pm = None if self.prim_mask is None else self.prim_mask.to(device, non_blocking=True)
        return GaussianTensors(**dev, prim_mask=pm)


class BatchRenderer:
    """render_views(pinned_scene, cams) -> list of (H, W, 3) float32 host arrays.

    Scenes are uploaded into one of two device-resident copies on a dedicated
    host-to-device stream, so with ``wait=False`` the upload of the next
    call's scene overlaps the renders and image read-backs of this one (the
    copy engines run both directions at once).  Every call still moves its
    whole scene host -> device and every image device -> host.

    Images are never silently truncated: every view's tile-entry overflow
    counter is gathered on the device and read once per call.  A view that
    outgrew its capacity grows it (dropping the graphs captured against the
    smaller workspace) and is re-rendered with the checked forward into the
    same host buffer -- at the end of the call with ``wait=True``, or, with
    ``wait=False``, when the call's slot is next used (the call after next)
    or at ``finish()``."""

    def __init__(self, rast: Rasterizer | None = None, device="cuda", streams: int = 8,
                 graphs: bool = True, slots: int = 2):
        self.rast = rast or Rasterizer(device=device)
        self.device = torch.device(device)
        self.h2d_stream = torch.cuda.Stream(device=self.device)
        self.streams = [torch.cuda.Stream(device=self.device) for _ in range(max(streams, 1))]
        # one read-back stream per render stream: an image leaves as soon as
        # its view is done, not behind an earlier view still rendering on
        # another stream (the link has only a few percent of slack)
        self.copy_streams = [torch.cuda.Stream(device=self.device) for _ in self.streams]
        self.copy_stream = self.copy_streams[0]
        self._host = {}
        self.slots = max(2, int(slots))  # calls in flight: device scene copies / image buffer sets
        self._dev = [None] * self.slots
        self._rendered = [[] for _ in range(self.slots)]  # per slot: the renders of its last use done
        self._copied = {}             # (slot, view): event, that device image's last read-back done
        self._pending = [None] * self.slots  # per slot: the unchecked overflow state of its last call
        self._ovf_dev = {}
        self._ovf_host = {}
        self._calls = 0
        self.graphs = graphs          # replay each (copy, view) render from a CUDA graph
        self._dev_out = {}
        self.rerendered = 0           # views re-rendered after an overflow (diagnostics)

    def _host_buf(self, k, shape):
        buf = self._host.get(k)
        if buf is None or tuple(buf.shape) != shape:
            buf = torch.empty(shape, dtype=torch.float32, pin_memory=True)
            self._host[k] = buf
        return buf

    def _ovf_bufs(self, slot: int, n: int):
        d = self._ovf_dev.get(slot)
        if d is None or d.shape[0] < n:
            d = torch.zeros((max(n, 1), 2), dtype=torch.int64, device=self.device)
            self._ovf_dev[slot] = d
            self._ovf_host[slot] = torch.zeros((max(n, 1), 2), dtype=torch.int64, pin_memory=True)
        return self._ovf_dev[slot], self._ovf_host[slot]

    def _upload(self, scene: PinnedScene, slot: int) -> GaussianTensors:
        dev = self._dev[slot]
        if dev is None or any(tuple(getattr(dev, f).shape) != tuple(t.shape)
                              for f, t in scene.arrays.items()) or \
                (dev.prim_mask is None) != (scene.prim_mask is None):
            with torch.cuda.stream(self.h2d_stream):
                for ev in self._rendered[slot]:
                    self.h2d_stream.wait_event(ev)
                arrs = {f: torch.empty(t.shape, dtype=torch.float32, device=self.device)
                        for f, t in scene.arrays.items()}
                pm = None if scene.prim_mask is None else torch.empty(
                    scene.prim_mask.shape, dtype=torch.float32, device=self.device)
            dev = GaussianTensors(**arrs, prim_mask=pm)
            self._dev[slot] = dev
        with torch.cuda.stream(self.h2d_stream):
            # the scene copy is overwritten once the renders that read it are
            # done -- its images' read-backs may still be in flight
            for ev in self._rendered[slot]:
                self.h2d_stream.wait_event(ev)
            for f, t in scene.arrays.items():
                getattr(dev, f).copy_(t, non_blocking=True)
            if scene.prim_mask is not None:
                dev.prim_mask.copy_(scene.prim_mask, non_blocking=True)
        return dev

    def _resolve(self, slot: int) -> None:
        """Check the overflow counters of the slot's last call (its device
        scene copy is still intact) and re-render every view that outgrew
        its capacity into that call's host buffer."""
        pend = self._pending[slot]
        if pend is None:
            return
        self._pending[slot] = None
        done, ovf_host, cams, outs, background = pend
        done.synchronize()
        o = ovf_host[:len(cams)].numpy()
        bad = [k for k in range(len(cams)) if o[k, 0]]
        if not bad:
            return
        g = self._dev[slot]
        for k in bad:
            self.rast.grow_capacity(g, cams[k], int(o[k, 1]))
        main = torch.cuda.current_stream(self.device)
        for k in bad:
            img = self.rast.forward(g, cams[k], background, check=True, track=False).img
            outs[k].copy_(img)
            self.rerendered += 1
        main.synchronize()

    def finish(self) -> None:
        """Wait for every call in flight and resolve its overflow checks:
        after this, every image a ``wait=False`` call returned is final."""
        torch.cuda.synchronize(self.device)
        for slot in range(self.slots):
            self._resolve(slot)

    def render_views(self, scene: PinnedScene, cams, background=(0.0, 0.0, 0.0), check=False,
                     wait: bool = True):
        """Upload the scene, render every view (spread over the render streams
        so binning of one view overlaps the raster of another), copy each
        image back as soon as it is done; returns the pinned host images.
        With ``wait=False`` the call returns once everything is enqueued: the
        images are complete after ``finish()`` or once the call after next
        returns (the host buffers are then reused by the call after that)."""
        cams = list(cams)
        slot = self._calls % self.slots
        self._calls += 1
        self._resolve(slot)  # the slot's last call: overflow checked before its copy is reused
        main = torch.cuda.current_stream(self.device)
        g = self._upload(scene, slot)  # waits for the renders and read-backs of the copy's last use
        up = torch.cuda.Event()
        up.record(self.h2d_stream)
        ovf_dev, ovf_host = self._ovf_bufs(slot, len(cams))
        outs = []
        for k, cam in enumerate(cams):
            s = self.streams[k % len(self.streams)]
            s.wait_event(up)
            if (slot, k) in self._copied:  # this device image buffer's previous read-back
                s.wait_event(self._copied[(slot, k)])
            with torch.cuda.stream(s):
                if self.graphs and not check:
                    H, W = int(cam.height), int(cam.width)
                    buf = self._dev_out.get((slot, k))
                    if buf is None or tuple(buf[0].shape) != (H, W, 3):
                        buf = (torch.empty((H, W, 3), dtype=torch.float32, device=self.device),
                               torch.empty((H, W), dtype=torch.float32, device=self.device))
                        self._dev_out[(slot, k)] = buf
                    ovf_dev[k].copy_(self.rast.graph_forward(g, cam, buf, background))
                    img = buf[0]
                else:
                    fr = self.rast.forward(g, cam, background, check=check, track=False)
                    fr.record_overflow(ovf_dev[k])
                    img = fr.img
                done = torch.cuda.Event()
                done.record(s)
            host = self._host_buf((slot, k), tuple(img.shape))
            cs = self.copy_streams[k % len(self.streams)]
            with torch.cuda.stream(cs):
                cs.wait_event(done)
                host.copy_(img, non_blocking=True)
                img.record_stream(cs)
                copied = torch.cuda.Event()
                copied.record(cs)
                self._copied[(slot, k)] = copied
            outs.append(host)
        rendered = []
        for s in self.streams:
            ev = torch.cuda.Event()
            ev.record(s)
            rendered.append(ev)
        self._rendered[slot] = rendered
        for s in self.streams + self.copy_streams[1:]:
            self.copy_stream.wait_stream(s)
        with torch.cuda.stream(self.copy_stream):
            ovf_host[:len(cams)].copy_(ovf_dev[:len(cams)], non_blocking=True)
        ready = torch.cuda.Event()
        ready.record(self.copy_stream)
        main.wait_stream(self.copy_stream)
        self._pending[slot] = (ready, ovf_host, cams, outs, background)
        if wait:
            self._resolve(slot)
        return outs

    @staticmethod
    def d2h_bytes(cams) -> int:
        return sum(int(c.width) * int(c.height) * 3 * 4 for c in cams)
