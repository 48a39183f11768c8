"""Multi-view training step with soft pruning (BASELINE configs[3]).

The reference's consumer of the render path is the ADMM pruning loop
(/root/reference/pkg/src/sgsplat/prune.py:162-201, gradient_step): per view
``loss_and_grads``, then plain gradient steps with per-group rates.  This
module is the device-resident equivalent for the soft-pruning setting of
configs[3]:

  m_p = sigmoid(prim_logit), m_l = sigmoid(lobe_logit)
  L = sum_views [(1-l) L1 + l (1 - SSIM)] / n_views
      + lambda_m (11 mean(m_p) + 7 mean(m_l))        (rho_o = 11, rho_s = 7,
                                                       scene.py:20-21)

Forward + backward per view run in libsgs.so; the per-view gradients are
accumulated into one flat bucket, all-reduced over ranks (NCCL) and averaged;
the masks' gradients flow through the sigmoid.  ``grad_fn`` can be injected
(tests use the CPU oracle under gloo).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from .render import GRAD_OPACITY_FLOOR
from .sharding import GradBucket, shard_views
from .rasterizer import GRAD_FIELDS, GaussianTensors, Rasterizer


@dataclass(frozen=True)
class TrainConfig:
    lambda_ssim: float = 0.2
    lambda_mask: float = 1e-3
    lr: dict = field(default_factory=lambda: {
        "position": 1e-3, "quat": 1e-3, "log_scale": 1e-3, "opacity": 1e-2, "diffuse": 1e-2,
        "axis_raw": 1e-3, "sharpness": 1e-2, "amplitude": 1e-2, "prim_logit": 1e-1,
        "lobe_logit": 1e-1})


def _world(group) -> int:
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group)
    return 1


class SoftPruneTrainer:
    """Holds device parameters + mask logits; ``step(cams, targets)`` runs one
    data-parallel training step over this rank's share of the views."""

    def __init__(self, arrays, prim_logit, lobe_logit, cfg: TrainConfig = TrainConfig(),
                 device="cuda", group=None, grad_fn=None, streams: int = 8, comm_chunks: int = 4,
                 chunk_single_rank: bool = False):
        """``streams``: views of a step in flight at once on this many CUDA
        streams (each with its own workspace); their parameter backwards
        (K7, which add into the shared gradient bucket) run in view order on
        one more stream.  ``comm_chunks``: with more than one rank the
        gradient bucket is split into this many primitive ranges, each
        all-reduced as soon as the last view's K7 has added its rows, so the
        collective overlaps the rest of the parameter backward
        (``chunk_single_rank``: chunk on one rank too -- tests)."""
        self.device = torch.device(device)
        self.cfg = cfg
        self.group = group
        self.params = {f: torch.as_tensor(getattr(arrays, f), dtype=torch.float32,
                                          device=self.device).contiguous() for f in GRAD_FIELDS}
        self.prim_logit = torch.as_tensor(prim_logit, dtype=torch.float32, device=self.device).contiguous()
        self.lobe_logit = torch.as_tensor(lobe_logit, dtype=torch.float32, device=self.device).contiguous()
        shapes = {f: t.shape for f, t in self.params.items()}
        shapes["prim_logit"] = self.prim_logit.shape
        shapes["lobe_logit"] = self.lobe_logit.shape
        n = int(self.prim_logit.shape[0])
        self.chunks = max(1, int(comm_chunks)) if (_world(group) > 1 or chunk_single_rank) else 1
        self.bucket = GradBucket(shapes, self.device, chunks=self.chunks, n=n)
        self.grad_fn = grad_fn
        self.rast = None if grad_fn is not None else Rasterizer(device=self.device)
        self.n_streams = max(1, int(streams)) if grad_fn is None else 1
        self._streams = ([torch.cuda.Stream(self.device) for _ in range(self.n_streams)],
                         torch.cuda.Stream(self.device)) if self.n_streams > 1 else None
        # step(graph=True) without a collective captures the reduction and the
        # update too; False keeps them eager, as a multi-rank step does
        self.graph_tail = True
        self._gstep = self._graph_warm = None

    def masks(self):
        return torch.sigmoid(self.prim_logit), torch.sigmoid(self.lobe_logit)

    def gaussians(self):
        m_p, m_l = self.masks()
        if self.device.type != "cuda":  # host-logic tests with an injected grad_fn
            from types import SimpleNamespace
            return SimpleNamespace(**self.params, lobe_mask=m_l.contiguous(), prim_mask=m_p.contiguous())
        return GaussianTensors(**self.params, lobe_mask=m_l.contiguous(), prim_mask=m_p.contiguous())

    def _bucket_out(self, c: int = 0) -> dict:
        out = {f: self.bucket.chunk_view(f, c) for f in GRAD_FIELDS}
        out["prim_mask"] = self.bucket.chunk_view("prim_logit", c)
        out["lobe_mask"] = self.bucket.chunk_view("lobe_logit", c)
        return out

    def _rows(self, c: int) -> slice:
        p0, p1 = self.bucket.bounds[c]
        return slice(p0, p1)

    def _chunk_gaussians(self, g: GaussianTensors, c: int) -> GaussianTensors:
        if self.chunks == 1:
            return g
        r = self._rows(c)
        return GaussianTensors(*(getattr(g, f)[r] for f in GRAD_FIELDS), lobe_mask=g.lobe_mask[r],
                               prim_mask=g.prim_mask[r])

    def _view_grads(self, g, cam, target, overflow=None):
        """Loss of one view; its gradients are added to the bucket (mask
        gradients through the sigmoid, i.e. with respect to the logits)."""
        if self.grad_fn is not None:
            val, gr = self.grad_fn(g, cam, target)
            m_p, m_l = g.prim_mask, g.lobe_mask
            d_mp = gr.pop("prim_mask")
            d_ml = gr.pop("lobe_mask")
            gr.pop("grad2d", None)
            gr["prim_logit"] = d_mp * m_p * (1 - m_p)
            gr["lobe_logit"] = d_ml * m_l * (1 - m_l)
            self.bucket.add_(gr)
            return val
        from .loss import image_loss
        from .render import LossConfig
        frame = self.rast.forward(g, cam, check=overflow is None, grad_floor=GRAD_OPACITY_FLOOR)
        if overflow is not None:
            frame.record_overflow(overflow)
        lo, dimg, _ = image_loss(frame.img, target, LossConfig(lambda_ssim=self.cfg.lambda_ssim), grad="f32")
        grad2d = self.rast.backward_raster(g, frame, dimg)
        for c in range(self.chunks):
            self.rast.backward_params(self._chunk_gaussians(g, c), frame.cam, grad2d[self._rows(c)],
                                      mask_grads=True, out=self._bucket_out(c), accumulate=True, mask_logit=True)
        return lo[0]

    def _views_pipelined(self, g: GaussianTensors, cams, targets, mine, ovf, capture: bool = False):
        """The step's views on ``n_streams`` streams: forward, loss and raster
        backward of view j on stream j mod S; then, on the accumulation stream
        once every view's partials are in, one K7 over all the views per
        primitive chunk (sgs_preprocess_backward_views: one writer, the views
        summed in order).  Returns the summed loss (device) and one event per
        chunk, recorded on the accumulation stream when that chunk's rows are
        complete.  The current stream waits for the views' streams only, not for K7
        (``capture``: inside a CUDA-graph capture -- no chunk events, every
        stream joined back, see _capture_views)."""
        from .loss import image_loss
        from .render import LossConfig
        main = torch.cuda.current_stream(self.device)
        views, acc = self._streams
        start = torch.cuda.Event()
        start.record(main)  # bucket zeroed, masks and overflow slots ready
        acc.wait_event(start)
        cfg = LossConfig(lambda_ssim=self.cfg.lambda_ssim)
        losses = []
        chunk_done = [torch.cuda.Event() for _ in range(self.chunks)]
        gc = [self._chunk_gaussians(g, c) for c in range(self.chunks)]
        outs = [self._bucket_out(c) for c in range(self.chunks)]
        c_cams, g2ds = [], []
        for j, v in enumerate(mine):
            st = views[j % len(views)]
            st.wait_event(start)
            with torch.cuda.stream(st):
                frame = self.rast.forward(g, cams[v], check=False, grad_floor=GRAD_OPACITY_FLOOR)
                frame.record_overflow(ovf[j])
                lo, dimg, _ = image_loss(frame.img, targets[v], cfg, grad="f32")
                grad2d = self.rast.backward_raster(g, frame, dimg)
                done = torch.cuda.Event()
                done.record(st)
            acc.wait_event(done)
            grad2d.record_stream(acc)
            c_cams.append(frame.cam)
            g2ds.append(grad2d)
            if not capture:
                lo.record_stream(main)
            losses.append(lo[0])
        # K7 once for all the views (they finish their raster backwards
        # together anyway): each primitive's parameters read and its bucket
        # rows written once per 8 views, the views summed in order
        if mine:
            with torch.cuda.stream(acc):
                for c in range(self.chunks):
                    r = self._rows(c)
                    self.rast.backward_params_views(gc[c], c_cams, [t[r] for t in g2ds], mask_grads=True,
                                                    out=outs[c], accumulate=True, mask_logit=True)
                    if not capture:
                        chunk_done[c].record(acc)
        if not mine and not capture:
            for c in range(self.chunks):
                chunk_done[c].record(acc)
        # join only the streams this step used: under capture, waiting on a
        # stream that never forked from the capture stream invalidates it
        used = views[:len(mine)] if capture else views
        for st in used + ([acc] if capture else []):
            main.wait_stream(st)
        loss = torch.stack(losses).sum() if losses else torch.zeros((), dtype=torch.float64, device=self.device)
        return loss, (None if capture else chunk_done)

    def _capture_views(self, cams, targets, mine, tail=None):
        """CUDA graph of the step's device work: bucket reset, masks, every
        view's forward, loss, K6 and K7 (captured from the same streams and
        workspaces an eager step just used) and, when the step has no
        collective (``tail`` = (n_views, apply)), the reduction, penalty and
        masked update too.  A one-view step launches ~80 kernels from Python:
        replayed, its host cost is one launch and the GPU no longer waits for
        it."""
        dev = self.device
        cur = torch.cuda.current_stream(dev)
        torch.cuda.synchronize(dev)
        if getattr(self, "_cap_stream", None) is None:
            self._cap_stream = torch.cuda.Stream(dev)
        cap = self._cap_stream
        ovf = torch.zeros((max(len(mine), 1), 2), dtype=torch.int64, device=dev)
        graph = torch.cuda.CUDAGraph()
        cap.wait_stream(cur)
        loss = need = None
        with torch.cuda.graph(graph, stream=cap):
            self.bucket.zero()
            g = self.gaussians()
            ovf.zero_()
            loss_sum, _ = self._views_pipelined(g, cams, targets, mine, ovf[:len(mine)], capture=True)
            if tail is not None:
                loss, need = self._tail(g, ovf[:len(mine)], loss_sum, None, mine, tail[0], False, tail[1],
                                        capture=True)
        cur.wait_stream(cap)
        return {"graph": graph, "ovf": ovf[:len(mine)], "loss": loss_sum, "g": g, "full": tail is not None,
                "step_loss": loss, "need": need,
                "key": self._graph_key(cams, targets, mine, tail), "hint": dict(self.rast._cap_hint)}

    def _graph_key(self, cams, targets, mine, tail=None):
        from .camera import to_sgs
        cfg = (tuple(sorted(self.cfg.lr.items())), self.cfg.lambda_mask, self.cfg.lambda_ssim)
        # the graph reads the parameters and targets through these pointers:
        # replaced (not updated in place) tensors need a new capture
        ptrs = tuple(t.data_ptr() for t in self.params.values()) + (self.prim_logit.data_ptr(),
                                                                     self.lobe_logit.data_ptr())
        return (tuple(mine), tuple(bytes(to_sgs(cams[v], grad_floor=GRAD_OPACITY_FLOOR)) for v in mine),
                tuple(targets[v].data_ptr() for v in mine), tail, cfg, ptrs)

    def step(self, cams, targets, rank: int = 0, world: int = 1, apply: bool = True, sync: bool = True,
             graph: bool = False):
        """One step over all views (this rank renders its round-robin share);
        returns the global mean loss -- a float, or with ``sync=False`` a
        0-dim float64 device tensor (the step then synchronises the host only
        once, for the tile-capacity check).  ``graph``: replay the views'
        device work from a CUDA graph, captured on the first step whose
        capacities an eager step has already sized (recaptured when views,
        targets or capacities change); the reductions stay eager."""
        import torch.distributed as dist
        n_views = len(cams)
        mine = shard_views(n_views, rank, world)
        multi = dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1
        chunk_done = None
        use_graph = graph and self._streams is not None and len(mine) >= 1
        tail = None if (multi or not self.graph_tail) else (n_views, apply)  # no collective: one graph
        gs = self._gstep
        if use_graph:
            key = self._graph_key(cams, targets, mine, tail)
            if gs is not None and (gs["key"] != key or gs["hint"] != self.rast._cap_hint):
                gs = self._gstep = None
            if gs is None and self._graph_warm == key:
                gs = self._gstep = self._capture_views(cams, targets, mine, tail)
        if use_graph and gs is not None:
            gs["graph"].replay()  # bucket reset, masks, views (and the tail): one launch
            g, ovf = gs["g"], gs["ovf"]
            if gs["full"]:
                loss, need = gs["step_loss"].clone(), gs["need"]
            else:
                loss, need = self._tail(g, ovf, gs["loss"].clone(), None, mine, n_views, multi, apply)
        else:
            self.bucket.zero()
            g = self.gaussians()
            loss_sum = torch.zeros((), dtype=torch.float64, device=self.device)
            # tile-entry overflow is checked once per step (no host round trip per view)
            ovf = None if self.grad_fn is not None else torch.zeros((len(mine), 2), dtype=torch.int64,
                                                                    device=self.device)
            if self._streams is not None and len(mine) >= 1:  # one view too: K7 chunks overlap the reduction
                ls, chunk_done = self._views_pipelined(g, cams, targets, mine, ovf)
                loss_sum += ls
                if use_graph:  # an eager step sized this configuration: capture from the next one
                    self._graph_warm = self._graph_key(cams, targets, mine, tail)
            else:
                for j, v in enumerate(mine):
                    loss_sum += self._view_grads(g, cams[v], targets[v], None if ovf is None else ovf[j])
            loss, need = self._tail(g, ovf, loss_sum, chunk_done, mine, n_views, multi, apply)
        if need is not None and int(need.item()):  # the step's one host synchronisation
            o = ovf.cpu()
            self._gstep = None            # its workspaces are about to be replaced
            self._graph_warm = None
            torch.cuda.synchronize(self.device)
            for j, v in enumerate(mine):
                if o[j, 0]:
                    self.rast.grow_capacity(g, cams[v], int(o[j, 1]))
            return self.step(cams, targets, rank, world, apply, sync, graph)
        return float(loss) if sync else loss

    def _tail(self, g, ovf, loss_sum, chunk_done, mine, n_views, multi, apply, capture=False):
        """Everything after the views, enqueued before the host reads the
        overflow flag: the update is masked on the device by `ok` (no view
        outgrew its tile capacity, on any rank), so the GPU never waits for
        the host.  On overflow nothing was applied: capacities grow and the
        step is redone.  Returns (loss, need) as device tensors."""
        import torch.distributed as dist
        m_p, m_l = g.prim_mask, g.lobe_mask
        need = None
        if ovf is not None:
            need = (ovf[:, 0].max() if len(mine) else torch.zeros((), dtype=torch.int64,
                                                                   device=self.device)).reshape(1)
            if multi:  # every rank redoes together, so the collectives stay matched
                dist.all_reduce(need, op=dist.ReduceOp.MAX, group=self.group)
        ok = None if need is None else (need[0] == 0)
        # bucketed all-reduce: chunk c leaves as soon as its rows are complete,
        # while the accumulation stream still adds the later chunks
        works = []
        main = torch.cuda.current_stream(self.device) if self.device.type == "cuda" else None
        for c in range(self.chunks):
            if chunk_done is not None:
                main.wait_event(chunk_done[c])
            if multi:
                works.append(dist.all_reduce(self.bucket.chunk_flat(c), op=dist.ReduceOp.SUM, group=self.group,
                                             async_op=True))
        stats = torch.stack([loss_sum, torch.full((), float(len(mine)), dtype=torch.float64,
                                                  device=self.device)])
        if multi:
            dist.all_reduce(stats, group=self.group)
        loss = stats[0] / n_views
        lam = self.cfg.lambda_mask
        if lam:  # sparsity penalty lambda_m (11 mean m_p + 7 mean m_l), through the sigmoid
            loss = loss + lam * (11.0 * m_p.double().mean() + 7.0 * m_l.double().mean())
        for c in range(self.chunks):
            if works:
                works[c].wait()
            self.bucket.chunk_flat(c).div_(n_views)
            r = self._rows(c)
            if lam:
                mp, ml = m_p[r], m_l[r]
                self.bucket.chunk_view("prim_logit", c).add_(lam * 11.0 / m_p.numel() * mp * (1 - mp))
                self.bucket.chunk_view("lobe_logit", c).add_(lam * 7.0 / m_l.numel() * ml * (1 - ml))
            if apply:
                self._apply_chunk(c, ok)
        if self._streams is not None and not capture:
            torch.cuda.current_stream(self.device).wait_stream(self._streams[1])
        return loss, need

    def _apply_chunk(self, c: int, ok=None):
        """Plain gradient step on primitive range c (opacity kept in [0, 1],
        prune.py:185; sharpness >= 0), masked by the device bool ``ok``.  On
        the GPU one fused kernel updates every parameter class
        (sgs_admm_update, stage 2 without penalties); the mask logits follow."""
        lr = self.cfg.lr
        r = self._rows(c)
        with torch.no_grad():
            if self.device.type == "cuda":
                import ctypes as C
                from . import _ffi
                from .admm import _CLASSES, _fields
                p = {f: self.params[f][r] for f in _CLASSES}
                gr = {f: self.bucket.chunk_view(f, c) for f in _CLASSES}
                rates = _ffi.SgsAdmmRates(*(float(lr[f]) for f in _CLASSES), 1.0, 0.0, 0.0)
                okb = None if ok is None else ok.to(torch.uint8)
                L = int(p["sharpness"].shape[1]) if p["sharpness"].dim() > 1 else 0
                _ffi.call("sgs_admm_update", int(p["opacity"].numel()), L, 2, 1, C.byref(_fields(p)),
                          C.byref(_fields(gr)), gr["sharpness"].data_ptr(), None, None, None, None, C.byref(rates),
                          None if okb is None else okb.data_ptr(),
                          C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream))
            else:
                for f, t in self.params.items():
                    upd = t[r] - lr[f] * self.bucket.chunk_view(f, c)
                    t[r].copy_(upd if ok is None else torch.where(ok, upd, t[r]))
                self.params["opacity"][r].clamp_(0.0, 1.0)
                self.params["sharpness"][r].clamp_(min=0.0)
            for name, t in (("prim_logit", self.prim_logit), ("lobe_logit", self.lobe_logit)):
                upd = t[r] - lr[name] * self.bucket.chunk_view(name, c)
                t[r].copy_(upd if ok is None else torch.where(ok, upd, t[r]))

    def apply(self):
        for c in range(self.chunks):
            self._apply_chunk(c)

    def grads(self) -> dict:
        return self.bucket.as_dict()
