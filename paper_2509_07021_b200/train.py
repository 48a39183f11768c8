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


class SoftPruneTrainer:
    """Holds device parameters + mask logits; ``step(cams, targets)`` runs one
    data-parallel training step over this rank's share of the views."""

    def __init__(self, arrays, prim_logit, lobe_logit, cfg: TrainConfig = TrainConfig(),
                 device="cuda", group=None, grad_fn=None, streams: int = 4):
        """``streams``: views of a step in flight at once on this many CUDA
        streams (each with its own workspace); their parameter backwards
        (K7, which add into the shared gradient bucket) run in view order on
        one more stream."""
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
        self.bucket = GradBucket(shapes, self.device)
        self.grad_fn = grad_fn
        self.rast = None if grad_fn is not None else Rasterizer(device=self.device)
        self.n_streams = max(1, int(streams)) if grad_fn is None else 1
        self._streams = ([torch.cuda.Stream(self.device) for _ in range(self.n_streams)],
                         torch.cuda.Stream(self.device)) if self.n_streams > 1 else None

    def masks(self):
        return torch.sigmoid(self.prim_logit), torch.sigmoid(self.lobe_logit)

    def gaussians(self):
        m_p, m_l = self.masks()
        if self.device.type != "cuda":  # host-logic tests with an injected grad_fn
            from types import SimpleNamespace
            return SimpleNamespace(**self.params, lobe_mask=m_l.contiguous(), prim_mask=m_p.contiguous())
        return GaussianTensors(**self.params, lobe_mask=m_l.contiguous(), prim_mask=m_p.contiguous())

    def _bucket_out(self) -> dict:
        out = {f: self.bucket.view(f) for f in GRAD_FIELDS}
        out["prim_mask"] = self.bucket.view("prim_logit")
        out["lobe_mask"] = self.bucket.view("lobe_logit")
        return out

    def _view_grads(self, g: GaussianTensors, cam, target, overflow=None):
        """Loss of one view; its gradients are added to the bucket (mask
        gradients through the sigmoid, i.e. with respect to the logits)."""
        if self.grad_fn is not None:
            val, gr = self.grad_fn(g, cam, target)
            m_p, m_l = g.prim_mask, g.lobe_mask
            d_mp = gr.pop("prim_mask")
            d_ml = gr.pop("lobe_mask")
            gr.pop("grad2d", None)
            self.bucket.add_(gr)
            self.bucket.view("prim_logit").add_(d_mp * m_p * (1 - m_p))
            self.bucket.view("lobe_logit").add_(d_ml * m_l * (1 - m_l))
            return val
        from .render import LossConfig, loss_and_grads_device
        val, _ = loss_and_grads_device(g, cam, target, LossConfig(lambda_ssim=self.cfg.lambda_ssim),
                                       rast=self.rast, mask_grads=True, sync=False, overflow_out=overflow,
                                       grads_out=self._bucket_out(), accumulate=True, mask_logit=True)
        return val

    def _views_pipelined(self, g: GaussianTensors, cams, targets, mine, ovf):
        """The step's views on ``n_streams`` streams: forward, loss and raster
        backward of view j on stream j mod S, then its K7 into the bucket on
        the accumulation stream in view order (one writer: the bucket update
        is a plain read-modify-write).  Returns the summed loss (device)."""
        from .loss import image_loss
        from .render import LossConfig
        main = torch.cuda.current_stream(self.device)
        views, acc = self._streams
        start = torch.cuda.Event()
        start.record(main)  # bucket zeroed, masks and overflow slots ready
        acc.wait_event(start)
        cfg = LossConfig(lambda_ssim=self.cfg.lambda_ssim)
        out = self._bucket_out()
        losses = []
        for j, v in enumerate(mine):
            st = views[j % len(views)]
            st.wait_event(start)
            with torch.cuda.stream(st):
                frame = self.rast.forward(g, cams[v], check=False)
                frame.record_overflow(ovf[j])
                lo, dimg, _ = image_loss(frame.img, targets[v], cfg, grad="f32")
                grad2d = self.rast.backward_raster(g, frame, dimg)
                done = torch.cuda.Event()
                done.record(st)
            acc.wait_event(done)
            grad2d.record_stream(acc)
            with torch.cuda.stream(acc):
                self.rast.backward_params(g, frame.cam, grad2d, mask_grads=True, out=out, accumulate=True,
                                          mask_logit=True)
            lo.record_stream(main)
            losses.append(lo[0])
        for st in views + [acc]:
            main.wait_stream(st)
        return torch.stack(losses).sum() if losses else torch.zeros((), dtype=torch.float64, device=self.device)

    def step(self, cams, targets, rank: int = 0, world: int = 1, apply: bool = True) -> float:
        """One step over all views (this rank renders its round-robin share);
        returns the global mean loss."""
        n_views = len(cams)
        mine = shard_views(n_views, rank, world)
        self.bucket.zero()
        g = self.gaussians()
        m_p, m_l = g.prim_mask, g.lobe_mask
        loss_sum = torch.zeros((), dtype=torch.float64, device=self.device)
        # tile-entry overflow is checked once per step (no host round trip per view)
        ovf = None if self.grad_fn is not None else torch.zeros((len(mine), 2), dtype=torch.int64,
                                                                device=self.device)
        if self._streams is not None and len(mine) > 1:
            loss_sum += self._views_pipelined(g, cams, targets, mine, ovf)
        else:
            for j, v in enumerate(mine):
                loss_sum += self._view_grads(g, cams[v], targets[v], None if ovf is None else ovf[j])
        if ovf is not None:
            # some view outgrew its capacity: size it and redo the step (on every
            # rank together, so the collectives below stay matched)
            import torch.distributed as dist
            need = (ovf[:, 0].max() if len(mine) else torch.zeros((), dtype=torch.int64,
                                                                   device=self.device)).reshape(1)
            if dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1:
                dist.all_reduce(need, op=dist.ReduceOp.MAX, group=self.group)
            if int(need.item()):
                o = ovf.cpu()
                for j, v in enumerate(mine):
                    if o[j, 0]:
                        self.rast.grow_capacity(g, cams[v], int(o[j, 1]))
                return self.step(cams, targets, rank, world, apply)
        # all-reduce the summed view gradients and the loss, then average
        stats = torch.stack([loss_sum, torch.tensor(float(len(mine)), dtype=torch.float64,
                                                    device=self.device)])
        self.bucket.allreduce_(self.group, average_over=n_views)
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.all_reduce(stats, group=self.group)
        loss = float(stats[0]) / n_views
        # sparsity penalty lambda_m (11 mean m_p + 7 mean m_l), through the sigmoid
        lam = self.cfg.lambda_mask
        if lam:
            loss += lam * (11.0 * float(m_p.mean()) + 7.0 * float(m_l.mean()))
            self.bucket.view("prim_logit").add_(lam * 11.0 / m_p.numel() * m_p * (1 - m_p))
            self.bucket.view("lobe_logit").add_(lam * 7.0 / m_l.numel() * m_l * (1 - m_l))
        if apply:
            self.apply()
        return loss

    def apply(self):
        lr = self.cfg.lr
        with torch.no_grad():
            for f, t in self.params.items():
                t.sub_(lr[f] * self.bucket.view(f))
            self.params["opacity"].clamp_(0.0, 1.0)      # prune.py:185 keeps opacity in [0, 1]
            self.params["sharpness"].clamp_(min=0.0)
            self.prim_logit.sub_(lr["prim_logit"] * self.bucket.view("prim_logit"))
            self.lobe_logit.sub_(lr["lobe_logit"] * self.bucket.view("lobe_logit"))

    def grads(self) -> dict:
        return self.bucket.as_dict()
