"""Device-resident ADMM sparsification step.

Restates the reference's budget-constrained pruning loop
(/root/reference/pkg/src/sgsplat/prune.py:162-299) with every array on the
GPU:

  gradient_step   prune.py:162-201  penalized descent; with delta != 0 the
                                    sharpness gradient is taken after the
                                    opacity update (second backward pass)
  prox_project    prune.py:216-271  factorized top-k keep (magnitude /
                                    importance / dynamic-range scores),
                                    ties keep the lower index
  dual_update     prune.py:274-278  duals += primal - proxy
  run_state       prune.py:312-354  schedule, proximal events, final zeroing

The renders, losses and gradients run in libsgs.so (loss_and_grads_device);
the top-k keep masks run in libsgs.so's stable radix sort (sgs_topk_mask);
each stage of the penalized update is one fused kernel (sgs_admm_update);
the proximal event's bookkeeping uses PyTorch tensor ops on the device.  Parameters
are float32 (the renderer's precision); scores are float64.  Configs are
duck-typed: the reference's PrunerConfig / GroupRates work as well as the
mirrors below.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _ffi
from .rasterizer import GRAD_FIELDS, GaussianTensors, Rasterizer
from .render import LossConfig, loss_and_grads_device

BASE_PARAMS_PER_PRIMITIVE = 11   # scene.py:20 (rho_o)
PARAMS_PER_LOBE = 7              # scene.py:21 (rho_s)
_OPACITY_OPERATORS = ("magnitude", "importance")
_SHARPNESS_OPERATORS = ("sharpness", "range")


class ConfigError(ValueError):
    """Invalid pruning configuration (scene.py ConfigError)."""


class NumericalFailure(RuntimeError):
    """Non-finite gradient (scene.py NumericalFailure); ``index`` = primitive."""

    def __init__(self, msg, index=None):
        super().__init__(msg)
        self.index = index


@dataclass(frozen=True)
class GroupRates:
    """Per-parameter-group learning-rate multipliers (prune.py:29-40)."""

    position: float = 1e-3
    quat: float = 1e-3
    log_scale: float = 2e-3
    opacity: float = 2.5e-2
    diffuse: float = 5e-3
    axis_raw: float = 2e-3
    sharpness: float = 2.5e-2
    amplitude: float = 5e-3


@dataclass(frozen=True)
class PrunerConfig:
    """Budget, penalties and schedule (prune.py:43-117)."""

    kappa: int
    kappa_o: int
    kappa_s: int
    delta: float = 5e-3
    eta: float = 1.0
    iters: int = 1000
    prox_every: int | None = 50
    opacity_operator: str = "magnitude"
    sharpness_operator: str = "sharpness"
    seed: int = 0
    group_rates: GroupRates = field(default_factory=GroupRates)
    loss_cfg: LossConfig = field(default_factory=LossConfig)
    background: tuple = (0.0, 0.0, 0.0)

    def __post_init__(self):
        if self.prox_every is not None and self.prox_every < 1:
            raise ConfigError("prox_every must be >= 1 (or None to disable)")
        if self.opacity_operator not in _OPACITY_OPERATORS:
            raise ConfigError(f"unknown opacity operator {self.opacity_operator!r}")
        if self.sharpness_operator not in _SHARPNESS_OPERATORS:
            raise ConfigError(f"unknown sharpness operator {self.sharpness_operator!r}")
        if self.kappa_o < 0 or self.kappa_s < 0:
            raise ConfigError("keep counts must be non-negative")
        if BASE_PARAMS_PER_PRIMITIVE * self.kappa_o + PARAMS_PER_LOBE * self.kappa_s > self.kappa:
            raise ConfigError(f"split kappa_o={self.kappa_o}, kappa_s={self.kappa_s} "
                              f"exceeds budget kappa={self.kappa}")

    @property
    def delta_o(self) -> float:
        return self.delta * BASE_PARAMS_PER_PRIMITIVE

    @property
    def delta_s(self) -> float:
        return self.delta * PARAMS_PER_LOBE


def _delta_o(cfg) -> float:
    return float(cfg.delta) * BASE_PARAMS_PER_PRIMITIVE


def _delta_s(cfg) -> float:
    return float(cfg.delta) * PARAMS_PER_LOBE


def _dev() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2509_07021_b200.admm needs a CUDA device; there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _t(a, dtype=torch.float32) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=_dev(), dtype=dtype).contiguous()
    return torch.as_tensor(np.asarray(a), dtype=dtype, device=_dev()).contiguous()


# ------------------------------------------------------------------ top-k
def topk_mask(scores: torch.Tensor, k: int) -> torch.Tensor:
    """Boolean keep mask of the k largest scores, ties keep the lower index
    (prune.py:204-213) -- libsgs.so's stable radix sort on float64 keys."""
    s = _t(scores, torch.float64).reshape(-1)
    n = s.numel()
    keep = torch.zeros(n, dtype=torch.uint8, device=s.device)
    if k <= 0 or n == 0:
        return keep.bool()
    if k >= n:
        return torch.ones(n, dtype=torch.bool, device=s.device)
    nb = C.c_uint64()
    _ffi.call("sgs_topk_mask_temp_size", n, C.byref(nb))
    tmp = torch.empty(int(nb.value), dtype=torch.uint8, device=s.device)
    _ffi.call("sgs_topk_mask", s.data_ptr(), n, int(k), keep.data_ptr(), tmp.data_ptr(), tmp.numel(),
              C.c_void_p(torch.cuda.current_stream(s.device).cuda_stream))
    return keep.bool()


def dynamic_range(sharpness: torch.Tensor, amplitude: torch.Tensor) -> torch.Tensor:
    """||a|| (1 - exp(-2 s)) per lobe (sg.py:183-187, dynamic_range_many), float64."""
    s = _t(sharpness, torch.float64)
    a = _t(amplitude, torch.float64).reshape(s.shape + (3,))
    return torch.linalg.vector_norm(a, dim=-1) * -torch.expm1(-2.0 * s)


def prox_project(o_in, s_in, cfg, importance=None, range_sharpness=None, range_amplitude=None,
                 slot_mask=None):
    """Project (opacity, sharpness) onto the factorized budget set
    (prune.py:216-271).  Returns device float32 tensors shaped like the inputs."""
    o = _t(o_in)
    s = _t(s_in)
    s_flat = s.reshape(-1)
    if cfg.kappa_o > o.numel():
        raise ConfigError(f"kappa_o={cfg.kappa_o} exceeds {o.numel()} primitives")
    n_slots = s_flat.numel() if slot_mask is None else int(_t(slot_mask, torch.bool).sum())
    if cfg.kappa_s > n_slots:
        raise ConfigError(f"kappa_s={cfg.kappa_s} exceeds {n_slots} lobe slots")
    if cfg.opacity_operator == "importance":
        if importance is None:
            raise ConfigError("importance scores required for the importance operator")
        o_scores = _t(importance, torch.float64)
        if tuple(o_scores.shape) != tuple(o.shape):
            raise ConfigError("importance shape does not match opacity")
    else:
        o_scores = o.to(torch.float64).abs()
    if cfg.sharpness_operator == "range":
        if range_sharpness is None or range_amplitude is None:
            raise ConfigError("range operator needs current sharpness and amplitudes")
        s_scores = dynamic_range(_t(range_sharpness).reshape(-1),
                                 _t(range_amplitude).reshape(-1, 3))
    else:
        s_scores = s_flat.to(torch.float64).abs()
    if slot_mask is not None:
        s_scores = torch.where(_t(slot_mask, torch.bool).reshape(-1), s_scores,
                               torch.full_like(s_scores, -np.inf))
    o_keep = topk_mask(o_scores, cfg.kappa_o)
    s_keep = topk_mask(s_scores, cfg.kappa_s)
    return (torch.where(o_keep.reshape(o.shape), o, torch.zeros_like(o)),
            torch.where(s_keep, s_flat, torch.zeros_like(s_flat)).reshape(s.shape))


# ------------------------------------------------------------------ state
class DevicePrunerState:
    """Primal parameters (float32 device tensors, SceneParams layout) plus the
    proxy and dual vectors (prune.py:119-133)."""

    def __init__(self, params: dict, lobe_mask: torch.Tensor):
        self.params = params
        self.lobe_mask = lobe_mask  # float 0/1 (N, L)
        self.proxy_o = params["opacity"].clone()
        self.proxy_s = params["sharpness"].clone()
        self.dual_o = torch.zeros_like(params["opacity"])
        self.dual_s = torch.zeros_like(params["sharpness"])
        self.iteration = 0

    @staticmethod
    def init(p) -> "DevicePrunerState":
        """From any object with SceneParams attributes (numpy or torch)."""
        params = {f: _t(getattr(p, f)) for f in GRAD_FIELDS}
        lm = getattr(p, "lobe_mask", None)
        lm = torch.ones_like(params["sharpness"]) if lm is None else _t(lm)
        return DevicePrunerState(params, lm)

    def gaussians(self) -> GaussianTensors:
        return GaussianTensors(**self.params, lobe_mask=self.lobe_mask)

    def to_numpy(self) -> dict:
        return {f: t.detach().to(torch.float64).cpu().numpy() for f, t in self.params.items()}


class _Failure:
    """A non-finite gradient found on the device, reported at the next host
    synchronisation (prune.py:151-159 raises at once; the device loop defers
    the check so a step costs no host round trip).  From the failing step on
    every update is masked off, so the state is the one the reference leaves
    behind when it raises."""

    def __init__(self, device):
        self.flag = torch.zeros((), dtype=torch.bool, device=device)      # any failure so far
        self.index = torch.zeros((), dtype=torch.int64, device=device)    # first bad primitive
        self.field = torch.zeros((), dtype=torch.int64, device=device)    # its first bad class
        self.iteration = torch.zeros((), dtype=torch.int64, device=device)

    def observe(self, grads: dict, n: int, iteration: int) -> torch.Tensor:
        """Record the step's failure (if it is the first); returns the device
        bool 'this step may update'."""
        rows = torch.stack([~torch.isfinite(grads[f].reshape(n, -1)).all(dim=1) for f in GRAD_FIELDS])
        bad_row = rows.any(dim=0)
        bad = bad_row.any()
        i = torch.argmax(bad_row.to(torch.int8))                  # first bad primitive
        code = torch.argmax(rows[:, i].to(torch.int8))            # first bad class there
        new = bad & ~self.flag
        self.index = torch.where(new, i, self.index)
        self.field = torch.where(new, code, self.field)
        self.iteration = torch.where(new, torch.full_like(self.iteration, iteration), self.iteration)
        self.flag = self.flag | bad
        return ~self.flag

    def raise_if_failed(self, state=None) -> None:
        if bool(self.flag):
            i, f = int(self.index), GRAD_FIELDS[int(self.field)]
            if state is not None:
                state.iteration = int(self.iteration)
            raise NumericalFailure(f"non-finite gradient in {f} at primitive {i}", index=i)


def _failure(state: DevicePrunerState) -> _Failure:
    f = getattr(state, "_failure", None)
    if f is None:
        f = _Failure(state.params["opacity"].device)
        state._failure = f
    return f


_CLASSES = ("position", "quat", "log_scale", "opacity", "diffuse", "axis_raw", "sharpness", "amplitude")


def _fields(d: dict) -> _ffi.SgsAdmmFields:
    f = _ffi.SgsAdmmFields()
    for k in _CLASSES:
        t = d[k]
        if t.dtype != torch.float32 or not t.is_contiguous():
            raise ValueError(f"{k} must be a contiguous float32 tensor")
        setattr(f, k, t.data_ptr())
    return f


def _update(state, stage: int, g1: dict, g_sharp, cfg, ok: torch.Tensor, update_o: bool, delta_s: float):
    """One fused device pass of the step (sgs_admm_update, select.cu)."""
    r = cfg.group_rates
    rates = _ffi.SgsAdmmRates(*(float(getattr(r, k)) for k in _CLASSES), float(cfg.eta),
                              float(_delta_o(cfg)), float(delta_s))
    p = state.params
    okb = ok.to(torch.uint8)
    ptr = lambda t: None if t is None else t.data_ptr()  # noqa: E731
    _ffi.call("sgs_admm_update", int(p["opacity"].numel()), int(p["sharpness"].shape[1]) if p["sharpness"].dim() > 1
              else 0, int(stage), int(update_o), C.byref(_fields(p)), C.byref(_fields(g1)), ptr(g_sharp),
              ptr(state.proxy_o), ptr(state.dual_o), ptr(state.proxy_s), ptr(state.dual_s), C.byref(rates),
              okb.data_ptr(), C.c_void_p(torch.cuda.current_stream(p["opacity"].device).cuda_stream))


def gradient_step(state: DevicePrunerState, view, cfg, rast: Rasterizer | None = None, sync: bool = True,
                  deterministic: bool = True):
    """One penalized descent step on one view; returns the data loss
    (prune.py:162-201, same update order).

    No host synchronisation with ``sync=False``: the loss is returned as a
    0-dim float64 device tensor and a non-finite gradient is reported at the
    next synchronisation (run_state's trace rows), with the state as the
    reference leaves it.  ``deterministic``: bitwise-reproducible gradient
    sums (Rasterizer.backward), so repeated runs take identical steps."""
    cam, target = view
    tgt = _t(target)
    g = state.gaussians()
    n = g.n
    fail = _failure(state)
    loss_val, g1 = loss_and_grads_device(g, cam, tgt, cfg.loss_cfg, cfg.background, rast=rast,
                                         sync=False, deterministic=deterministic)
    ok = fail.observe(g1, n, state.iteration)
    with torch.no_grad():
        if cfg.delta == 0.0:
            _update(state, 2, g1, g1["sharpness"], cfg, ok, update_o=True, delta_s=0.0)
        else:
            _update(state, 1, g1, None, cfg, ok, update_o=False, delta_s=0.0)
            _, g2 = loss_and_grads_device(g, cam, tgt, cfg.loss_cfg, cfg.background, rast=rast,
                                          sync=False, deterministic=deterministic)
            ok = fail.observe(g2, n, state.iteration)
            _update(state, 2, g1, g2["sharpness"], cfg, ok, update_o=False, delta_s=_delta_s(cfg))
    state.iteration += 1
    if sync:
        fail.raise_if_failed(state)
        return float(loss_val)
    return loss_val


def dual_update(state: DevicePrunerState) -> DevicePrunerState:
    """Advance the multipliers by the primal-proxy residual (prune.py:274-278)."""
    with torch.no_grad():
        state.dual_o += state.params["opacity"] - state.proxy_o
        state.dual_s += state.params["sharpness"] - state.proxy_s
    return state


def _prox_inputs(state: DevicePrunerState, cfg, views, rast: Rasterizer):
    """Importance scores (prune.py:281-290 -> render.py:416-428): every view's
    composited weights added as exact fixed point, then float64 -- the same
    bits whatever order the views' tiles finish in."""
    if cfg.opacity_operator != "importance":
        return None
    if not views:
        raise ConfigError("importance operator needs training views")
    g = state.gaussians()
    fx = torch.zeros(g.n, dtype=torch.int64, device=g.device)
    bg = tuple(float(v) for v in np.asarray(cfg.background, dtype=np.float64).reshape(3))
    for cam, _ in views:
        rast.forward(g, cam, bg, weight_fx=fx, track=False)
    return fx.to(torch.float64) * 2.0 ** -_ffi.WEIGHT_FRAC_BITS


def _proximal_event(state: DevicePrunerState, cfg, importance):
    p = state.params
    proxy_o, proxy_s = prox_project(p["opacity"] + state.dual_o, p["sharpness"] + state.dual_s, cfg,
                                    importance=importance, range_sharpness=p["sharpness"],
                                    range_amplitude=p["amplitude"], slot_mask=state.lobe_mask > 0)
    state.proxy_o, state.proxy_s = proxy_o, proxy_s
    active_o = int(torch.count_nonzero(proxy_o))
    active_s = int(torch.count_nonzero(proxy_s))
    units = BASE_PARAMS_PER_PRIMITIVE * active_o + PARAMS_PER_LOBE * active_s
    assert units <= cfg.kappa, "budget violated by the proximal projection"
    return active_o, active_s, units


@dataclass
class TraceRow:
    iteration: int
    loss: float
    residual_o: float
    residual_s: float
    active_primitives: int
    active_lobes: int
    budget_units: int


def run_state(state: DevicePrunerState, views, cfg, rast: Rasterizer | None = None,
              deterministic: bool = True) -> list[TraceRow]:
    """The full schedule (prune.py:312-354): view order from
    default_rng(seed) permutations, a proximal event + dual update every
    prox_every iterations, a terminal projection, then zeroing of primal
    entries outside the kept support.  The gradient steps between proximal
    events run without host synchronisation; ``deterministic`` (default)
    makes the whole run bitwise reproducible."""
    if not views:
        raise ConfigError("need at least one training view")
    rast = rast or Rasterizer(device=_dev())
    rng = np.random.default_rng(cfg.seed)
    p = state.params
    trace: list[TraceRow] = []
    order = rng.permutation(len(views))
    pos = 0
    loss_val = float("nan")

    fail = _failure(state)

    def record(iteration, active_o, active_s, units):
        fail.raise_if_failed(state)
        trace.append(TraceRow(
            iteration=iteration, loss=float(loss_val),
            residual_o=float(torch.linalg.vector_norm((p["opacity"] - state.proxy_o).double())),
            residual_s=float(torch.linalg.vector_norm((p["sharpness"] - state.proxy_s).double())),
            active_primitives=active_o, active_lobes=active_s, budget_units=units))

    ended_with_event = False
    for k in range(cfg.iters):
        if pos == len(order):
            order = rng.permutation(len(views))
            pos = 0
        loss_val = gradient_step(state, views[order[pos]], cfg, rast, sync=False, deterministic=deterministic)
        pos += 1
        ended_with_event = False
        if cfg.prox_every is not None and (k + 1) % cfg.prox_every == 0:
            importance = _prox_inputs(state, cfg, views, rast)
            record(k + 1, *_proximal_event(state, cfg, importance))
            dual_update(state)
            ended_with_event = True
    if cfg.prox_every is not None:
        if not ended_with_event:
            importance = _prox_inputs(state, cfg, views, rast)
            record(cfg.iters, *_proximal_event(state, cfg, importance))
        with torch.no_grad():
            p["opacity"].copy_(torch.where(state.proxy_o != 0.0, p["opacity"], torch.zeros_like(p["opacity"])))
            p["sharpness"].copy_(torch.where(state.proxy_s != 0.0, p["sharpness"],
                                             torch.zeros_like(p["sharpness"])))
    fail.raise_if_failed(state)
    return trace
