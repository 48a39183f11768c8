"""TEST INFRASTRUCTURE ONLY -- float64 NumPy restatement of the reference
renderer's algorithm (dense: every visible primitive against every pixel,
one global stable depth order, no tiles, no spatial cutoff).

Follows /root/reference/pkg/src/sgsplat/render.py:
  projection / EWA / SG color   _prepare           render.py:259-317
  dense front-to-back blend     _chunk_blend       render.py:355-390
  image + importance            _render_params     render.py:393-408
  L1 + SSIM and d/dimg          loss, _ssim_grad   render.py:435-509
  analytic backward             _backward_from_blend render.py:516-637
plus the soft masks of this build: float lobe_mask multiplies each lobe,
prim_mask multiplies opacity; their gradients dL/dm_p = o dL/do_eff and
dL/dm_l = (dL/dc_pre . a_l) e_l.

Pinned against fixtures produced by the reference itself
(tests/golden/make_golden.py -> tests/golden/*.npz; tests/test_oracle.py).
Used by tests/ and by bench.py's CPU baseline (``--impl reference`` and the
``cpu_baseline`` key); never by the product path.
"""

from __future__ import annotations

import numpy as np
from scipy.ndimage import correlate1d

ALPHA_MAX = 0.99
T_CUTOFF = 1e-4
LOWPASS = 0.3


def _f64(a):
    return np.asarray(a, dtype=np.float64)


def rotation_from_quat(q):
    """(..., 4) unit quaternions (w, x, y, z) -> (..., 3, 3)."""
    w, x, y, z = np.moveaxis(q, -1, 0)
    out = np.empty(q.shape[:-1] + (3, 3))
    out[..., 0, 0] = 1 - 2 * (y * y + z * z)
    out[..., 0, 1] = 2 * (x * y - w * z)
    out[..., 0, 2] = 2 * (x * z + w * y)
    out[..., 1, 0] = 2 * (x * y + w * z)
    out[..., 1, 1] = 1 - 2 * (x * x + z * z)
    out[..., 1, 2] = 2 * (y * z - w * x)
    out[..., 2, 0] = 2 * (x * z - w * y)
    out[..., 2, 1] = 2 * (y * z + w * x)
    out[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return out


class Projection:
    """Visible primitives in stable front-to-back order, with what the
    backward pass needs."""


def project(p, cam, lowpass=LOWPASS):
    Wm = _f64(cam.rotation).reshape(3, 3)
    tvec = _f64(cam.translation).reshape(3)
    pos = _f64(p.position)
    pc_all = pos @ Wm.T + tvec          # exactly the reference's expression (render.py:262)
    keep = np.flatnonzero(pc_all[:, 2] > getattr(cam, "near", 0.1))
    if keep.size == 0:
        return None
    pc = pc_all[keep]
    order = np.argsort(pc[:, 2], kind="stable")
    sel = keep[order]
    pc = pc[order]
    pr = Projection()
    pr.idx = sel
    pr.pc = pc
    x, y, z = pc.T
    pr.mean = np.stack([cam.fx * x / z + cam.cx, cam.fy * y / z + cam.cy], axis=1)
    q = _f64(p.quat)[sel]
    pr.qn = np.linalg.norm(q, axis=1)
    pr.qh = q / pr.qn[:, None]
    pr.R = rotation_from_quat(pr.qh)
    pr.D = np.exp(2.0 * _f64(p.log_scale)[sel])
    pr.Sigma = (pr.R * pr.D[:, None, :]) @ np.swapaxes(pr.R, 1, 2)
    J = np.zeros((sel.size, 2, 3))
    J[:, 0, 0] = cam.fx / z
    J[:, 0, 2] = -cam.fx * x / (z * z)
    J[:, 1, 1] = cam.fy / z
    J[:, 1, 2] = -cam.fy * y / (z * z)
    pr.M = J @ Wm
    cov = pr.M @ pr.Sigma @ np.swapaxes(pr.M, 1, 2)
    cov[:, 0, 0] += lowpass
    cov[:, 1, 1] += lowpass
    pr.cov = cov
    det = cov[:, 0, 0] * cov[:, 1, 1] - cov[:, 0, 1] * cov[:, 1, 0]
    pr.conic = np.stack([np.stack([cov[:, 1, 1], -cov[:, 0, 1]], -1),
                         np.stack([-cov[:, 1, 0], cov[:, 0, 0]], -1)], 1) / det[:, None, None]
    center = -Wm.T @ tvec
    d = pos[sel] - center
    pr.rd = np.linalg.norm(d, axis=1)
    pr.v = d / pr.rd[:, None]
    u = _f64(p.axis_raw)[sel]
    pr.un = np.linalg.norm(u, axis=2)
    pr.mu = u / pr.un[..., None]
    pr.dot = np.einsum("nlk,nk->nl", pr.mu, pr.v)
    pr.sharp = _f64(p.sharpness)[sel]
    pr.e = np.exp(pr.sharp * (pr.dot - 1.0))
    pr.lm = _f64(p.lobe_mask)[sel]
    pr.amp = _f64(p.amplitude)[sel]
    pr.c_pre = _f64(p.diffuse)[sel] + np.einsum("nl,nlc->nc", pr.e * pr.lm, pr.amp)
    pr.color = np.maximum(pr.c_pre, 0.0)
    pm = getattr(p, "prim_mask", None)
    pr.pm = np.ones(sel.size) if pm is None else _f64(pm)[sel]
    pr.op_raw = _f64(p.opacity)[sel]
    pr.op = pr.op_raw * pr.pm
    return pr


def _pixels(cam):
    cols, rows = np.meshgrid(np.arange(cam.width) + 0.5, np.arange(cam.height) + 0.5)
    return cols.ravel(), rows.ravel()


def _blend_block(pr, px, py):
    """Dense blend state for one block of pixels, arrays (V, B)."""
    dx = px[None, :] - pr.mean[:, :1]
    dy = py[None, :] - pr.mean[:, 1:]
    c00 = pr.conic[:, 0, 0][:, None]
    c01 = pr.conic[:, 0, 1][:, None]
    c11 = pr.conic[:, 1, 1][:, None]
    G = np.exp(-0.5 * (c00 * dx * dx + 2.0 * c01 * dx * dy + c11 * dy * dy))
    a = pr.op[:, None] * G
    one_minus = 1.0 - np.minimum(a, ALPHA_MAX)
    t_after = np.cumprod(one_minus, axis=0)
    t_before = np.vstack([np.ones((1, px.size)), t_after[:-1]])
    kept = t_after >= T_CUTOFF
    w = (1.0 - one_minus) * t_before * kept
    t_bg = np.where(kept, t_after, 1.0).min(axis=0)
    return dict(dx=dx, dy=dy, G=G, a=a, om=one_minus, tb=t_before, kept=kept, w=w, tbg=t_bg)


def render(p, cam, background=(0.0, 0.0, 0.0), weight_sums=None, block=1024):
    """Dense reference render: (H, W, 3) float64.  ``weight_sums`` (N) is
    accumulated in place with each primitive's composited weights."""
    bg = _f64(background).reshape(3)
    out = np.empty((cam.height * cam.width, 3))
    pr = project(p, cam)
    if pr is None:
        out[:] = bg
        return out.reshape(cam.height, cam.width, 3)
    px, py = _pixels(cam)
    for s in range(0, px.size, block):
        b = _blend_block(pr, px[s:s + block], py[s:s + block])
        out[s:s + block] = b["w"].T @ pr.color + b["tbg"][:, None] * bg
        if weight_sums is not None:
            np.add.at(weight_sums, pr.idx, b["w"].sum(axis=1))
    return out.reshape(cam.height, cam.width, 3)


# ---------------------------------------------------------------- loss
def gauss_window(n=11, sigma=1.5):
    t = np.arange(n) - (n - 1) / 2.0
    g = np.exp(-0.5 * (t / sigma) ** 2)
    return g / g.sum()


def _blur(x, k):
    return correlate1d(correlate1d(x, k, axis=0, mode="constant"), k, axis=1, mode="constant")


def loss_and_dimg(img, target, lambda_ssim=0.2, window=11, sigma=1.5, c1=0.01 ** 2, c2=0.03 ** 2):
    """(1-l) L1 + l (1 - mean SSIM) and its exact gradient w.r.t. img."""
    img = _f64(img)
    target = _f64(target)
    if img.shape != target.shape:
        raise ValueError(f"image shape {img.shape} != target {target.shape}")
    diff = img - target
    val = (1.0 - lambda_ssim) * np.abs(diff).mean()
    grad = (1.0 - lambda_ssim) * np.sign(diff) / diff.size
    if lambda_ssim == 0.0:
        return float(val), grad
    k = gauss_window(window, sigma)
    ssim_sum = 0.0
    dS = np.empty_like(img)
    for c in range(img.shape[-1]):
        x, y = img[..., c], target[..., c]
        mx, my = _blur(x, k), _blur(y, k)
        vx = _blur(x * x, k) - mx * mx
        vy = _blur(y * y, k) - my * my
        vxy = _blur(x * y, k) - mx * my
        A1, A2 = 2 * mx * my + c1, 2 * vxy + c2
        B1, B2 = mx * mx + my * my + c1, vx + vy + c2
        s = A1 * A2 / (B1 * B2)
        ssim_sum += s.sum()
        # dS/dmx, dS/dE[x^2], dS/dE[xy] at each window, then adjoint blur
        inv = 1.0 / (B1 * B2)
        d_A1, d_A2 = A2 * inv, A1 * inv
        d_B1, d_B2 = -s / B1, -s / B2
        g_mx = 2 * my * d_A1 - 2 * my * d_A2 + 2 * mx * d_B1 - 2 * mx * d_B2
        g_ex2 = d_B2
        g_exy = 2 * d_A2
        dS[..., c] = _blur(g_mx, k) + 2 * x * _blur(g_ex2, k) + y * _blur(g_exy, k)
    ssim_mean = ssim_sum / img.size
    val += lambda_ssim * (1.0 - ssim_mean)
    grad = grad - lambda_ssim * dS / img.size
    return float(val), grad


# ---------------------------------------------------------------- backward
def _drot(qh):
    """d R / d qhat : (V, 4, 3, 3)."""
    w, x, y, z = qh.T
    o = np.zeros_like(w)
    rows = [
        [[o, -z, y], [z, o, -x], [-y, x, o]],
        [[o, y, z], [y, -2 * x, -w], [z, w, -2 * x]],
        [[-2 * y, x, w], [x, o, z], [-w, z, -2 * y]],
        [[-2 * z, -w, x], [w, -2 * z, y], [x, y, o]],
    ]
    return 2.0 * np.moveaxis(np.array(rows), -1, 0)


def backward(p, cam, pr, dimg, background=(0.0, 0.0, 0.0), block=1024):
    """Analytic dL/dparams for dL/dimg (H, W, 3); dense, float64.  Returns a
    dict shaped like the parameters plus 'lobe_mask' and 'prim_mask'."""
    n, L = _f64(p.position).shape[0], _f64(p.axis_raw).shape[1]
    out = {"position": np.zeros((n, 3)), "quat": np.zeros((n, 4)), "log_scale": np.zeros((n, 3)),
           "opacity": np.zeros(n), "diffuse": np.zeros((n, 3)), "axis_raw": np.zeros((n, L, 3)),
           "sharpness": np.zeros((n, L)), "amplitude": np.zeros((n, L, 3)),
           "lobe_mask": np.zeros((n, L)), "prim_mask": np.zeros(n)}
    if pr is None:
        return out
    bg = _f64(background).reshape(3)
    g_all = _f64(dimg).reshape(-1, 3)
    px, py = _pixels(cam)
    acc = _backward_pixels(pr, g_all, px, py, bg, block)
    _backward_chain(p, cam, pr, acc, out)
    return out


def _backward_pixels(pr, g_all, px, py, bg, block=1024):
    """Per-primitive image-space partials (d colour, d o_eff, d mean, d conic)
    accumulated over the given pixels (render.py:535-573)."""
    V = pr.idx.size
    d_col = np.zeros((V, 3))
    d_oe = np.zeros(V)
    d_mean = np.zeros((V, 2))
    d_con = np.zeros((V, 2, 2))
    for s in range(0, px.size, block):
        b = _blend_block(pr, px[s:s + block], py[s:s + block])
        g = g_all[s:s + block]
        cg = pr.color @ g.T
        contrib = b["w"] * cg
        suffix = np.cumsum(contrib[::-1], axis=0)[::-1] - contrib
        suffix += b["tbg"][None, :] * (g @ bg)[None, :]
        dal = (b["tb"] * cg - suffix / b["om"]) * b["kept"] * (b["a"] < ALPHA_MAX)
        d_col += b["w"] @ g
        d_oe += (dal * b["G"]).sum(axis=1)
        dq = -0.5 * pr.op[:, None] * b["G"] * dal
        cdx = pr.conic[:, 0, 0][:, None] * b["dx"] + pr.conic[:, 0, 1][:, None] * b["dy"]
        cdy = pr.conic[:, 1, 0][:, None] * b["dx"] + pr.conic[:, 1, 1][:, None] * b["dy"]
        d_mean[:, 0] -= 2.0 * (dq * cdx).sum(axis=1)
        d_mean[:, 1] -= 2.0 * (dq * cdy).sum(axis=1)
        d_con[:, 0, 0] += (dq * b["dx"] ** 2).sum(axis=1)
        xy = (dq * b["dx"] * b["dy"]).sum(axis=1)
        d_con[:, 0, 1] += xy
        d_con[:, 1, 0] += xy
        d_con[:, 1, 1] += (dq * b["dy"] ** 2).sum(axis=1)
    return d_col, d_oe, d_mean, d_con


def _backward_chain(p, cam, pr, acc, out):
    """Chain rule from the image-space partials to every parameter class
    (render.py:575-637), scattered into ``out``."""
    d_col, d_oe, d_mean, d_con = acc
    Wm = _f64(cam.rotation).reshape(3, 3)
    d_cov = -pr.conic @ d_con @ pr.conic
    MT = np.swapaxes(pr.M, 1, 2)
    d_Sig = MT @ d_cov @ pr.M
    d_M = 2.0 * d_cov @ pr.M @ pr.Sigma
    d_J = d_M @ Wm.T
    x, y, z = pr.pc.T
    fx, fy = cam.fx, cam.fy
    d_pc = np.stack([
        d_J[:, 0, 2] * (-fx / z ** 2) + d_mean[:, 0] * fx / z,
        d_J[:, 1, 2] * (-fy / z ** 2) + d_mean[:, 1] * fy / z,
        d_J[:, 0, 0] * (-fx / z ** 2) + d_J[:, 1, 1] * (-fy / z ** 2)
        + d_J[:, 0, 2] * (2 * fx * x / z ** 3) + d_J[:, 1, 2] * (2 * fy * y / z ** 3)
        - d_mean[:, 0] * fx * x / z ** 2 - d_mean[:, 1] * fy * y / z ** 2], axis=1)
    d_R = 2.0 * (d_Sig @ pr.R) * pr.D[:, None, :]
    d_ls = 2.0 * pr.D * np.einsum("nak,nab,nbk->nk", pr.R, d_Sig, pr.R)
    d_qh = np.einsum("nij,nqij->nq", d_R, _drot(pr.qh))
    d_q = (d_qh - pr.qh * (pr.qh * d_qh).sum(1, keepdims=True)) / pr.qn[:, None]

    live = pr.c_pre > 0.0
    dcp = d_col * live
    em = pr.e * pr.lm
    da = np.einsum("nc,nlc->nl", dcp, pr.amp)
    ga = da * em
    d_amp = dcp[:, None, :] * em[:, :, None]
    d_sh = ga * (pr.dot - 1.0)
    dmu = (ga * pr.sharp)[:, :, None] * pr.v[:, None, :]
    d_ax = (dmu - pr.mu * (pr.mu * dmu).sum(-1, keepdims=True)) / pr.un[..., None]
    dv = np.einsum("nl,nlk->nk", ga * pr.sharp, pr.mu)
    d_pos_c = (dv - pr.v * (pr.v * dv).sum(1, keepdims=True)) / pr.rd[:, None]

    i = pr.idx
    out["position"][i] = d_pc @ Wm + d_pos_c
    out["quat"][i] = d_q
    out["log_scale"][i] = d_ls
    out["opacity"][i] = d_oe * pr.pm
    out["prim_mask"][i] = d_oe * pr.op_raw
    out["diffuse"][i] = dcp
    out["axis_raw"][i] = d_ax
    out["sharpness"][i] = d_sh
    out["amplitude"][i] = d_amp
    out["lobe_mask"][i] = da * pr.e


# ------------------------------------------- all host cores (CPU baseline)
_POOL_STATE: dict = {}


def _pool_render(job):
    s, e = job
    st = _POOL_STATE
    px, py = st["px"][s:e], st["py"][s:e]
    b = _blend_block(st["pr"], px, py)
    return s, b["w"].T @ st["pr"].color + b["tbg"][:, None] * st["bg"]


def _pool_backward(job):
    s, e = job
    st = _POOL_STATE
    return _backward_pixels(st["pr"], st["g"][s:e], st["px"][s:e], st["py"][s:e], st["bg"], st["block"])


def _jobs(npx, procs, block):
    per = max(block, -(-npx // (4 * procs)) // block * block or block)
    return [(s, min(s + per, npx)) for s in range(0, npx, per)]


def render_parallel(p, cam, procs, background=(0.0, 0.0, 0.0), block=512):
    """``render`` with the pixel blocks spread over ``procs`` forked host
    processes (same arithmetic per pixel; used for CPU-baseline timing)."""
    import multiprocessing as mp
    bg = _f64(background).reshape(3)
    pr = project(p, cam)
    out = np.empty((cam.height * cam.width, 3))
    if pr is None:
        out[:] = bg
        return out.reshape(cam.height, cam.width, 3)
    px, py = _pixels(cam)
    _POOL_STATE.update(pr=pr, px=px, py=py, bg=bg)
    with mp.get_context("fork").Pool(procs) as pool:
        for s, blk in pool.imap_unordered(_pool_render, _jobs(px.size, procs, block)):
            out[s:s + blk.shape[0]] = blk
    _POOL_STATE.clear()
    return out.reshape(cam.height, cam.width, 3)


def loss_and_grads_parallel(p, cam, target, procs, lambda_ssim=0.2, background=(0.0, 0.0, 0.0), block=512):
    """``loss_and_grads`` with the forward and the per-pixel backward spread
    over ``procs`` forked host processes; the partial sums are added and the
    parameter chain runs once."""
    import multiprocessing as mp
    img = render_parallel(p, cam, procs, background, block)
    val, dimg = loss_and_dimg(img, _f64(target), lambda_ssim)
    n, L = _f64(p.position).shape[0], _f64(p.axis_raw).shape[1]
    out = {"position": np.zeros((n, 3)), "quat": np.zeros((n, 4)), "log_scale": np.zeros((n, 3)),
           "opacity": np.zeros(n), "diffuse": np.zeros((n, 3)), "axis_raw": np.zeros((n, L, 3)),
           "sharpness": np.zeros((n, L)), "amplitude": np.zeros((n, L, 3)),
           "lobe_mask": np.zeros((n, L)), "prim_mask": np.zeros(n)}
    pr = project(p, cam)
    if pr is None:
        return val, out, img
    px, py = _pixels(cam)
    _POOL_STATE.update(pr=pr, px=px, py=py, bg=_f64(background).reshape(3), g=_f64(dimg).reshape(-1, 3),
                       block=block)
    acc = None
    with mp.get_context("fork").Pool(procs) as pool:
        for part in pool.imap_unordered(_pool_backward, _jobs(px.size, procs, block)):
            acc = part if acc is None else tuple(a + b for a, b in zip(acc, part))
    _POOL_STATE.clear()
    _backward_chain(p, cam, pr, acc, out)
    return val, out, img


def loss_and_grads(p, cam, target, lambda_ssim=0.2, background=(0.0, 0.0, 0.0)):
    target = _f64(target)
    if target.shape != (cam.height, cam.width, 3):
        raise ValueError(f"target shape {target.shape} does not match camera "
                         f"{(cam.height, cam.width, 3)}")
    img = render(p, cam, background)
    val, dimg = loss_and_dimg(img, target, lambda_ssim)
    return val, backward(p, cam, project(p, cam), dimg, background), img


def vram_model_counts(p, cam, tile_px=16):
    """Reference 3-sigma VRAM model (postprocess.py:118-135): (visible, entries)."""
    pr = project(p, cam)
    if pr is None:
        return 0, 0
    rx = 3.0 * np.sqrt(pr.cov[:, 0, 0])
    ry = 3.0 * np.sqrt(pr.cov[:, 1, 1])
    x0, x1 = pr.mean[:, 0] - rx, pr.mean[:, 0] + rx
    y0, y1 = pr.mean[:, 1] - ry, pr.mean[:, 1] + ry
    on = (x1 > 0) & (x0 < cam.width) & (y1 > 0) & (y0 < cam.height)
    tx = (cam.width + tile_px - 1) // tile_px
    ty = (cam.height + tile_px - 1) // tile_px
    c = lambda v, m: np.clip(np.floor(v / tile_px), 0, m - 1).astype(np.int64)  # noqa: E731
    ent = (c(x1, tx) - c(x0, tx) + 1) * (c(y1, ty) - c(y0, ty) + 1)
    return int(on.sum()), int(ent[on].sum())
