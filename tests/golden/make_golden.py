"""Generate golden fixtures by running the REFERENCE implementation
(/root/reference/pkg/src/sgsplat, imported read-only) on seeded inputs.

Run in the build container (the reference does not exist on GPU boxes):
    python tests/golden/make_golden.py [name ...]
Outputs tests/golden/<name>.npz.  Inputs are the float32 scenes of
paper_2509_07021_b200.scenes (upcast to float64 for the reference), stored
alongside the outputs (or, for the 1M/5M scenes, a SHA-256 of the float32
inputs so generator drift is detected).
"""

from __future__ import annotations

import hashlib
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import sgsplat  # noqa: E402,F401
from sgsplat import postprocess as P  # noqa: E402
from sgsplat.scene import ColorModel, GaussianPrimitive, Scene  # noqa: E402

from paper_2509_07021_b200 import scenes  # noqa: E402

R = sys.modules["sgsplat.render"]  # the module (sgsplat.render is shadowed by the function)
OUT = Path(__file__).resolve().parent
FIELDS = scenes.FIELDS


def ref_params(s, opacity_scale=None):
    kw = {f: np.asarray(getattr(s, f), dtype=np.float64) for f in FIELDS}
    if s.prim_mask is not None:
        kw["opacity"] = kw["opacity"] * np.asarray(s.prim_mask, np.float64)
    if opacity_scale is not None:
        kw["opacity"] = kw["opacity"] * opacity_scale
    lm = np.asarray(s.lobe_mask, np.float64)
    return R.SceneParams(**kw, lobe_mask=lm)


def ref_cam(c):
    return R.Camera(rotation=c.rotation, translation=c.translation, fx=c.fx, fy=c.fy, cx=c.cx,
                    cy=c.cy, width=c.width, height=c.height, near=c.near)


def cam_dict(c):
    return dict(cam_R=np.asarray(c.rotation), cam_t=np.asarray(c.translation),
                cam_intr=np.array([c.fx, c.fy, c.cx, c.cy, c.near]),
                cam_size=np.array([c.width, c.height]))


def scene_dict(s):
    d = {f: getattr(s, f) for f in FIELDS}
    d["lobe_mask"] = s.lobe_mask
    if s.prim_mask is not None:
        d["prim_mask"] = s.prim_mask
    return d


def digest(s):
    h = hashlib.sha256()
    for f in FIELDS + ("lobe_mask",):
        h.update(np.ascontiguousarray(getattr(s, f)).tobytes())
    if s.prim_mask is not None:
        h.update(np.ascontiguousarray(s.prim_mask).tobytes())
    return h.hexdigest()


def save(name, **kw):
    np.savez_compressed(OUT / f"{name}.npz", **kw)
    print(f"wrote {name}.npz", flush=True)


def gen_cfg0_full():
    s, cams = scenes.config0()
    t = time.time()
    img = R._render_params(ref_params(s), ref_cam(cams[0]), (0.0, 0.0, 0.0))
    save("cfg0_full", img=img, seconds=time.time() - t, **scene_dict(s), **cam_dict(cams[0]))


def gen_cfg0_grads():
    """loss_and_grads (default L1 + 0.2 SSIM) on a 64x48 crop, 2000-primitive subset."""
    s, cams = scenes.config0(n=2000)
    cam = cams[0].crop(96, 100, 64, 48)
    tgt = scenes.target_image(0, cam.height, cam.width)
    p = ref_params(s)
    out = {}
    for lam in (0.0, 0.2):
        val, g = R.loss_and_grads(p, ref_cam(cam), tgt.astype(np.float64), R.LossConfig(lambda_ssim=lam))
        out[f"loss_{lam}"] = np.array(val)
        for f in FIELDS:
            out[f"g{lam}_{f}"] = getattr(g, f)
    img = R._render_params(p, ref_cam(cam), (0.0, 0.0, 0.0))
    save("cfg0_crop_grads", img=img, target=tgt, **out, **scene_dict(s), **cam_dict(cam))


def gen_masks():
    """cfg1-style soft masks on a small scene: images with float lobe masks and
    prim masks folded into opacity, plus central-difference mask gradients."""
    s, cams = scenes.config1(n=400)
    rng = np.random.default_rng(5)
    s.prim_mask = rng.uniform(0.2, 1.0, size=s.n).astype(np.float32)
    s.lobe_mask = rng.uniform(0.0, 1.0, size=(s.n, 3)).astype(np.float32)
    cam = cams[0].crop(600, 330, 40, 32)
    tgt = scenes.target_image(1, cam.height, cam.width)
    cfg = R.LossConfig(lambda_ssim=0.2)
    rc = ref_cam(cam)

    def loss_of(sc):
        img = R._render_params(ref_params(sc), rc, (0.0, 0.0, 0.0))
        return R._loss_and_dimg(img, tgt.astype(np.float64), cfg)[0]

    val, g = R.loss_and_grads(ref_params(s), rc, tgt.astype(np.float64), cfg)
    img = R._render_params(ref_params(s), rc, (0.0, 0.0, 0.0))
    # FD mask gradients for primitives with the largest |dL/dopacity|
    pick = np.argsort(-np.abs(g.opacity))[:12]
    h = 1e-6
    fd_pm, fd_lm = np.zeros(len(pick)), np.zeros((len(pick), 3))
    for j, i in enumerate(pick):
        for l in range(-1, 3):
            sp = s.subset(np.arange(s.n))
            sm = s.subset(np.arange(s.n))
            sp.prim_mask, sm.prim_mask = s.prim_mask.astype(np.float64), s.prim_mask.astype(np.float64)
            sp.lobe_mask, sm.lobe_mask = s.lobe_mask.astype(np.float64), s.lobe_mask.astype(np.float64)
            if l < 0:
                sp.prim_mask[i] += h
                sm.prim_mask[i] -= h
                fd_pm[j] = (loss_of(sp) - loss_of(sm)) / (2 * h)
            else:
                sp.lobe_mask[i, l] += h
                sm.lobe_mask[i, l] -= h
                fd_lm[j, l] = (loss_of(sp) - loss_of(sm)) / (2 * h)
    out = {f"g_{f}": getattr(g, f) for f in FIELDS}
    save("masks_grads", img=img, target=tgt, loss=np.array(val), pick=pick, fd_prim_mask=fd_pm,
         fd_lobe_mask=fd_lm, **out, **scene_dict(s), **cam_dict(cam))


def gen_accept_grads():
    """The reference acceptance-suite gradient scenes (test_acceptance.py:117-170):
    5 primitives, 2 lobes, 16x16, seeds 0..4, default LossConfig."""
    out = {}
    for seed in range(5):
        rng = np.random.default_rng(seed)
        cam = R.Camera.look_at(eye=(0, -2.5, 0.3), target=(0, 0, 0), width=16, height=16, fx=20)
        n, lmax = 5, 2
        p = R.SceneParams(
            position=rng.normal(scale=0.4, size=(n, 3)), quat=rng.normal(size=(n, 4)),
            log_scale=np.log(rng.uniform(0.1, 0.3, size=(n, 3))),
            opacity=rng.uniform(0.3, 0.8, size=n), diffuse=rng.uniform(0.35, 0.9, size=(n, 3)),
            axis_raw=rng.normal(size=(n, lmax, 3)), sharpness=rng.uniform(0.5, 6.0, size=(n, lmax)),
            amplitude=rng.uniform(-0.1, 0.3, size=(n, lmax, 3)),
            lobe_mask=np.ones((n, lmax), dtype=bool))
        for f in FIELDS:  # round to float32 so the GPU sees the same inputs
            setattr(p, f, getattr(p, f).astype(np.float32).astype(np.float64))
        noise = (rng.uniform(0.02, 0.08, size=(16, 16, 3)) * rng.choice([-1.0, 1.0], size=(16, 16, 3)))
        target = R._render_params(p, cam, (0, 0, 0)) + noise
        val, g = R.loss_and_grads(p, cam, target, R.LossConfig())
        out[f"s{seed}_target"] = target
        out[f"s{seed}_loss"] = np.array(val)
        out[f"s{seed}_img"] = R._render_params(p, cam, (0, 0, 0))
        for f in FIELDS:
            out[f"s{seed}_{f}"] = getattr(p, f)
            out[f"s{seed}_g_{f}"] = getattr(g, f)
    out.update(cam_dict(cam))
    save("accept_grads", **out)


def gen_crop(name, cfg, cam_index, x0, y0, w, h):
    s, cams = scenes.CONFIGS[cfg]()
    cam = cams[cam_index].crop(x0, y0, w, h)
    R._PIXEL_CHUNK = 64
    sys.modules["sgsplat.render"]._PIXEL_CHUNK = 64
    t = time.time()
    img = R._render_params(ref_params(s), ref_cam(cam), (0.0, 0.0, 0.0))
    sec = time.time() - t
    save(name, img=img, seconds=np.array(sec), digest=np.array(digest(s)), cfg=np.array(cfg),
         cam_index=np.array(cam_index), crop=np.array([x0, y0, w, h]), **cam_dict(cam))


def gen_aniso_grads():
    """Anisotropic gradients (configs[4] scale distribution: one log-scale axis
    N(-2.5, 0.5), two N(-5, 0.5)): loss_and_grads (default L1 + 0.2 SSIM) on a
    32x24 crop of the 4K camera, for the primitives of config4(n=500k) whose
    opacity-aware support box (q <= 2 ln(o/1e-7)) meets the crop.  Checks the
    backward's projection chain on elongated splats."""
    from oracle import ref_dense
    s, (cam0,) = scenes.config4(n=500_000)
    x0, y0, w, h = 1200, 700, 32, 24
    pr = ref_dense.project(s, cam0)
    o = np.asarray(s.opacity, np.float64)[pr.idx]
    qmax = np.maximum(2 * np.log(np.maximum(o, 1e-30) / 1e-7), 0.0)
    hx, hy = np.sqrt(qmax * pr.cov[:, 0, 0]) + 1, np.sqrt(qmax * pr.cov[:, 1, 1]) + 1
    mx, my = pr.mean[:, 0], pr.mean[:, 1]
    m = (qmax > 0) & (mx + hx > x0) & (mx - hx < x0 + w) & (my + hy > y0) & (my - hy < y0 + h)
    idx = np.sort(pr.idx[m]).astype(np.int64)
    sub = s.subset(idx)
    cam = cam0.crop(x0, y0, w, h)
    tgt = scenes.target_image(4, cam.height, cam.width)
    p = ref_params(sub)
    val, g = R.loss_and_grads(p, ref_cam(cam), tgt.astype(np.float64), R.LossConfig())
    img = R._render_params(p, ref_cam(cam), (0.0, 0.0, 0.0))
    out = {f"g_{f}": getattr(g, f) for f in FIELDS}
    save("aniso_grads", idx=idx, img=img, target=tgt, loss=np.array(val), digest=np.array(digest(s)),
         crop=np.array([x0, y0, w, h]), **out, **cam_dict(cam))


def gen_zero_opacity():
    """Primitives at opacity exactly 0 (the pruning loop clamps there,
    prune.py:185): the reference's dense blend still gives them
    dL/do = sum G dL/dalpha (render.py:538-560).  configs[0] distributions,
    2000 primitives, every fifth one at opacity 0, a 64x48 crop."""
    s, cams = scenes.config0(n=2000, seed=5)
    s.opacity[::5] = np.float32(0.0)
    cam = cams[0].crop(96, 100, 64, 48)
    tgt = scenes.target_image(5, cam.height, cam.width)
    p = ref_params(s)
    val, g = R.loss_and_grads(p, ref_cam(cam), tgt.astype(np.float64), R.LossConfig())
    out = {f"g_{f}": getattr(g, f) for f in FIELDS}
    save("zero_opacity", target=tgt, loss=np.array(val), **out, **scene_dict(s), **cam_dict(cam))


def gen_vram():
    """estimate_vram (postprocess.py:101-137) on seeded random scenes."""
    out = {}
    rng = np.random.default_rng(11)
    for k in range(4):
        n = [1, 25, 200, 1000][k]
        prims = [GaussianPrimitive(position=rng.uniform(-2, 2, 3), rotation=rng.normal(size=4) / 2,
                                   scale=rng.uniform(0.01, 0.6, 3), opacity=float(rng.uniform()),
                                   diffuse=rng.uniform(0, 1, 3)) for _ in range(n)]
        for p in prims:
            p.rotation = (p.rotation / np.linalg.norm(p.rotation)).astype(np.float32)
        sc = Scene(prims, ColorModel.sg(3))
        cam = R.Camera.look_at(eye=(0.3, -3.0, 0.8), target=(0, 0, 0), width=96, height=64, fx=80)
        for tile in (8, 16):
            est = P.estimate_vram(sc, cam, tile_px=tile)
            out[f"k{k}_t{tile}"] = np.array([est.static_bytes, est.dynamic_bytes])
        out[f"k{k}_position"] = np.stack([p.position for p in prims])
        out[f"k{k}_quat"] = np.stack([p.rotation for p in prims])
        out[f"k{k}_scale"] = np.stack([p.scale for p in prims])
        out[f"k{k}_opacity"] = np.array([p.opacity for p in prims], np.float32)
    out.update(cam_dict(cam))
    save("vram_model", **out)


def gen_admm():
    """The reference ADMM loop (prune.run_state) on a small scene: 3 views of
    24x20 crops, 8 iterations, proximal event every 3 (magnitude and range
    operators), plus one prox_project on random scores with ties."""
    from sgsplat import prune as PR
    s, cams = scenes.config0(n=300, seed=3)
    views = []
    for k, (x0, y0) in enumerate([(116, 118), (100, 110), (130, 124)]):
        cam = cams[0].crop(x0, y0, 24, 20)
        tgt = scenes.target_image(7, cam.height, cam.width, view=k)
        views.append((cam, tgt))
    out = {}
    for op in ("sharpness", "range"):
        p = ref_params(s)
        p.lobe_mask = np.asarray(s.lobe_mask) > 0.5
        cfg = PR.PrunerConfig.from_keep_ratios(s.n, int(p.lobe_mask.sum()), 0.6, 0.5, delta=5e-3,
                                               iters=8, prox_every=3, sharpness_operator=op, seed=1)
        st = PR.PrunerState.init(p)
        trace = PR.run_state(st, [(ref_cam(c), t.astype(np.float64)) for c, t in views], cfg)
        for f in FIELDS:
            out[f"{op}_{f}"] = getattr(p, f)
        out[f"{op}_proxy_o"], out[f"{op}_proxy_s"] = st.proxy_o, st.proxy_s
        out[f"{op}_dual_o"], out[f"{op}_dual_s"] = st.dual_o, st.dual_s
        out[f"{op}_trace"] = np.array([[r.iteration, r.loss, r.residual_o, r.residual_s,
                                        r.active_primitives, r.active_lobes, r.budget_units]
                                       for r in trace])
        out[f"{op}_kappa"] = np.array([cfg.kappa, cfg.kappa_o, cfg.kappa_s])
    rng = np.random.default_rng(4)
    o_in = np.round(rng.normal(size=500), 1)        # many ties
    s_in = np.round(rng.normal(size=(500, 3)), 1)
    cfgp = PR.PrunerConfig(kappa=11 * 137 + 7 * 611, kappa_o=137, kappa_s=611)
    po, ps = PR.prox_project(o_in, s_in, cfgp)
    out.update(prox_o_in=o_in, prox_s_in=s_in, prox_o=po, prox_s=ps)
    for k, (c, t) in enumerate(views):
        out.update({f"v{k}_{key}": v for key, v in cam_dict(c).items()})
        out[f"v{k}_target"] = t
    save("admm", **out, **scene_dict(s))


def gen_compact():
    """A MEGS2 compact file written by the reference (io.write_compact) and
    what its read_compact + SceneParams.from_scene make of it: varying lobe
    counts (0..5, so max_lobes exceeds the default 3)."""
    from sgsplat import io as IO
    from sgsplat.scene import SGLobe
    rng = np.random.default_rng(21)
    prims = []
    for i in range(257):
        nl = int(rng.integers(0, 4)) if i != 100 else 5
        q = rng.normal(size=4)
        lobes = []
        for _ in range(nl):
            ax = rng.normal(size=3)
            lobes.append(SGLobe(axis=ax / np.linalg.norm(ax), sharpness=float(rng.uniform(0, 40)),
                                amplitude=rng.normal(0, 0.3, 3)))
        prims.append(GaussianPrimitive(position=rng.uniform(-1, 1, 3), rotation=q / np.linalg.norm(q),
                                       scale=np.exp(rng.normal(-3, 0.5, 3)), opacity=float(rng.uniform()),
                                       diffuse=rng.uniform(0, 1, 3), lobes=lobes))
    sc = Scene(prims, ColorModel.sg(5))
    data = IO.write_compact(sc)
    back = IO.read_compact(data)
    p = R.SceneParams.from_scene(back)
    out = {f: getattr(p, f) for f in FIELDS}
    out["lobe_mask"] = p.lobe_mask
    out["raw"] = np.frombuffer(data, np.uint8)
    out["scale"] = np.stack([q.scale for q in prims])
    out["n_lobes"] = np.array([len(q.lobes) for q in prims])
    save("compact", **out)


GENERATORS = {
    "compact": gen_compact,
    "admm": gen_admm,
    "accept_grads": gen_accept_grads,
    "vram_model": gen_vram,
    "masks_grads": gen_masks,
    "cfg0_crop_grads": gen_cfg0_grads,
    "cfg0_full": gen_cfg0_full,
    "cfg2_crop": lambda: gen_crop("cfg2_crop", 2, 0, 952, 532, 16, 16),
    "cfg3_crop": lambda: gen_crop("cfg3_crop", 3, 0, 632, 352, 16, 16),
    "cfg1_crop": lambda: gen_crop("cfg1_crop", 1, 0, 632, 352, 24, 16),
    "cfg4_crop": lambda: gen_crop("cfg4_crop", 4, 0, 1912, 1072, 8, 8),
    # round 2: three reference crops per config, other
    # cameras and positions, incl. the configs[4] cluster centre at 16x16
    "cfg1_crop_b": lambda: gen_crop("cfg1_crop_b", 1, 0, 200, 150, 16, 16),
    "cfg1_crop_c": lambda: gen_crop("cfg1_crop_c", 1, 0, 1000, 560, 16, 16),
    "cfg2_crop_b": lambda: gen_crop("cfg2_crop_b", 2, 21, 400, 300, 16, 16),
    "cfg2_crop_c": lambda: gen_crop("cfg2_crop_c", 2, 45, 1500, 800, 16, 16),
    "cfg3_crop_b": lambda: gen_crop("cfg3_crop_b", 3, 3, 300, 200, 16, 16),
    "cfg3_crop_c": lambda: gen_crop("cfg3_crop_c", 3, 6, 900, 500, 16, 16),
    "cfg4_crop_b": lambda: gen_crop("cfg4_crop_b", 4, 0, 1904, 1064, 16, 16),
    "cfg4_crop_c": lambda: gen_crop("cfg4_crop_c", 4, 0, 1200, 700, 16, 16),
    "aniso_grads": gen_aniso_grads,
    "zero_opacity": gen_zero_opacity,
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(GENERATORS)
    for nm in names:
        t = time.time()
        GENERATORS[nm]()
        print(f"  {nm}: {time.time() - t:.1f}s", flush=True)
