"""GPU parity: libsgs.so (through the C ABI) against the CPU tiled oracle.

Bit-exact: preprocess integer outputs and records, tile key lists, sorted
orders, per-tile ranges, visibility counts.  Tolerance: images (<= 1e-5 vs
the oracle's fp32 raster; the 1e-4 reference bar is checked in
test_gpu_reference.py) and gradients (composite criterion).
"""

import numpy as np
import pytest
import torch

from oracle import tiled
from helpers import image_parity
from paper_2509_07021_b200 import _ffi, scenes
from paper_2509_07021_b200.rasterizer import GaussianTensors, Rasterizer, sort_pairs_u64

pytestmark = pytest.mark.gpu

MODES = [_ffi.SORT_DEPTH_FIRST, _ffi.SORT_KEY64]


def _gpu_frame(scene, cam, mode=_ffi.SORT_DEPTH_FIRST, bg=(0.0, 0.0, 0.0), tile_rows=None):
    rast = Rasterizer(sort_mode=mode)
    g = GaussianTensors.from_arrays(scene)
    frame = rast.forward(g, cam, bg, tile_rows=tile_rows)
    torch.cuda.synchronize()
    return rast, g, frame


def _check_bins(rast, frame, ref):
    st = frame.stats()
    assert st["n_visible"] == ref.n_visible
    assert st["n_emitting"] == ref.n_emitting
    assert st["n_entries"] == ref.n_entries
    keys, vals, ranges = rast.export_bins(frame)
    assert np.array_equal(keys.cpu().numpy().view(np.uint64), ref.keys)
    assert np.array_equal(vals.cpu().numpy().view(np.uint32), ref.vals)
    assert np.array_equal(ranges.cpu().numpy().view(np.uint32), ref.ranges)


def _check_projected(rast, frame, ref):
    depth, rect, tt, rec = (t.cpu().numpy() for t in rast.export_projected(frame))
    assert np.array_equal(depth.view(np.uint32), ref.depth_bits)
    assert np.array_equal(tt.view(np.uint32), ref.tiles_touched)
    emit = ref.tiles_touched > 0
    assert np.array_equal(rect.view(np.uint32)[emit], ref.rect[emit])
    assert np.array_equal(rec[emit].view(np.uint32), ref.records[emit].view(np.uint32))


def _img_ok(frame, ref):
    # device ex2.approx vs host exp2f: <= 1e-5 except rare termination flips
    image_parity(frame.img.cpu().numpy(), ref.img, ref.T, tol=1e-5, flip_frac=1e-4, flip_tol=2e-4)


@pytest.mark.parametrize("mode", MODES)
def test_config0_bit_exact_bins(mode):
    scene, cams = scenes.config0()
    ref = tiled.render(scene, cams[0])
    rast, g, frame = _gpu_frame(scene, cams[0], mode)
    _check_projected(rast, frame, ref)
    _check_bins(rast, frame, ref)
    _img_ok(frame, ref)
    assert np.array_equal(frame.ncontrib.cpu().numpy().view(np.uint32) > 0, ref.nc > 0)


@pytest.mark.parametrize("mode", MODES)
def test_config1_masks_bit_exact(mode):
    scene, cams = scenes.config1()
    ref = tiled.render(scene, cams[0])
    rast, g, frame = _gpu_frame(scene, cams[0], mode)
    _check_projected(rast, frame, ref)
    _check_bins(rast, frame, ref)
    _img_ok(frame, ref)


def test_config2_camera0_bit_exact():
    scene, cams = scenes.config2(n_cams=1)
    ref = tiled.preprocess(scene, cams[0])
    tiled.bin(ref)
    rast, g, frame = _gpu_frame(scene, cams[0])
    _check_projected(rast, frame, ref)
    _check_bins(rast, frame, ref)


def test_background_and_importance():
    scene, cams = scenes.config0(n=3000)
    cam = cams[0].crop(32, 40, 96, 80)
    bg = (0.2, 0.5, 0.9)
    ref = tiled.render(scene, cam, bg, importance=True)
    rast = Rasterizer()
    g = GaussianTensors.from_arrays(scene)
    ws = torch.zeros(g.n, dtype=torch.float32, device="cuda")
    frame = rast.forward(g, cam, bg, weight_sums=ws)
    assert np.abs(frame.img.cpu().numpy() - ref.img).max() <= 1e-5
    assert np.abs(frame.final_T.cpu().numpy() - ref.T).max() <= 1e-5
    np.testing.assert_allclose(ws.cpu().numpy(), ref.weight_sums, rtol=1e-4, atol=1e-4)


@pytest.mark.parametrize("mode", MODES)
def test_strips_equal_full_frame(mode):
    """Tile-row windows (the strip path: emitting depth keys compacted before
    the depth sort) in both sort modes: bins bit-exact, strips tile the frame."""
    scene, cams = scenes.config0()
    cam = cams[0]
    rast = Rasterizer(sort_mode=mode)
    g = GaussianTensors.from_arrays(scene)
    full = rast.forward(g, cam).img.clone()
    parts = torch.zeros_like(full)
    for y0, y1 in [(0, 5), (5, 11), (11, 16)]:
        f = rast.forward(g, cam, tile_rows=(y0, y1))
        parts[y0 * 16:y1 * 16] = f.img[y0 * 16:y1 * 16]
        ref = tiled.render(scene, cam, tile_rows=(y0, y1))
        _check_bins(rast, f, ref)
    assert torch.equal(full, parts)


def test_empty_and_culled():
    scene, cams = scenes.config0(n=50)
    cam = cams[0]
    behind = scene.subset(np.arange(50))
    behind.position = (np.asarray(cam.center) * 2.0 + np.zeros((50, 3))).astype(np.float32)
    rast, g, frame = _gpu_frame(behind, cam, bg=(0.3, 0.3, 0.3))
    st = frame.stats()
    assert st["n_emitting"] == 0 and st["n_entries"] == 0
    assert torch.allclose(frame.img, torch.full_like(frame.img, 0.3))
    zero_op = scene.subset(np.arange(50))
    zero_op.opacity = np.zeros(50, np.float32)
    rast, g, frame = _gpu_frame(zero_op, cam)
    assert frame.stats()["n_entries"] == 0
    assert float(frame.img.abs().max()) == 0.0


def test_capacity_growth():
    scene, cams = scenes.config0()
    rast = Rasterizer(initial_capacity=1000)
    g = GaussianTensors.from_arrays(scene)
    frame = rast.forward(g, cams[0])
    ref = tiled.render(scene, cams[0])
    st = frame.stats()
    assert frame.ws.capacity >= st["n_bin_entries"] > 1000 and not st["overflow"]
    _check_bins(rast, frame, ref)


@pytest.mark.parametrize("n,bits", [(1, 8), (1000, 13), (70_001, 45), (1_000_003, 40), (5000, 64)])
def test_sort_pairs_u64(n, bits):
    rng = np.random.default_rng(n)
    hi = np.uint64((1 << bits) - 1) if bits < 64 else np.uint64(0xFFFFFFFFFFFFFFFF)
    keys = rng.integers(0, 1 << 62, size=n, dtype=np.uint64) * np.uint64(3) & hi
    keys[: n // 3] = keys[0]  # many ties -> stability matters
    vals = np.arange(n, dtype=np.uint32)
    kt = torch.from_numpy(keys.view(np.int64).copy()).cuda()
    vt = torch.from_numpy(vals.view(np.int32).copy()).cuda()
    sort_pairs_u64(kt, vt, bits)
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(kt.cpu().numpy().view(np.uint64), keys[order])
    assert np.array_equal(vt.cpu().numpy().view(np.uint32), vals[order])


def _composite_ok(a, b, rel=1e-3, floor=1e-5):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    tol = rel * np.abs(b) + floor * max(np.abs(b).max(), 1e-30)
    return np.abs(a - b) <= tol


@pytest.mark.parametrize("bg", [(0.0, 0.0, 0.0), (0.3, 0.6, 0.1)])
def test_backward_matches_oracle(bg):
    scene, cams = scenes.config0()
    cam = cams[0].crop(64, 64, 128, 96)
    target = scenes.target_image(0, cam.height, cam.width)
    ref = tiled.render(scene, cam, bg)
    rast = Rasterizer()
    g = GaussianTensors.from_arrays(scene)
    frame = rast.forward(g, cam, bg)
    dimg = np.sign(frame.img.cpu().numpy() - target) / target.size
    grads = rast.backward(g, frame, torch.from_numpy(dimg.astype(np.float32)).cuda())
    tiled.raster_backward(ref, dimg)
    og = tiled.preprocess_backward(ref)
    g2 = grads["grad2d"].cpu().numpy()
    assert _composite_ok(g2, ref.grad2d, floor=1e-4).all()
    for k in ("position", "quat", "log_scale", "opacity", "diffuse", "axis_raw", "sharpness",
              "amplitude", "lobe_mask", "prim_mask"):
        ok = _composite_ok(grads[k].cpu().numpy(), og[k])
        assert ok.mean() == 1.0, f"{k}: {np.count_nonzero(~ok)} of {ok.size} outside tolerance"


@pytest.mark.parametrize("mode", MODES)
def test_untracked_render_equals_tracked(mode):
    """The image-only forward (no contributor counts) renders the same bits."""
    scene, cams = scenes.config1(n=20_000)
    cam = cams[0]
    rast = Rasterizer(sort_mode=mode)
    g = GaussianTensors.from_arrays(scene)
    a = rast.forward(g, cam, (0.1, 0.2, 0.3))
    img_a, T_a = a.img.clone(), a.final_T.clone()
    b = rast.forward(g, cam, (0.1, 0.2, 0.3), track=False)
    assert b.ncontrib is None
    assert torch.equal(img_a, b.img) and torch.equal(T_a, b.final_T)
    with pytest.raises(ValueError):
        rast.backward(g, b, torch.zeros_like(b.img))


def test_large_splats_overflow_row_span_store():
    """Splats spanning many tile rows exhaust the preprocess's row-span store
    (8 rows per primitive on average): the primitives that did not fit are
    re-solved by the emission.  Lists stay bit-exact, image within 1e-5."""
    scene, cams = scenes.config0(n=1500)
    rng = np.random.default_rng(7)
    scene.log_scale = rng.normal(-1.2, 0.3, size=scene.log_scale.shape).astype(np.float32)
    cam = cams[0].crop(0, 0, 256, 256)
    ref = tiled.render(scene, cam)
    rows = (ref.rect[:, 1] >> 16).astype(np.int16).astype(np.int64) - (ref.rect[:, 1] & 0xffff) + 1
    assert rows[ref.tiles_touched > 0].mean() > 8  # the store cannot hold every row
    rast, g, frame = _gpu_frame(scene, cam)
    _check_projected(rast, frame, ref)
    _check_bins(rast, frame, ref)
    _img_ok(frame, ref)


@pytest.mark.parametrize("mode", MODES)
def test_bin_is_repeatable_after_one_preprocess(mode):
    """sgs_bin leaves the preprocess outputs intact (the depth sort reads the
    preprocess's keys in place): binning twice gives the same lists."""
    import ctypes as C
    scene, cams = scenes.config0(n=5000)
    cam = cams[0]
    rast, g, frame = _gpu_frame(scene, cam, mode)
    k1, v1, r1 = (t.cpu().numpy().copy() for t in rast.export_bins(frame))
    _ffi.call("sgs_bin", C.byref(frame.cam), C.byref(frame.ws.desc),
              C.c_void_p(torch.cuda.current_stream().cuda_stream))
    k2, v2, r2 = (t.cpu().numpy() for t in rast.export_bins(frame))
    assert np.array_equal(k1, k2) and np.array_equal(v1, v2) and np.array_equal(r1, r2)


@pytest.mark.parametrize("w,h", [(1, 1), (37, 23), (17, 250), (130, 9)])
def test_odd_image_sizes(w, h):
    """Partial tiles and super-tiles at the right / bottom edges (image sizes
    that are no multiple of 16 or 64): lists bit-exact, image and backward
    partials as the oracle's."""
    scene, cams = scenes.config0(n=3000)
    cam = cams[0].crop(100, 90, w, h)
    ref = tiled.render(scene, cam)
    rast, g, frame = _gpu_frame(scene, cam)
    _check_projected(rast, frame, ref)
    _check_bins(rast, frame, ref)
    _img_ok(frame, ref)
    dimg = np.random.default_rng(3).normal(size=ref.img.shape)
    tiled.raster_backward(ref, dimg)
    gr = rast.backward_raster(g, frame, torch.as_tensor(dimg, dtype=torch.float32, device="cuda"))
    assert _composite_ok(gr.cpu().numpy().reshape(ref.grad2d.shape), ref.grad2d, floor=1e-4).all()


@pytest.mark.parametrize("mode", MODES)
def test_grad_floor_bins_and_backward_match_oracle(mode):
    """Gradient renders with the opacity floor (sgs_camera.grad_floor):
    primitives at o_eff = 0 and below the floor are binned with the floor's
    support -- lists bit-exact with the CPU restatement under the same floor,
    the image unchanged where they blend with alpha = 0 -- and the backward
    gives them dL/do (per-unit-opacity partials) against the oracle."""
    scene, cams = scenes.config0(n=4000)
    s = scene.subset(np.arange(scene.n))
    s.opacity[::4] = np.float32(0.0)
    s.opacity[1::8] = np.float32(2e-6)
    cam = cams[0].crop(64, 64, 128, 96)
    floor = 1e-3
    ref = tiled.render(s, cam, grad_floor=floor)
    rast = Rasterizer(sort_mode=mode)
    g = GaussianTensors.from_arrays(s)
    plain = rast.forward(g, cam, track=False, private=True)
    frame = rast.forward(g, cam, grad_floor=floor)
    _check_bins(rast, frame, ref)
    assert frame.stats()["n_entries"] > plain.stats()["n_entries"]
    _img_ok(frame, ref)
    assert float((frame.img - plain.img).abs().max()) < 1e-6     # alpha = 0 records add nothing
    target = scenes.target_image(3, cam.height, cam.width)
    dimg = np.sign(frame.img.cpu().numpy() - target) / target.size
    grads = rast.backward(g, frame, torch.from_numpy(dimg.astype(np.float32)).cuda())
    tiled.raster_backward(ref, dimg)
    og = tiled.preprocess_backward(ref)
    for k in ("position", "quat", "log_scale", "opacity", "diffuse", "axis_raw", "sharpness", "amplitude",
              "lobe_mask", "prim_mask"):
        ok = _composite_ok(grads[k].cpu().numpy(), og[k])
        assert ok.mean() == 1.0, f"{k}: {np.count_nonzero(~ok)} of {ok.size} outside tolerance"
    zo = og["opacity"][::4]
    assert np.count_nonzero(np.abs(zo) > 1e-3 * np.abs(og["opacity"]).max()) > 10


def test_autograd_function_matches_explicit_backward():
    """render_torch (torch.autograd.Function over K5/K6/K7, SURVEY §8(b)'s
    fast path): gradients of a torch-composed L1 loss equal the explicit
    Rasterizer.backward on the same dL/dimg, mask gradients included."""
    from paper_2509_07021_b200.rasterizer import GRAD_FIELDS, render_torch
    scene, cams = scenes.config1(n=3000)
    cam = cams[0].crop(560, 300, 128, 96)
    tgt = torch.from_numpy(scenes.target_image(2, cam.height, cam.width)).cuda()
    rast = Rasterizer()
    leaves = {f: torch.from_numpy(np.ascontiguousarray(getattr(scene, f))).cuda().requires_grad_(True)
              for f in GRAD_FIELDS}
    lm = torch.from_numpy(np.ascontiguousarray(scene.lobe_mask)).cuda().requires_grad_(True)
    pm = torch.from_numpy(np.ascontiguousarray(scene.prim_mask)).cuda().requires_grad_(True)
    img = render_torch(rast, cam, (0.0, 0.0, 0.0), *(leaves[f] for f in GRAD_FIELDS), lm, pm)
    loss = (img - tgt).abs().mean()
    loss.backward()
    g = GaussianTensors.from_arrays(scene)
    frame = rast.forward(g, cam)
    assert torch.equal(frame.img, img.detach())
    dimg = torch.sign(frame.img - tgt) / img.numel()
    want = rast.backward(g, frame, dimg, mask_grads=True)
    for f in GRAD_FIELDS:
        assert torch.allclose(leaves[f].grad, want[f], rtol=1e-5, atol=1e-7 * float(want[f].abs().max())), f
    assert torch.allclose(lm.grad, want["lobe_mask"], rtol=1e-5, atol=1e-7 * float(want["lobe_mask"].abs().max()))
    assert torch.allclose(pm.grad, want["prim_mask"], rtol=1e-5, atol=1e-7 * float(want["prim_mask"].abs().max()))


def test_multi_view_parameter_backward_equals_sequential():
    """sgs_preprocess_backward_views (K7 over several views, rows written
    once) is bit-identical to one sgs_preprocess_backward per view in view
    order, accumulating -- including more views than one launch takes."""
    scene, cams = scenes.config3(n=20000, n_views=10)
    rast = Rasterizer()
    g = GaussianTensors.from_arrays(scene)
    c_cams, g2ds = [], []
    for v, cam in enumerate(cams):
        f = rast.forward(g, cam, grad_floor=0.001)
        tgt = torch.from_numpy(scenes.target_image(0, cam.height, cam.width, v)).cuda()
        dimg = (f.img - tgt) * 1e-3
        g2ds.append(rast.backward_raster(g, f, dimg).clone())
        c_cams.append(f.cam)
    seq = None
    for c, t in zip(c_cams, g2ds):
        seq = rast.backward_params(g, c, t, mask_grads=True, out=seq, accumulate=seq is not None, mask_logit=True)
    multi = rast.backward_params_views(g, c_cams, g2ds, mask_grads=True, mask_logit=True)
    torch.cuda.synchronize()
    for k in seq:
        assert torch.equal(seq[k], multi[k]), k
    assert float(multi["position"].abs().sum()) > 0
