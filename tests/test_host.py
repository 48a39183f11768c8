"""CPU: the C ABI library loads and exports every symbol include/sgs.h
declares; host-only entry points validate arguments like the reference API;
host-side helpers (camera, scenes, packing, sharding) behave."""

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2509_07021_b200 import _ffi, scenes
from paper_2509_07021_b200.camera import Camera, to_sgs
from paper_2509_07021_b200.sharding import balanced_strips, row_costs_from_rects, shard_views

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "sgs.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int32_t|const char\*)\s+(sgs_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _ffi.load()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _ffi.SIGNATURES, f"{s} missing from the ctypes binding"
    assert lib.sgs_version() >= 100


def test_struct_layouts_match_header():
    # sizes of the ABI structs as C sees them (x86-64 SysV)
    assert C.sizeof(_ffi.SgsCamera) == 4 * 9 + 4 * 3 + 4 * 5 + 4 * 4 + 4 + 8 * 4 + 8 + 8
    # ... and as the library itself was compiled
    sizes = (C.c_uint64 * 4)()
    assert _ffi.load().sgs_abi_sizes(sizes) == _ffi.SGS_OK
    assert list(sizes) == [C.sizeof(_ffi.SgsCamera), C.sizeof(_ffi.SgsParams), C.sizeof(_ffi.SgsWorkspace),
                           C.sizeof(_ffi.SgsStats)]
    assert C.sizeof(_ffi.SgsParams) == 10 * 8 + 8 + 8
    assert C.sizeof(_ffi.SgsWorkspace) == 8 + 8 + 8 + 4 * 4 + 8
    assert C.sizeof(_ffi.SgsStats) == 8 * 8


def _ws(n=1000, L=3, W=256, H=256, cap=1 << 16, mode=0):
    w = _ffi.SgsWorkspace()
    w.n, w.n_lobes, w.width, w.height, w.sort_mode, w.entry_capacity = n, L, W, H, mode, cap
    return w


def test_workspace_size_is_deterministic_and_monotone():
    lib = _ffi.load()
    sizes = []
    for cap in (1 << 10, 1 << 16, 1 << 20):
        b = C.c_uint64()
        assert lib.sgs_workspace_size(C.byref(_ws(cap=cap)), C.byref(b)) == 0
        sizes.append(b.value)
    assert sizes[0] < sizes[1] < sizes[2]
    b1, b2 = C.c_uint64(), C.c_uint64()
    lib.sgs_workspace_size(C.byref(_ws(mode=0)), C.byref(b1))
    lib.sgs_workspace_size(C.byref(_ws(mode=1)), C.byref(b2))
    assert b2.value > b1.value  # 64-bit keys need more room than 16-bit tile keys


@pytest.mark.parametrize("bad", [dict(n=-1), dict(W=0), dict(L=9), dict(mode=7), dict(cap=1 << 31)])
def test_workspace_rejects_bad_descriptors(bad):
    kw = dict(n=10, L=3, W=64, H=64, cap=100, mode=0)
    kw.update(bad)
    b = C.c_uint64()
    rc = _ffi.load().sgs_workspace_size(C.byref(_ws(**kw)), C.byref(b))
    assert rc == _ffi.SGS_E_ARG
    assert b"invalid" in _ffi.load().sgs_last_error()


def test_null_and_mismatched_arguments_fail_without_touching_the_device():
    lib = _ffi.load()
    p = _ffi.SgsParams()
    p.n, p.n_lobes = 5, 3  # null arrays
    cam = to_sgs(Camera.look_at((0, -3, 0), (0, 0, 0), width=64, height=64))
    ws = _ws(n=5, W=64, H=64)
    ws.base, ws.bytes = 1, 1  # too small -> rejected before any CUDA call
    assert lib.sgs_preprocess(C.byref(p), C.byref(cam), C.byref(ws), None) == _ffi.SGS_E_WORKSPACE
    g = _ffi.SgsGrads()
    assert lib.sgs_preprocess_backward(C.byref(p), C.byref(cam), None, C.byref(g), None) == _ffi.SGS_E_ARG
    bad = to_sgs(Camera.look_at((0, -3, 0), (0, 0, 0), width=64, height=64), tile_rows=(3, 2))
    assert lib.sgs_project_records(C.byref(p), C.byref(bad), None, None) == _ffi.SGS_E_ARG


def test_loss_entry_validates_before_touching_the_device():
    lib = _ffi.load()
    nb = C.c_uint64()
    assert lib.sgs_loss_workspace_size(720, 1280, C.byref(nb)) == _ffi.SGS_OK
    # three float64 planes + one (l1, ssim) slot pair per block for the
    # fixed-order loss reduction
    assert 3 * 720 * 1280 * 3 * 8 < nb.value <= 3 * 720 * 1280 * 3 * 8 + 2 * 8 * 4096
    assert lib.sgs_loss_workspace_size(0, 4, C.byref(nb)) == _ffi.SGS_E_ARG
    cfg = _ffi.SgsLossConfig(0.2, 10, 1.5, 1e-4, 9e-4)  # even window
    out = C.c_void_p(1)
    assert lib.sgs_image_loss(1, 0, 1, 0, 4, 4, C.byref(cfg), None, None, None, out, 1, 1 << 20,
                              None) == _ffi.SGS_E_ARG
    cfg.window = 11
    assert lib.sgs_image_loss(1, 0, 1, 0, 4, 4, C.byref(cfg), None, None, None, out, 1, 8,
                              None) == _ffi.SGS_E_WORKSPACE


def test_camera_conventions_match_reference():
    cam = Camera.look_at(eye=(0.0, -2.5, 0.3), target=(0, 0, 0), width=16, height=16, fx=20)
    R = cam.rotation
    np.testing.assert_allclose(R @ R.T, np.eye(3), atol=1e-12)
    np.testing.assert_allclose(cam.center, [0.0, -2.5, 0.3], atol=1e-12)
    fwd = -np.asarray(cam.center) / np.linalg.norm(cam.center)
    np.testing.assert_allclose(R[2], fwd, atol=1e-12)   # rows: right, down, forward
    assert cam.cx == 8.0 and cam.fy == 20
    with pytest.raises(ValueError):
        Camera(rotation=np.eye(3), translation=np.zeros(3), fx=0, fy=1, cx=0, cy=0, width=4, height=4)
    with pytest.raises(ValueError):
        Camera(rotation=np.eye(3), translation=np.zeros(3), fx=1, fy=1, cx=0, cy=0, width=0, height=4)
    c2 = cam.crop(3, 5, 8, 4)
    assert (c2.width, c2.height, c2.cx, c2.cy) == (8, 4, cam.cx - 3, cam.cy - 5)


def test_scene_generators_are_seeded_and_match_configs():
    s0, cams0 = scenes.config0()
    s0b, _ = scenes.config0()
    for f in scenes.FIELDS:
        assert np.array_equal(getattr(s0, f), getattr(s0b, f))
        assert getattr(s0, f).dtype == np.float32
    assert s0.n == 10_000 and cams0[0].width == 256
    assert cams0[0].fy == pytest.approx(128 / np.tan(np.radians(30)), rel=1e-12)  # 221.70
    s1, c1 = scenes.config1(n=5000)
    assert 0.55 < s1.prim_mask.mean() < 0.65
    k = s1.lobe_mask.sum(1)
    assert set(np.unique(k)) <= {0, 1, 2, 3}
    assert np.all(np.diff(s1.lobe_mask, axis=1) <= 0)  # lobe l active iff l < K
    assert (c1[0].width, c1[0].height) == (1280, 720)
    s3, c3 = scenes.config3(n=1000)
    assert len(c3) == 8 and s3.extra["prim_logit"].shape == (1000,)
    _, c2 = scenes.config2(n=1000)
    assert len(c2) == 64 and c2[0].width == 1920


def test_scene_params_from_scene_packs_like_the_reference():
    from paper_2509_07021_b200.render import ColorModelError, SceneParams

    class Lobe:
        def __init__(self, a, s, amp):
            self.axis, self.sharpness, self.amplitude = np.float32(a), s, np.float32(amp)

    class Prim:
        def __init__(self, n_lobes):
            self.position = np.float32([1, 2, 3])
            self.rotation = np.float32([1, 0, 0, 0])
            self.scale = np.float32([0.5, 0.25, 2.0])
            self.opacity = 0.25
            self.diffuse = np.float32([0.1, 0.2, 0.3])
            self.lobes = [Lobe([0, 1, 0], 2.0 + j, [0.1, 0, 0]) for j in range(n_lobes)]

    class CM:
        kind, max_lobes = "sg", 3

    class Scene:
        primitives = [Prim(0), Prim(2)]
        color_model = CM()

    p = SceneParams.from_scene(Scene())
    assert p.n == 2 and p.max_lobes == 3
    np.testing.assert_allclose(p.log_scale[0], np.log([0.5, 0.25, 2.0]))
    assert p.lobe_mask.tolist() == [[False] * 3, [True, True, False]]
    np.testing.assert_array_equal(p.axis_raw[0, :, 2], 1.0)  # placeholder axis for padded slots
    assert p.sharpness[1, 1] == 3.0

    class SH:
        kind, max_lobes = "sh", 0

    class Bad:
        primitives = []
        color_model = SH()

    with pytest.raises(ColorModelError):
        SceneParams.from_scene(Bad())


def test_view_sharding_covers_every_view_once():
    for world in (1, 2, 3, 4, 8):
        got = sorted(v for r in range(world) for v in shard_views(64, r, world))
        assert got == list(range(64))


def test_balanced_strips_partition_rows():
    rng = np.random.default_rng(0)
    for world in (1, 2, 4, 8):
        cost = rng.gamma(2.0, size=135)
        cost[60:80] *= 20  # a dense band
        strips = balanced_strips(cost, world)
        assert strips[0][0] == 0 and strips[-1][1] == 135
        assert all(a < b for a, b in strips)
        assert all(strips[i][1] == strips[i + 1][0] for i in range(world - 1))
        loads = [cost[a:b].sum() for a, b in strips]
        assert max(loads) <= cost.sum() / world + cost.max() + 1e-9


def test_row_costs_spread_counts_over_rows():
    rect = np.array([[0, (0) | (2 << 16)], [0, 5 | (5 << 16)], [0, 0]], np.uint32)
    tt = np.array([6, 4, 0], np.uint32)
    c = row_costs_from_rects(rect, tt, 8)
    np.testing.assert_allclose(c, [2, 2, 2, 0, 0, 4, 0, 0])
