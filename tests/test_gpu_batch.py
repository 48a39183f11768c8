"""Host-buffer batch API (batch.py): pinned uploads into two device copies,
renders spread over streams, read-backs on a copy stream.  Every image must
equal the single-view render of the scene that call uploaded."""

import numpy as np
import pytest
import torch

from paper_2509_07021_b200 import scenes
from paper_2509_07021_b200.batch import BatchRenderer, PinnedScene
from paper_2509_07021_b200.rasterizer import GaussianTensors, Rasterizer

pytestmark = pytest.mark.gpu


def _reference_images(scene, cams):
    rast = Rasterizer()
    g = GaussianTensors.from_arrays(scene)
    return [rast.forward(g, c, track=False).img.cpu().numpy().copy() for c in cams]


def test_render_views_matches_single_view_renders():
    scene, cams = scenes.config1(n=20_000)
    cams = [c.crop(0, 0, 320, 180) for c in cams[:1]] * 3
    want = _reference_images(scene, cams)
    br = BatchRenderer(streams=2)
    got = br.render_views(PinnedScene(scene), cams)
    for a, b in zip(got, want):
        assert np.array_equal(a.numpy(), b)


def test_pipelined_calls_render_their_own_scene():
    sa, cams = scenes.config1(n=20_000, seed=0)
    sb, _ = scenes.config1(n=20_000, seed=1)
    cams = [cams[0].crop(100, 50, 256, 128), cams[0].crop(0, 0, 200, 100)]
    wa, wb = _reference_images(sa, cams), _reference_images(sb, cams)
    br = BatchRenderer(streams=3)
    pa, pb = PinnedScene(sa), PinnedScene(sb)
    snaps = []
    for k in range(5):
        outs = br.render_views(pa if k % 2 == 0 else pb, cams, wait=False)
        if k >= 3:
            torch.cuda.synchronize()
            snaps.append([o.numpy().copy() for o in outs])
    # calls 3 (scene b) and 4 (scene a)
    for got, want in zip(snaps, (wb, wa)):
        for a, b in zip(got, want):
            assert np.array_equal(a, b)


def test_graph_forward_replays_current_scene():
    """A captured view re-reads the scene buffers at every replay."""
    scene, cams = scenes.config1(n=20_000)
    cam = cams[0].crop(200, 100, 320, 200)
    rast = Rasterizer()
    g = GaussianTensors.from_arrays(scene)
    out = (torch.empty((200, 320, 3), device="cuda"), torch.empty((200, 320), device="cuda"))
    rast.graph_forward(g, cam, out)
    want = rast.forward(g, cam, track=False).img
    assert torch.equal(out[0], want)
    g.diffuse.mul_(0.5)  # in-place parameter update, same buffers
    rast.graph_forward(g, cam, out)
    want2 = rast.forward(g, cam, track=False).img
    assert torch.equal(out[0], want2) and not torch.equal(want, want2)


def _denser(scene, by=1.5):
    """Same primitive count (same workspace key), much larger splats."""
    d = scenes.SceneArrays(**{f: getattr(scene, f).copy() for f in scenes.FIELDS},
                           lobe_mask=scene.lobe_mask.copy(), prim_mask=scene.prim_mask)
    d.log_scale += np.float32(by)
    return d


def test_denser_scene_after_capture_is_rerendered_not_truncated():
    """VERDICT r1 item 2 / ADVICE: graphs captured for a sparse scene must not
    replay into a freed workspace or return truncated images when a denser
    scene (same N, same cameras) is uploaded into the same slot."""
    sparse, cams = scenes.config1(n=20_000)
    dense = _denser(sparse)
    cams = [cams[0].crop(320, 180, 640, 360), cams[0].crop(0, 0, 480, 272)]
    want_sparse, want_dense = _reference_images(sparse, cams), _reference_images(dense, cams)
    rast = Rasterizer()
    br = BatchRenderer(rast, streams=2)
    ps, pd = PinnedScene(sparse), PinnedScene(dense)
    for a, b in zip(br.render_views(ps, cams), want_sparse):
        assert np.array_equal(a.numpy(), b)
    # same slot (call 2) holds the dense scene: its captured graphs overflow
    br.render_views(ps, cams)
    got = [o.numpy().copy() for o in br.render_views(pd, cams)]
    assert br.rerendered > 0
    for a, b in zip(got, want_dense):
        assert np.array_equal(a, b)
    # pipelined calls alternate densities; every image is final after finish()
    snaps = []
    for k in range(4):
        snaps.append(br.render_views(pd if k % 2 else ps, cams, wait=False))
    br.finish()
    for k in (2, 3):
        want = want_dense if k % 2 else want_sparse
        for a, b in zip(snaps[k], want):
            assert np.array_equal(a.numpy(), b)


def test_graph_replay_reports_overflow_and_recaptures_after_growth():
    sparse, cams = scenes.config1(n=20_000)
    dense = _denser(sparse)
    cam = cams[0].crop(320, 180, 640, 360)
    rast = Rasterizer()
    g = GaussianTensors.from_arrays(sparse)
    out = (torch.empty((360, 640, 3), device="cuda"), torch.empty((360, 640), device="cuda"))
    ovf = rast.graph_forward(g, cam, out)
    assert int(ovf[0]) == 0
    gd = GaussianTensors.from_arrays(dense)
    for f in scenes.FIELDS:  # in-place upload of the denser scene into the captured buffers
        getattr(g, f).copy_(getattr(gd, f))
    ovf = rast.graph_forward(g, cam, out)
    torch.cuda.synchronize()
    assert int(ovf[0]) != 0, "the captured capacity should overflow on the denser scene"
    rast.grow_capacity(g, cam, int(ovf[1]))
    ovf = rast.graph_forward(g, cam, out)  # recaptured against the grown workspace
    torch.cuda.synchronize()
    assert int(ovf[0]) == 0
    want = rast.forward(g, cam, track=False, check=True).img
    assert torch.equal(out[0], want)


def test_graph_cache_is_bounded():
    """Captured graphs hold their buffers alive; the cache keeps the most
    recently replayed max_graphs and replays stay correct after eviction."""
    scene, cams = scenes.config1(n=5_000)
    views = [cams[0].crop(64 * k, 0, 64, 64) for k in range(6)]
    rast = Rasterizer(max_graphs=4)
    g = GaussianTensors.from_arrays(scene)
    outs = [(torch.empty((64, 64, 3), device="cuda"), torch.empty((64, 64), device="cuda")) for _ in views]
    for _ in range(2):
        for v, o in zip(views, outs):
            rast.graph_forward(g, v, o)
    torch.cuda.synchronize()
    assert len(rast._graphs) == 4
    for v, o in zip(views, outs):
        assert torch.equal(o[0], rast.forward(g, v, track=False).img)


def test_staged_upload_matches_numpy_conversion_and_alignment():
    """GaussianTensors.from_arrays narrows host float64 arrays through one
    pinned arena (rasterizer._PinnedArena): the same float32 values as
    numpy's astype, every field 256-byte aligned (the kernels' float4 loads),
    and the float64 download is exact."""
    from paper_2509_07021_b200 import render as R
    from paper_2509_07021_b200.rasterizer import GRAD_FIELDS, device_to_host_f64
    scene, _ = scenes.config0(n=1001)   # odd sizes: offsets must be padded
    p = R.SceneParams(**{f: getattr(scene, f).astype(np.float64) + 1e-9 for f in scenes.FIELDS},
                      lobe_mask=scene.lobe_mask)
    g = GaussianTensors.from_arrays(p)
    for f in GRAD_FIELDS + ("lobe_mask",):
        t = getattr(g, f)
        assert t.data_ptr() % 256 == 0, f
        assert np.array_equal(t.cpu().numpy(), np.asarray(getattr(p, f), dtype=np.float32)), f
    x = torch.rand((300, 400, 3), device="cuda")
    assert np.array_equal(device_to_host_f64(x), x.cpu().numpy().astype(np.float64))
