"""GPU: the configs[3] training step (soft pruning, L1 + SSIM, multi-view)
runs through the CUDA path, its gradients match the CPU oracle, and a few
steps reduce the loss."""

import numpy as np
import pytest
import torch

from helpers import composite_ok
from paper_2509_07021_b200 import scenes
from paper_2509_07021_b200.train import SoftPruneTrainer, TrainConfig

pytestmark = pytest.mark.gpu


def _setup(n=3000, views=4):
    scene, cams = scenes.config3(n=n, n_views=views)
    cams = [c.crop(560, 300, 160, 120) for c in cams]
    targets = [torch.from_numpy(scenes.target_image(0, c.height, c.width, v)).cuda().double()
               for v, c in enumerate(cams)]
    return scene, cams, targets


def test_train_step_gradients_match_oracle():
    from oracle import ref_dense, tiled
    scene, cams, targets = _setup()
    tr = SoftPruneTrainer(scene, scene.extra["prim_logit"], scene.extra["lobe_logit"],
                          TrainConfig(lambda_mask=0.0))
    tr.step(cams, targets, apply=False)
    gpu = {k: v.cpu().numpy() for k, v in tr.grads().items()}
    acc = {}
    for cam, t in zip(cams, targets):
        r = tiled.render(scene, cam)
        _, dimg = ref_dense.loss_and_dimg(r.img.astype(np.float64), t.cpu().numpy(), 0.2)
        tiled.raster_backward(r, dimg)
        for k, v in tiled.preprocess_backward(r).items():
            acc[k] = acc.get(k, 0) + v / len(cams)
    m_p = 1 / (1 + np.exp(-scene.extra["prim_logit"].astype(np.float64)))
    m_l = 1 / (1 + np.exp(-scene.extra["lobe_logit"].astype(np.float64)))
    acc["prim_logit"] = acc.pop("prim_mask") * m_p * (1 - m_p)
    acc["lobe_logit"] = acc.pop("lobe_mask") * m_l * (1 - m_l)
    for k, v in acc.items():
        ok = composite_ok(gpu[k], v, floor=2e-5)
        assert ok.mean() == 1.0, f"{k}: {np.count_nonzero(~ok)}"


def test_train_steps_reduce_loss():
    scene, cams, targets = _setup(n=2000, views=2)
    tr = SoftPruneTrainer(scene, scene.extra["prim_logit"], scene.extra["lobe_logit"], TrainConfig())
    losses = [tr.step(cams, targets) for _ in range(6)]
    assert losses[-1] < losses[0]
    assert all(np.isfinite(losses))


def test_step_redoes_views_that_outgrow_capacity():
    """A deliberately tiny tile-entry capacity: the deferred per-step check
    grows it and redoes the step, matching a step with ample capacity."""
    import numpy as np
    import torch
    from paper_2509_07021_b200 import scenes
    from paper_2509_07021_b200.rasterizer import Rasterizer
    from paper_2509_07021_b200.train import SoftPruneTrainer
    scene, cams = scenes.config3(n=3000, n_views=2)
    cams = [c.crop(400, 200, 256, 160) for c in cams]
    tg = [torch.from_numpy(scenes.target_image(0, c.height, c.width, v)).cuda() for v, c in enumerate(cams)]
    out = []
    for cap in (64, None):
        tr = SoftPruneTrainer(scene, scene.extra["prim_logit"], scene.extra["lobe_logit"])
        tr.rast = Rasterizer(initial_capacity=cap)
        loss = tr.step(cams, tg, apply=False)
        out.append((loss, {k: v.clone() for k, v in tr.grads().items()}))
    assert out[0][0] == pytest.approx(out[1][0], rel=1e-6)
    for k in out[0][1]:
        np.testing.assert_allclose(out[0][1][k].cpu().numpy(), out[1][1][k].cpu().numpy(), rtol=1e-4, atol=1e-7)


def test_backward_accumulate_and_mask_logit_flags():
    """SGS_GRADS_ACCUMULATE adds into the outputs; SGS_GRADS_MASK_LOGIT takes
    the mask gradients through the sigmoid (x m (1 - m))."""
    from paper_2509_07021_b200.rasterizer import GRAD_FIELDS, GaussianTensors, Rasterizer
    scene, cams, targets = _setup(n=3000, views=1)
    g = GaussianTensors.from_arrays(scene)
    g.prim_mask = torch.sigmoid(torch.as_tensor(scene.extra["prim_logit"], device="cuda")).float().contiguous()
    g.lobe_mask = torch.sigmoid(torch.as_tensor(scene.extra["lobe_logit"], device="cuda")).float().contiguous()
    rast = Rasterizer()
    fr = rast.forward(g, cams[0])
    dimg = torch.randn_like(fr.img)
    ref = rast.backward(g, fr, dimg, mask_grads=True)
    acc = {f: torch.full_like(ref[f], 0.5) for f in GRAD_FIELDS + ("lobe_mask", "prim_mask")}
    # (float4 quaternion rows need 16-byte alignment; fresh torch allocations have it)
    rast.backward(g, fr, dimg, mask_grads=True, out=acc, accumulate=True, mask_logit=True)
    rast.backward(g, fr, dimg, mask_grads=True, out=acc, accumulate=True, mask_logit=True)
    # the raster's float atomics sum in a different order on every call
    for f in GRAD_FIELDS:
        want = 0.5 + 2 * ref[f]
        assert torch.allclose(acc[f], want, rtol=1e-4, atol=1e-5 * float(ref[f].abs().max())), f
    for f in ("lobe_mask", "prim_mask"):
        m = getattr(g, f)
        want = 0.5 + 2 * ref[f] * m * (1 - m)
        assert torch.allclose(acc[f], want, rtol=1e-4, atol=1e-5 * float(ref[f].abs().max())), f
    with pytest.raises(ValueError):
        rast.backward(g, fr, dimg, accumulate=True)


def test_chunked_bucket_step_equals_single_bucket():
    """The bucketed step (K7 per primitive range into a chunk-major bucket,
    chunk-by-chunk reduction and update -- the multi-rank path, forced on one
    rank) gives the single-bucket step's gradients and parameters."""
    scene, cams, targets = _setup(n=3001, views=4)
    a = SoftPruneTrainer(scene, scene.extra["prim_logit"], scene.extra["lobe_logit"], TrainConfig())
    b = SoftPruneTrainer(scene, scene.extra["prim_logit"], scene.extra["lobe_logit"], TrainConfig(),
                         comm_chunks=3, chunk_single_rank=True)
    assert b.chunks == 3
    la = a.step(cams, targets, apply=False)
    lb = b.step(cams, targets, apply=False)
    assert la == pytest.approx(lb, rel=1e-9)
    ga, gb = a.grads(), b.grads()
    for k in ga:
        ref = ga[k].double()
        assert torch.allclose(gb[k].double(), ref, rtol=1e-5, atol=1e-6 * float(ref.abs().max())), k
    a.step(cams, targets)
    b.step(cams, targets)
    for k in a.params:
        assert torch.allclose(a.params[k], b.params[k], rtol=1e-5, atol=1e-6), k


@pytest.mark.parametrize("views,tail", [(1, True), (3, True), (3, False)])
def test_graph_step_equals_eager_step(views, tail):
    """step(graph=True): the views' device work replayed from a CUDA graph
    (captured after an eager step sized the workspaces) gives the eager
    step's losses and parameters, and recaptures when the capacity grows."""
    scene, cams, targets = _setup(n=3000, views=views)
    a = SoftPruneTrainer(scene, scene.extra["prim_logit"], scene.extra["lobe_logit"], TrainConfig())
    b = SoftPruneTrainer(scene, scene.extra["prim_logit"], scene.extra["lobe_logit"], TrainConfig())
    b.graph_tail = tail                              # False: reduction and update eager (multi-rank form)
    la = [a.step(cams, targets) for _ in range(4)]
    lb = [b.step(cams, targets, graph=True) for _ in range(4)]
    assert b._gstep is not None                      # steps 2-4 replayed the graph
    np.testing.assert_allclose(lb, la, rtol=1e-6)
    for k in a.params:
        assert torch.allclose(a.params[k], b.params[k], rtol=1e-5, atol=1e-6), k
    # a denser scene in the same buffers overflows the captured capacity: the
    # step redoes itself eagerly, then recaptures
    for f in ("log_scale",):
        b.params[f].add_(1.0)
        a.params[f].add_(1.0)
    la2 = a.step(cams, targets)
    lb2 = b.step(cams, targets, graph=True)
    assert lb2 == pytest.approx(la2, rel=1e-6)
    for k in a.params:
        assert torch.allclose(a.params[k], b.params[k], rtol=1e-5, atol=1e-6), k
