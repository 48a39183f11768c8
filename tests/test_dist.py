"""CPU, world_size 2 (gloo): the data-parallel training step's gradient
all-reduce, and view / strip sharding, with the CPU oracle standing in for
the CUDA per-view gradients (the collective and bookkeeping are what is
under test; the per-view math is covered by the GPU parity tests)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_07021_b200 import scenes
from paper_2509_07021_b200.sharding import GradBucket, shard_views
from paper_2509_07021_b200.train import SoftPruneTrainer, TrainConfig


def _oracle_grad_fn(g, cam, target):
    from oracle import ref_dense, tiled

    arrays = scenes.SceneArrays(*(g.__dict__[f].numpy() for f in scenes.FIELDS),
                                lobe_mask=g.lobe_mask.numpy(), prim_mask=g.prim_mask.numpy())
    r = tiled.render(arrays, cam)
    val, dimg = ref_dense.loss_and_dimg(r.img.astype(np.float64), np.asarray(target), 0.2)
    tiled.raster_backward(r, dimg)
    out = tiled.preprocess_backward(r)
    return val, {k: torch.from_numpy(v.astype(np.float32)) for k, v in out.items()}


def _setup():
    scene, cams = scenes.config3(n=300, n_views=4)
    cams = [c.crop(600, 330, 48, 40) for c in cams]
    targets = [scenes.target_image(0, c.height, c.width, v) for v, c in enumerate(cams)]
    return scene, cams, targets


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    scene, cams, targets = _setup()
    tr = SoftPruneTrainer(scene, scene.extra["prim_logit"], scene.extra["lobe_logit"],
                          TrainConfig(), device="cpu", grad_fn=_oracle_grad_fn)
    assert tr.chunks == 4 and tr.bucket.chunks == 4   # bucketed, per-chunk async all-reduce
    loss = tr.step(cams, targets, rank=rank, world=world, apply=False)
    grads = {k: v.clone().numpy() for k, v in tr.grads().items()}
    tr.step(cams, targets, rank=rank, world=world, apply=True)
    params = {k: v.clone().numpy() for k, v in tr.params.items()}
    params["prim_logit"] = tr.prim_logit.clone().numpy()
    q.put((rank, loss, grads, params))
    dist.barrier()
    dist.destroy_process_group()


def test_grad_allreduce_matches_single_process():
    scene, cams, targets = _setup()
    single = SoftPruneTrainer(scene, scene.extra["prim_logit"], scene.extra["lobe_logit"],
                              TrainConfig(), device="cpu", grad_fn=_oracle_grad_fn)
    loss1 = single.step(cams, targets, apply=False)
    ref = {k: v.clone().numpy() for k, v in single.grads().items()}
    single.step(cams, targets, apply=True)
    ref_params = {k: v.clone().numpy() for k, v in single.params.items()}
    ref_params["prim_logit"] = single.prim_logit.clone().numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, loss, grads, params in res:
        assert loss == pytest.approx(loss1, rel=1e-6)
        for k, v in ref.items():
            np.testing.assert_allclose(grads[k], v, rtol=1e-5, atol=1e-9 * max(1.0, np.abs(v).max()))
        for k, v in ref_params.items():   # the chunk-by-chunk update equals the one-bucket update
            np.testing.assert_allclose(params[k], v, rtol=1e-6, atol=1e-7)
    assert np.abs(ref["position"]).max() > 0 and np.abs(ref["prim_logit"]).max() > 0


def test_bucket_roundtrip_and_average():
    b = GradBucket({"a": (3, 2), "b": (4,)}, "cpu")
    b.add_({"a": torch.ones(3, 2), "b": torch.arange(4.0)})
    b.add_({"a": torch.ones(3, 2)})
    b.allreduce_(average_over=2.0)
    assert torch.equal(b.view("a"), torch.ones(3, 2))
    assert torch.equal(b.view("b"), torch.arange(4.0) / 2)
    assert b.numel == 12  # each view starts on a 16-byte boundary: 6 -> 8, + 4


def test_chunked_bucket_layout():
    """Chunk-major bucket: every chunk is one contiguous all-reduce unit and
    holds every field's rows of its primitive range, 16-byte aligned."""
    shapes = {"position": (10, 3), "quat": (10, 4), "opacity": (10,), "lobe": (10, 3)}
    b = GradBucket(shapes, "cpu", chunks=3, n=10)
    assert b.bounds == [(0, 4), (4, 8), (8, 10)]
    g = {k: torch.randn(shp) for k, shp in shapes.items()}
    b.add_(g)
    back = b.as_dict()
    assert all(torch.equal(back[k], g[k]) for k in shapes)
    for c in range(3):
        flat = b.chunk_flat(c)
        assert flat.numel() == b.chunk_off[c + 1] - b.chunk_off[c]
        for k in shapes:
            v = b.chunk_view(k, c)
            assert v.data_ptr() % 16 == 0 and flat.data_ptr() <= v.data_ptr() < flat.data_ptr() + 4 * flat.numel()
    with pytest.raises(ValueError):
        b.view("position")


def test_strip_sharding_reassembles_the_frame_cpu_oracle():
    """Tile strips rendered independently (as N ranks would) tile the frame
    exactly: the oracle restatement of the GPU strip contract."""
    from oracle import tiled

    scene, cams = scenes.config0(n=3000)
    cam = cams[0]
    full = tiled.render(scene, cam).img
    parts = np.zeros_like(full)
    for y0, y1 in [(0, 4), (4, 9), (9, 16)]:
        r = tiled.render(scene, cam, tile_rows=(y0, y1))
        parts[y0 * 16:y1 * 16] = r.img[y0 * 16:y1 * 16]
    assert np.array_equal(full, parts)
    assert sorted(sum((shard_views(64, r, 8) for r in range(8)), [])) == list(range(64))


def test_strip_plan_refinement_equalises_measured_times():
    """sharding.refine_row_costs: a strip plan re-balanced from measured strip
    times (each strip's rows rescaled to its time) equalises a cost the
    per-row model did not see -- here a fixed cost per strip plus a
    quadratic per-row term."""
    from paper_2509_07021_b200.sharding import balanced_strips, refine_row_costs
    rows = 135
    model = np.ones(rows)                       # what the planner believes
    truth = 0.2 + 4.0 * (np.arange(rows) / rows - 0.5) ** 2

    def measure(plan):
        return [0.3 + truth[y0:y1].sum() for y0, y1 in plan]   # + a per-strip constant
    plan = balanced_strips(model, 8)
    t0 = measure(plan)
    cost = model
    for _ in range(3):
        cost = refine_row_costs(cost, plan, measure(plan))
        plan = balanced_strips(cost, 8)
    t1 = measure(plan)
    assert max(t1) / min(t1) < max(t0) / min(t0)
    assert max(t1) < max(t0)
    assert plan[0][0] == 0 and plan[-1][1] == rows and all(a[1] == b[0] for a, b in zip(plan, plan[1:]))
