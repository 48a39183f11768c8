"""Predicted multi-GPU efficiency from 1-GPU measurements (no multi-GPU box
is available to this build): each rank's share of the work is timed on one
B200 exactly as that rank would run it, the slowest rank sets the step time.

  configs[2]  64 views, rank r renders 64/N of them (8 streams, graphs)
  configs[3]  8-view training step, rank r runs 8/N views + the bucket
              all-reduce (modelled: 2 (N-1)/N x bucket bytes / busbw)
  configs[4]  profiles/strips (per-strip stage times, measured-cost strips)

  python profiles/predict_scaling.py > profiles/r02_predicted_scaling.json
"""
import gc
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_07021_b200 import scenes  # noqa: E402
from paper_2509_07021_b200.rasterizer import GaussianTensors, Rasterizer  # noqa: E402
from paper_2509_07021_b200.train import SoftPruneTrainer  # noqa: E402

NVLINK_BUSBW_GBS = 360.0  # conservative NCCL all-reduce bus bandwidth for a 78 MB bucket on NVLink 5 (assumed)
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
gc.collect()
gc.disable()  # no collection pauses inside the event-timed shares
out = {"assumptions": {"allreduce_busbw_GBs": NVLINK_BUSBW_GBS}}

# ---- configs[2]
scene, cams = scenes.config2()
rast = Rasterizer()
g = GaussianTensors.from_arrays(scene)
NSTREAMS = 8
streams = [torch.cuda.current_stream()] + [torch.cuda.Stream() for _ in range(NSTREAMS - 1)]
for k, c in enumerate(cams):
    rast.forward(g, c, check=True, track=False)
bufs = [(torch.empty((c.height, c.width, 3), device="cuda"), torch.empty((c.height, c.width), device="cuda"))
        for c in cams]


def render(views, reps=5):
    main = streams[0]

    def step():
        for j, v in enumerate(views):
            with torch.cuda.stream(streams[j % NSTREAMS]):
                rast.graph_forward(g, cams[v], bufs[v])
    for s in streams[1:]:
        s.wait_stream(main)
    step()
    for s in streams[1:]:
        main.wait_stream(s)
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record(main)
    for s in streams[1:]:
        s.wait_stream(main)
    for _ in range(reps):
        step()
    for s in streams[1:]:
        main.wait_stream(s)
    b.record(main)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


c2 = {}
t1 = render(list(range(64)))
for n in (1, 2, 4, 8):
    tn = max(render(list(range(r, 64, n))) for r in range(n)) if n > 1 else t1
    c2[n] = {"step_ms": tn, "fps": 64 / (tn / 1e3), "efficiency": t1 / tn / n}
out["configs[2]"] = c2
del g, rast, bufs

# ---- configs[3]
scene, cams = scenes.config3()
dev = torch.device("cuda")
targets = [torch.from_numpy(scenes.target_image(0, c.height, c.width, v)).to(dev) for v, c in enumerate(cams)]
tr = SoftPruneTrainer(scene, scene.extra["prim_logit"], scene.extra["lobe_logit"], device=dev)
tr.graph_tail = False   # a multi-rank step replays the views' graph; its all-reduce and update stay eager
bucket_bytes = tr.bucket.numel * 4
c3 = {}
base = None
for n in (1, 2, 4, 8):
    mine = list(range(0, 8, n))    # rank 0's share (round-robin); shares are equal-sized
    sub_c, sub_t = [cams[v] for v in mine], [targets[v] for v in mine]
    for _ in range(3):
        tr.step(sub_c, sub_t, graph=True)
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record()
    for _ in range(5):
        tr.step(sub_c, sub_t, sync=False, graph=True)
    b.record()
    torch.cuda.synchronize()
    comp = a.elapsed_time(b) / 5
    ar = 0.0 if n == 1 else 2 * (n - 1) / n * bucket_bytes / (NVLINK_BUSBW_GBS * 1e9) * 1e3
    tn = comp + ar
    base = base or tn
    c3[n] = {"compute_ms": comp, "allreduce_ms_model": ar, "step_ms": tn, "views_per_s": 8 / (tn / 1e3),
             "efficiency": base / tn / n}
out["configs[3]"] = c3
out["configs[3]"]["bucket_bytes"] = bucket_bytes
print(json.dumps(out, indent=1))
