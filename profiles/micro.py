"""Quick per-variant measurements (CUDA events): configs[2] frames/s over 16
cameras on 4 streams with graphs, single-stream stage times, configs[3]
K6 ms/view and training views/s.  SGS_LIB selects the library."""
import json, os, sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_07021_b200 import scenes
from paper_2509_07021_b200.rasterizer import GaussianTensors, Rasterizer
from paper_2509_07021_b200.loss import image_loss
from paper_2509_07021_b200.render import LossConfig
from paper_2509_07021_b200.train import SoftPruneTrainer

what = sys.argv[1] if len(sys.argv) > 1 else "all"
out = {"lib": os.environ.get("SGS_LIB", "default")}
dev = torch.device("cuda")
ev = lambda: torch.cuda.Event(enable_timing=True)
if what in ("all", "render"):
    scene, cams = scenes.config2(n_cams=64)
    cams = cams[:16]
    rast = Rasterizer()
    g = GaussianTensors.from_arrays(scene)
    S = int(os.environ.get("MICRO_STREAMS", "8"))  # as bench.py
    streams = [torch.cuda.current_stream()] + [torch.cuda.Stream() for _ in range(S - 1)]
    for _ in range(3):
        for k, c in enumerate(cams):
            with torch.cuda.stream(streams[k % S]):
                rast.forward(g, c, check=True, track=False)
    torch.cuda.synchronize()
    bufs = [(torch.empty((c.height, c.width, 3), device=dev), torch.empty((c.height, c.width), device=dev)) for c in cams]
    def step():
        for k, c in enumerate(cams):
            with torch.cuda.stream(streams[k % S]):
                rast.graph_forward(g, c, bufs[k])
    main = streams[0]
    for s in streams[1:]: s.wait_stream(main)
    step()
    for s in streams[1:]: main.wait_stream(s)
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record(main)
    for s in streams[1:]: s.wait_stream(main)
    for _ in range(10): step()
    for s in streams[1:]: main.wait_stream(s)
    b.record(main)
    torch.cuda.synchronize()
    out["fps"] = 160 / (a.elapsed_time(b) / 1e3)
    evs = [[ev() for _ in range(4)] for _ in range(16)]
    for k, c in enumerate(cams):
        rast.forward(g, c, check=False, out=(*bufs[k], None), track=False, _events=evs[k])
    torch.cuda.synchronize()
    out["raster_ms"] = float(np.mean([e[0].elapsed_time(e[1]) for e in evs]))
    out["prep_ms"] = float(np.mean([e[2].elapsed_time(e[3]) for e in evs]))
    out["bin_ms"] = float(np.mean([e[3].elapsed_time(e[0]) for e in evs]))
if what in ("all", "train"):
    scene, cams = scenes.config3()
    targets = [torch.from_numpy(scenes.target_image(0, c.height, c.width, v)).to(dev) for v, c in enumerate(cams)]
    tr = SoftPruneTrainer(scene, scene.extra["prim_logit"], scene.extra["lobe_logit"], device=dev)
    for _ in range(3): tr.step(cams, targets, graph=True)
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record()
    for _ in range(5): tr.step(cams, targets, sync=False, graph=True)
    b.record()
    torch.cuda.synchronize()
    out["train_vps"] = 40 / (a.elapsed_time(b) / 1e3)
    g = tr.gaussians(); rast = tr.rast
    k6 = []
    for v, c in enumerate(cams):
        fr = rast.forward(g, c, check=True)
        _, dimg, _ = image_loss(fr.img, targets[v], LossConfig())
        for rep in range(3):  # the first launch of a view is not timed
            e0, e1 = ev(), ev()
            torch.cuda._sleep(2_000_000)  # the host enqueues while the GPU is busy
            e0.record(); rast.backward_raster(g, fr, dimg); e1.record()
            torch.cuda.synchronize()
            if rep:
                k6.append(e0.elapsed_time(e1))
    out["k6_ms"] = float(np.mean(k6))
print(json.dumps(out))
