"""configs[4]: per-strip stage times (CUDA events, one stream) of the 1/2/4/8-rank
partitions (CUDA events, one stream) -> predicted strong-scaling efficiency."""
import json, sys
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_07021_b200 import scenes
from paper_2509_07021_b200.rasterizer import GaussianTensors, Rasterizer
from paper_2509_07021_b200.sharding import (balanced_strips, refine_row_costs, row_costs_from_rects,
                                            row_costs_measured)
scene, (cam,) = scenes.config4()
rast = Rasterizer()
g = GaussianTensors.from_arrays(scene)
_, rect, tt = rast.preprocess_only(g, cam)
ty = (cam.height + 15) // 16
ent = row_costs_from_rects(rect.cpu().numpy().view(np.uint32), tt.cpu().numpy().view(np.uint32), ty)
img = torch.empty((cam.height, cam.width, 3), device="cuda"); T = torch.empty((cam.height, cam.width), device="cuda")
ev = lambda: torch.cuda.Event(enable_timing=True)
e4 = [ev() for _ in range(4)]
for _ in range(2):
    full = rast.forward(g, cam, check=True, _events=e4)
torch.cuda.synchronize()
meas = row_costs_measured(full.ncontrib.cpu().numpy(), ent, e4[0].elapsed_time(e4[1]), e4[3].elapsed_time(e4[0]))
cost = meas if (len(sys.argv) < 2 or sys.argv[1] != "entries") else ent
# argv[2]: refinement rounds from measured strip times (default 2)
def time_strips(strips):
    per = []
    for (y0, y1) in strips:
        for _ in range(2):
            rast.forward(g, cam, check=True, tile_rows=(y0, y1), out=(img, T, None), track=False)
        reps = []
        for _ in range(3):
            e = [ev() for _ in range(4)]
            rast.forward(g, cam, check=False, tile_rows=(y0, y1), out=(img, T, None), track=False, _events=e)
            torch.cuda.synchronize()
            reps.append((e[2].elapsed_time(e[3]), e[3].elapsed_time(e[0]), e[0].elapsed_time(e[1])))
        p, b, r = np.median(np.array(reps), axis=0)
        st = rast.forward(g, cam, check=True, tile_rows=(y0, y1), out=(img, T, None), track=False).stats()
        per.append({"rows": [y0, y1], "prep_ms": p, "bin_ms": b, "raster_ms": r, "total_ms": p + b + r,
                    "emitting": st["n_emitting"], "entries": st["n_entries"]})
    return per


refine = int(sys.argv[2]) if len(sys.argv) > 2 else 2
res = {}
for world in (1, 2, 4, 8):
    c = cost
    strips = balanced_strips(c, world)
    per = time_strips(strips)
    for _ in range(refine if world > 1 else 0):  # re-plan from the measured strip times
        c = refine_row_costs(c, strips, [x["total_ms"] for x in per])
        strips = balanced_strips(c, world)
        per = time_strips(strips)
    res[world] = {"max_rank_ms": max(x["total_ms"] for x in per), "strips": per}
t1 = res[1]["max_rank_ms"]
for w in (1, 2, 4, 8):
    res[w]["predicted_speedup"] = t1 / res[w]["max_rank_ms"]
    res[w]["predicted_efficiency"] = t1 / res[w]["max_rank_ms"] / w
print(json.dumps(res))
