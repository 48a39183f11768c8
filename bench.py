#!/usr/bin/env python
"""Benchmark: BASELINE.json metric "frames/s & Mpix/s at 1080p, 1M Gaussians,
3 SG lobes (1/2/4/8 B200); peak render VRAM" on configs[2].

  python bench.py [--gpus N] [--steps K] [--warmup W] [--views V] [--impl ours|reference]

One process per GPU (torchrun for N > 1).  A step = V forward renders per
rank of the config[2] scene (1M Gaussians, 3 lobes, 1920x1080): rank r renders
cameras (r*V + k) mod 64, Gaussians replicated, no collective on the data
path (weak scaling; at N=8, V=8 one step is exactly the 64-camera batch).
`value` = all ranks' frames / max-over-ranks device time.  `e2e` = the same
metric through the host-buffer batch API (pinned H2D of the scene + D2H of
every image inside the timed region).

--impl reference times the reference algorithm (dense float64 NumPy
restatement, oracle/ref_dense.py -- the reference package cannot travel to
the GPU box) on the host cores, rank 0 only, on bounded pixel samples of the
same workload, extrapolated to frames/s.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "frames/s & Mpix/s at 1080p, 1M Gaussians, 3 SG lobes (1/2/4/8 B200); peak render VRAM"
UNIT = "frames/s"
WORKLOAD = "configs[2]: 1,000,000 Gaussians (64 clusters), 3 SG lobes, 1920x1080, FoV 60"
# libsgs kernels per forward frame (depth-first mode, 1080p): preprocess (also
# accumulates the depth-digit histograms); 4 onesweep passes
# (depth sort); the one-pass offsets scan; emit_entries (also the cell
# histogram and the range reset); 1 onesweep pass (super-tile
# sort + ranges); cell_order, raster_fwd (profiles/r01_launches_v10.csv)
KERNELS_PER_FRAME = 10


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--views", type=int, default=8)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sort-mode", type=int, default=0)
    ap.add_argument("--streams", type=int, default=4,
                    help="concurrent CUDA streams the views of a step are spread over")
    ap.add_argument("--no-graphs", action="store_true",
                    help="launch every kernel from the host instead of replaying per-view CUDA graphs")
    ap.add_argument("--workload", default="render", choices=["render", "train", "stress"],
                    help="render: configs[2] headline; train: configs[3] training step; "
                         "stress: configs[4] 4K frame in tile strips")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.proc = None
        self.path = Path(f"/tmp/bench_clocks_{os.getpid()}.csv")
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"], stdout=self.fh,
                stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.path.read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() in ("active", "1"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(smax)),
                "reasons": sorted(reasons), "samples": len(sm)}


def profiled_traffic(kernel: str):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of
    `kernel` from the committed `ncu --set full` capture (profiles/traffic.json)."""
    p = ROOT / "profiles" / "traffic.json"
    if not p.exists():
        return None
    return json.loads(p.read_text()).get(kernel, {}).get("bytes_per_launch")


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


# --------------------------------------------------------------- CPU baseline
_CPU_STATE = {}


def _cpu_worker(job):
    """Blend a block of pixels against every visible primitive (reference
    algorithm, dense f64) using the parent's projection (fork, copy-on-write)."""
    from oracle import ref_dense
    px, py = job
    pr = _CPU_STATE["pr"]
    t = time.perf_counter()
    b = ref_dense._blend_block(pr, px, py)
    _ = b["w"].T @ pr.color
    return time.perf_counter() - t, px.size


def cpu_reference_rate(scene, cam, n_jobs: int, px_per_job: int = 4, procs: int | None = None):
    """Reference algorithm (dense f64 restatement of render.py) timed on the
    host: the per-frame preprocess of all primitives once, then `n_jobs`
    blocks of `px_per_job` random pixels blended in parallel over `procs`
    processes.  Returns (frames/s extrapolated to the full frame, details)."""
    import multiprocessing as mp

    from oracle import ref_dense
    procs = procs or cpu_procs()
    t = time.perf_counter()
    pr = ref_dense.project(scene, cam)
    t_prep = time.perf_counter() - t
    _CPU_STATE["pr"] = pr
    rng = np.random.default_rng(0)
    jobs = []
    for _ in range(n_jobs):
        xs = rng.integers(0, cam.width, size=px_per_job) + 0.5
        ys = rng.integers(0, cam.height, size=px_per_job) + 0.5
        jobs.append((xs.astype(np.float64), ys.astype(np.float64)))
    t = time.perf_counter()
    with mp.get_context("fork").Pool(procs) as pool:
        res = pool.map(_cpu_worker, jobs)
    wall = time.perf_counter() - t
    px = sum(r[1] for r in res)
    per_px = sum(r[0] for r in res) / px          # seconds per pixel on one core
    P = cam.width * cam.height
    frame_s = t_prep + P * per_px / procs
    return 1.0 / frame_s, dict(t_prep=t_prep, s_per_px_one_core=per_px, wall=wall, pixels=px,
                               cores=procs, frame_s=frame_s)


def cpu_procs() -> int:
    # all host threads, capped so the forked dense (V x block) float64 temporaries fit in RAM
    return max(1, min(os.cpu_count() or 1, 32))


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    from paper_2509_07021_b200 import scenes
    scene, cams = scenes.config2(n=args.n, n_cams=1)
    cam = cams[0]
    procs = cpu_procs()
    for _ in range(max(args.warmup, 0)):
        cpu_reference_rate(scene, cam, n_jobs=procs, procs=procs)
    rates, details = [], []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r, d = cpu_reference_rate(scene, cam, n_jobs=procs, procs=procs)
        rates.append(r)
        details.append(d)
    elapsed = time.perf_counter() - t0
    value = float(np.median(rates))
    sample = (f"per step: float64 dense restatement of the reference renderer (oracle/ref_dense.py): "
              f"preprocess of all {args.n} Gaussians for camera 0, then {procs} blocks of 4 random "
              f"pixels blended against every visible Gaussian in parallel over {procs} host "
              f"processes; frames/s extrapolated linearly to 1920x1080 (the reference blend is "
              f"exactly O(V*P))")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / max(args.steps, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded configs[2] distributions)", "impl": "reference",
            "config": {"workload": WORKLOAD, "sample": "4-pixel blocks"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "port",
                             "sample": sample, "s_per_px_one_core": float(np.median(
                                 [d["s_per_px_one_core"] for d in details])),
                             "preprocess_s": float(np.median([d["t_prep"] for d in details]))},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2509_07021_b200 import _ffi, scenes
    from paper_2509_07021_b200.batch import BatchRenderer, PinnedScene
    from paper_2509_07021_b200.rasterizer import GaussianTensors, Rasterizer

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    scene, cams64 = scenes.config2(n=args.n)
    V = args.views
    my_cams = [cams64[(rank * V + k) % len(cams64)] for k in range(V)]
    rast = Rasterizer(sort_mode=args.sort_mode, device=dev)
    torch.cuda.reset_peak_memory_stats(dev)
    g = GaussianTensors.from_arrays(scene, device=dev)
    torch.cuda.synchronize(dev)
    static_bytes = torch.cuda.memory_allocated(dev)

    # warm-up: size the tile-entry capacity on every camera this rank renders,
    # on every stream's workspace
    streams = [torch.cuda.current_stream(dev)] + [torch.cuda.Stream(device=dev)
                                                  for _ in range(max(args.streams, 1) - 1)]
    for _ in range(max(args.warmup, 3)):
        for k, cam in enumerate(my_cams):
            with torch.cuda.stream(streams[k % len(streams)]):
                rast.forward(g, cam, check=True)
    torch.cuda.synchronize(dev)
    stats = []
    pairs = torch.zeros(1, dtype=torch.int64, device=dev)
    for cam in my_cams:
        f = rast.forward(g, cam, check=True, pair_count=pairs, track=False)
        st = f.stats()
        assert not st["overflow"]
        stats.append(st)
    torch.cuda.synchronize(dev)
    pairs_per_view = float(pairs.item()) / V
    # reference VRAM model (3-sigma AABB, postprocess.py:101-137) on camera 0
    from paper_2509_07021_b200.camera import to_sgs
    import ctypes as C
    ws = rast.workspace(g, my_cams[0])
    _ffi.call("sgs_vram_model", C.byref(g.c_params()), C.byref(to_sgs(my_cams[0])), 16,
              C.byref(ws.desc), C.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    vs = ws.stats()
    model3s = 40 * vs["vram3s_visible"] + 12 * vs["vram3s_entries"]
    # per-frame dynamic render VRAM: one frame on a fresh workspace
    from paper_2509_07021_b200.postprocess import measured_render_vram
    frame_vram = measured_render_vram(g, my_cams[0], rast=rast)
    inflight_bytes = sum(w.nbytes for w in rast._shared.values())

    # ---- timed region (device time, CUDA events on the launching stream).
    # The views of a step are spread round-robin over `streams` so one view's
    # latency-bound binning overlaps another view's raster.
    stream = torch.cuda.current_stream(dev)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out_bufs = [(torch.empty((c.height, c.width, 3), device=dev),
                 torch.empty((c.height, c.width), device=dev),
                 torch.empty((c.height, c.width), dtype=torch.int32, device=dev)) for c in my_cams]
    def step_renders():
        for k, cam in enumerate(my_cams):
            with torch.cuda.stream(streams[k % len(streams)]):
                if args.no_graphs:
                    rast.forward(g, cam, check=False, out=out_bufs[k], track=False)
                else:  # one CUDA-graph launch per view (captured on first use)
                    rast.graph_forward(g, cam, out_bufs[k][:2])

    for s in streams[1:]:
        s.wait_stream(stream)
    step_renders()  # captures the graphs outside the timed region
    for s in streams[1:]:
        stream.wait_stream(s)
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize(dev)
    start.record(stream)
    for s in streams[1:]:
        s.wait_stream(stream)
    for _ in range(args.steps):
        step_renders()
    for s in streams[1:]:
        stream.wait_stream(s)
    stop.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    clk = clocks.stop()
    t_ms = start.elapsed_time(stop)

    # ---- dominant-kernel timing for the roofline: the same renders on ONE
    # stream, CUDA events bracketing each raster launch on its stream
    n_ev = args.steps * V
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(n_ev)]
    e = 0
    for _ in range(args.steps):
        for k, cam in enumerate(my_cams):
            rast.forward(g, cam, check=False, out=out_bufs[k], track=False, _events=ev[e])
            e += 1
    torch.cuda.synchronize(dev)
    raster_ms = [a[0].elapsed_time(a[1]) for a in ev]
    prep_ms = [a[2].elapsed_time(a[3]) for a in ev]
    bin_ms = [a[3].elapsed_time(a[0]) for a in ev]   # sgs_bin: depth sort, scan, emission, tile sort
    # overflow guard: the timed frames reused capacities sized in warm-up
    for cam in my_cams:
        assert not rast.forward(g, cam, check=True).stats()["overflow"]

    # ---- e2e through the host-buffer batch API
    pinned = PinnedScene(scene)
    br = BatchRenderer(rast, device=dev)
    for _ in range(2):
        br.render_views(pinned, my_cams, wait=False)
    torch.cuda.synchronize(dev)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        # every step uploads the whole scene and reads back every image; the
        # next step's upload overlaps this step's renders (double-buffered)
        br.render_views(pinned, my_cams, wait=False)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    t_e2e = e0.elapsed_time(e1)

    # ---- max over ranks
    vals = torch.tensor([t_ms, t_e2e, float(np.mean(raster_ms)), pairs_per_view], device=dev,
                        dtype=torch.float64)
    if world > 1:
        mx = vals.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        t_ms, t_e2e = float(mx[0]), float(mx[1])
    frames = world * V * args.steps
    value = frames / (t_ms / 1e3)
    e2e = frames / (t_e2e / 1e3)
    mpix = value * 1920 * 1080 / 1e6

    if rank == 0:
        peaks, src = measured_peaks()
        sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
        import torch.cuda as tc
        n_sm = tc.get_device_properties(dev).multi_processor_count
        # nominal 18 FP32 instructions + 1 EX2 per pair evaluation
        peak_pairs = n_sm * sm_mhz * 1e6 * min(128.0 / 18.0, 16.0)
        achieved = pairs_per_view / (float(np.mean(raster_ms)) / 1e3)
        E = float(np.mean([s["n_entries"] for s in stats]))
        Es = float(np.mean([s["n_bin_entries"] for s in stats]))
        n_emit = float(np.mean([s["n_emitting"] for s in stats]))
        N = float(args.n)
        hbm = float(peaks.get("hbm_gbs", 6549.1))

        def stage(ms_list, nbytes, what):
            ms = float(np.mean(ms_list))
            gbs = nbytes / (ms / 1e3) / 1e9
            return {"ms_per_view": ms, "algorithmic_bytes": int(nbytes), "GB_per_s": gbs,
                    "frac_of_hbm": gbs / hbm, "bytes_model": what}
        # algorithmic bytes per view: preprocess reads the
        # 152 B SoA row and writes 20 B of keys/rects/counts for every
        # primitive plus 80 B of records for every emitting one; binning =
        # depth sort (copy 8 + histogram 4 + 4 passes x 16 B per primitive),
        # offsets scan (24 B), emission reads (76 B per primitive) and writes
        # 8 B per super-tile entry, and the super-tile sort (histogram 4 +
        # pass 12 B per entry)
        stages = {
            "preprocess": stage(prep_ms, N * (152 + 20) + n_emit * 80,
                                "152 B read + 20 B written per primitive + 80 B records per emitting"),
            "binning": stage(bin_ms, N * (8 + 4 + 64 + 24 + 76) + Es * (8 + 16),
                             "176 B per primitive + 24 B per super-tile entry"),
        }
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded BASELINE configs[2] distributions, random-init scene)",
            "config": {"workload": WORKLOAD, "views_per_step_per_gpu": V,
                       "parallelism": f"view-sharded x{world}, Gaussians replicated",
                       "streams_per_gpu": len(streams),
                       "launch": "host launches" if args.no_graphs else "one CUDA graph per view",
                       "sort_mode": ["depth_first", "key64"][args.sort_mode],
                       "l2": "inputs larger than L2 (140 MB scene + ~0.5 GB key tables per view)"},
            "mpix_per_s": mpix,
            "vram": {"peak_dynamic_bytes_per_frame": int(frame_vram["peak_dynamic_bytes"]),
                     "workspace_bytes_per_frame": int(frame_vram["workspace_bytes"]),
                     "workspace_bytes_in_flight": int(inflight_bytes),
                     "reference_model_3sigma_bytes": int(model3s),
                     "static_scene_bytes": int(static_bytes),
                     "tile_entries_per_view": E},
            "roofline": {"bound": "fp32_issue", "kernel": "raster_fwd_kernel",
                         "achieved": achieved / 1e9, "peak": peak_pairs / 1e9, "unit": "Gpair/s",
                         "frac": achieved / peak_pairs, "traffic": profiled_traffic("raster_fwd_kernel"),
                         "note": f"pairs/view={pairs_per_view:.4g} (GPU counter); peak = SMs x "
                                 f"{sm_mhz:.0f} MHz ({src} sm_max) x 128/18 pairs/clk/SM; the "
                                 f"kernel's DRAM traffic is "
                                 f"{(profiled_traffic('raster_fwd_kernel') or 0) / (float(np.mean(raster_ms)) / 1e3) / 1e9:.0f}"
                                 f" GB/s ({(profiled_traffic('raster_fwd_kernel') or 0) / (float(np.mean(raster_ms)) / 1e3) / 1e9 / float(peaks.get('hbm_gbs', 6549.1)):.3f} of HBM): not memory-bound",
                         "raster_ms_per_view": float(np.mean(raster_ms))},
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": int(pinned.nbytes),
                    "d2h_bytes_per_step": int(BatchRenderer.d2h_bytes(my_cams))},
            "stages": stages,
            "super_tile_entries_per_view": Es,
            "gpu_launches": int(args.steps * V * KERNELS_PER_FRAME),
            "clocks": clk,
        }
        if not args.no_cpu_baseline:
            procs = cpu_procs()
            rate, d = cpu_reference_rate(scene, cams64[0], n_jobs=2 * procs, procs=procs)
            line["cpu_baseline"] = {
                "value": rate, "unit": UNIT, "cores": procs, "kind": "port",
                "sample": (f"camera 0: preprocess of all Gaussians + {2 * procs} blocks of 4 random "
                           f"pixels (dense f64 reference restatement, oracle/ref_dense.py) over "
                           f"{procs} processes; extrapolated to 1920x1080"),
                "s_per_px_one_core": d["s_per_px_one_core"], "preprocess_s": d["t_prep"]}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# -------------------------------------------------------- configs[3] training
def run_train(args):
    """configs[3]: 500k Gaussians, 8 views 1280x720 per step, forward + fused
    L1/SSIM loss + backward per view, mask gradients through the sigmoid,
    gradients all-reduced (NCCL) over ranks.  Views are split over the ranks
    (strong scaling: the 8-view step is fixed)."""
    import torch
    import torch.distributed as dist

    from paper_2509_07021_b200 import scenes
    from paper_2509_07021_b200.render import LossConfig, loss_and_grads_device
    from paper_2509_07021_b200.train import SoftPruneTrainer

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD
    n = args.n if args.n != 1_000_000 else 500_000
    scene, cams = scenes.config3(n=n)
    targets = [torch.from_numpy(scenes.target_image(0, c.height, c.width, v)).to(dev)
               for v, c in enumerate(cams)]
    tr = SoftPruneTrainer(scene, scene.extra["prim_logit"], scene.extra["lobe_logit"], device=dev,
                          group=group)
    for _ in range(max(args.warmup, 3)):
        tr.step(cams, targets, rank, world, apply=True)  # steady state: capacities sized
    torch.cuda.synchronize(dev)
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0.record(stream)
    for _ in range(args.steps):
        tr.step(cams, targets, rank, world, apply=True)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    t_ms = e0.elapsed_time(e1)
    # per-phase device time of one view (camera 0) on one stream
    g = tr.gaussians()
    rast = tr.rast
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    phases = {"forward": [], "loss": [], "backward": []}
    from paper_2509_07021_b200.loss import image_loss
    for _ in range(5):
        ev[0].record(stream)
        fr = rast.forward(g, cams[0], check=False)
        ev[1].record(stream)
        out, dimg, _ = image_loss(fr.img, targets[0], LossConfig())
        ev[2].record(stream)
        rast.backward(g, fr, dimg, mask_grads=True)
        ev[3].record(stream)
        torch.cuda.synchronize(dev)
        phases["forward"].append(ev[0].elapsed_time(ev[1]))
        phases["loss"].append(ev[1].elapsed_time(ev[2]))
        phases["backward"].append(ev[2].elapsed_time(ev[3]))
    t = torch.tensor([t_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms = float(t[0])
    views = len(cams) * args.steps
    if rank == 0:
        line = {"metric": "training views/s (configs[3]: fwd + L1/SSIM + bwd + mask grads + allreduce)",
                "value": views / (t_ms / 1e3), "unit": "views/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (seeded configs[3] distributions, U(0,1) targets)",
                "config": {"workload": f"configs[3]: {n} Gaussians, 3 lobes, 8 views 1280x720, "
                                       "soft masks, lambda_ssim 0.2",
                           "parallelism": f"views split over {world} ranks, NCCL gradient allreduce"},
                "phase_ms_per_view": {k: float(np.median(v)) for k, v in phases.items()},
                "clocks": clk}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------ configs[4] stress
def run_stress(args):
    """configs[4]: 5M Gaussians, one 3840x2160 frame split into horizontal
    tile strips balanced by a per-row cost estimate; rank r renders strip r
    (Gaussians replicated, no collective).  One GPU renders all strips."""
    import torch
    import torch.distributed as dist

    from paper_2509_07021_b200 import scenes
    from paper_2509_07021_b200.rasterizer import GaussianTensors, Rasterizer
    from paper_2509_07021_b200.sharding import balanced_strips, row_costs_from_rects

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n = args.n if args.n != 1_000_000 else 5_000_000
    scene, (cam,) = scenes.config4(n=n)
    rast = Rasterizer(device=dev)
    g = GaussianTensors.from_arrays(scene, device=dev)
    tiles_y = (cam.height + 15) // 16
    # cost estimate from one preprocess pass (host-side strip planning)
    f0 = rast.forward(g, cam, check=True, tile_rows=(0, 1), track=False)
    _, rect, tt, _ = rast.export_projected(f0)
    cost = row_costs_from_rects(rect.cpu().numpy().view(np.uint32), tt.cpu().numpy().view(np.uint32),
                                tiles_y)
    img = torch.empty((cam.height, cam.width, 3), device=dev)
    T = torch.empty((cam.height, cam.width), device=dev)
    # strips per rank: as few as keep one bin call under its entry limit
    from paper_2509_07021_b200._ffi import CapacityError
    per_rank = 1
    while True:
        strips = balanced_strips(cost, world * per_rank)[rank * per_rank:(rank + 1) * per_rank]
        ok = 1.0
        try:
            for y0, y1 in strips:
                rast.forward(g, cam, check=True, tile_rows=(y0, y1), out=(img, T, None), track=False)
        except CapacityError:
            ok = 0.0
        if world > 1:  # every rank must use the same strip partition
            f = torch.tensor([ok], device=dev)
            dist.all_reduce(f, op=dist.ReduceOp.MIN)
            ok = float(f[0])
        if ok:
            break
        per_rank *= 2

    def frame():
        for y0, y1 in strips:
            rast.forward(g, cam, check=False, tile_rows=(y0, y1), out=(img, T, None), track=False)

    for _ in range(max(args.warmup, 3)):
        frame()
    torch.cuda.synchronize(dev)
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0.record(stream)
    for _ in range(args.steps):
        frame()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    t = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_ms = float(t[0])
    ent = 0
    for y0, y1 in strips:
        ent += rast.forward(g, cam, check=True, tile_rows=(y0, y1), out=(img, T, None),
                            track=False).stats()["n_entries"]
    if rank == 0:
        line = {"metric": "frames/s (configs[4]: 5M Gaussians, 3840x2160, tile strips)",
                "value": args.steps / (t_ms / 1e3), "unit": "frames/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (seeded configs[4] distributions)",
                "config": {"workload": f"configs[4]: {n} Gaussians, 3840x2160, FoV 60, radius 2.5",
                           "strips": [list(s) for s in strips], "ranks": world},
                "tile_entries_rank0": int(ent), "clocks": clk}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "train":
        run_train(args)
    elif args.workload == "stress":
        run_stress(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
