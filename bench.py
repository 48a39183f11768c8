#!/usr/bin/env python
"""Benchmark: BASELINE.json metric "frames/s & Mpix/s at 1080p, 1M Gaussians,
3 SG lobes (1/2/4/8 B200); peak render VRAM" on configs[2].

  python bench.py [--gpus N] [--steps K] [--warmup W] [--views V] [--impl ours|reference]

One process per GPU (torchrun for N > 1).  A step = the configs[2] batch:
the 64 cameras of the 1M-Gaussian, 3-lobe scene at 1920x1080, sharded
round-robin over the ranks (rank r renders cameras r, r+N, ...), Gaussians
replicated, no collective on the data path (strong scaling: the 64-view
batch is fixed).  `value` = 64 x steps / max-over-ranks device time.
`e2e` = the same metric through the host-buffer batch API (pinned H2D of the
scene + D2H of every image inside the timed region).

The default run (--workload all) adds `workloads`: configs[1] (frames/s and
measured vs modelled dynamic VRAM), configs[3] (training views/s, backward
raster roofline), configs[4] (4K stress frame in tile strips) and the
north_star's literal 64-bit-key sort mode on configs[2].

--impl reference times the reference algorithm (dense float64 NumPy
restatement, oracle/ref_dense.py, pinned to the reference's own outputs) on
the host cores, rank 0 only, on bounded pixel samples of the same workload,
extrapolated to frames/s.
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
SHARED_NOTE = "SGS_BENCH_SHARED_GPU: all ranks shared one GPU over gloo; not a measurement"
WORKLOAD = "configs[2]: 1,000,000 Gaussians (64 clusters), 3 SG lobes, 64 cameras 1920x1080, FoV 60"
N_CAMS = 64
# libsgs kernels per forward frame (depth-first mode, 1080p): preprocess (also
# accumulates the depth-digit histograms); 4 onesweep passes
# (depth sort); the one-pass offsets scan; emit_entries (also the cell
# histogram and the range reset); 1 onesweep pass (super-tile
# sort + ranges); cell_order, raster_fwd (profiles/r01_launches_v10.csv)
KERNELS_PER_FRAME = 10


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", "--gaussians", dest="n", type=int, default=None, help="override the workload's Gaussian count")
    ap.add_argument("--cams", type=int, default=N_CAMS, help="configs[2] cameras per step (the batch)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sort-mode", type=int, default=0)
    ap.add_argument("--streams", type=int, default=8,
                    help="concurrent CUDA streams the views of a step are spread over")
    ap.add_argument("--no-graphs", action="store_true",
                    help="launch every kernel from the host instead of replaying per-view CUDA graphs")
    ap.add_argument("--workload", default="all", choices=["all", "render", "train", "stress", "cfg1"],
                    help="all: configs[2] headline + configs[1]/[3]/[4] sub-workloads; render: the "
                         "headline alone; train / stress / cfg1: one sub-workload as its own line")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def headline_config(world: int, cams: int = N_CAMS) -> dict:
    """The configs[2] `config` both arms print (same dict, so the driver's
    same_config check compares like with like)."""
    return {"workload": WORKLOAD, "views_per_step": cams,
            "parallelism": f"view-sharded x{world} (round-robin), Gaussians replicated",
            "l2": "inputs larger than L2 (152 MB scene + ~0.23 GB key tables per view)"}


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


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


def cfg0_full_frame_cpu(procs: int) -> dict:
    """The reference algorithm on configs[0] at the FULL 256x256 frame, not
    extrapolated: the dense float64 restatement's
    _render_params and loss_and_grads (L1, lambda_ssim = 0; render.py:393-408,
    645-678) with the pixel blocks spread over all `procs` host processes."""
    from oracle import ref_dense
    from paper_2509_07021_b200 import scenes
    scene, (cam,) = scenes.config0()
    target = scenes.target_image(0, cam.height, cam.width)
    t = time.perf_counter()
    ref_dense.render_parallel(scene, cam, procs)
    t_fwd = time.perf_counter() - t
    t = time.perf_counter()
    ref_dense.loss_and_grads_parallel(scene, cam, target, procs, lambda_ssim=0.0)
    t_lg = time.perf_counter() - t
    return {"render_s": t_fwd, "loss_and_grads_s": t_lg, "frames_per_s": 1.0 / t_fwd,
            "cores": procs, "kind": "port", "config": "configs[0]: 10k Gaussians, 256x256, full frame",
            "note": "dense float64 restatement of render.py (oracle/ref_dense.py), every pixel, no "
                    "extrapolation; loss_and_grads = forward + L1 + analytic backward"}


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    from paper_2509_07021_b200 import scenes
    n = args.n or 1_000_000
    scene, cams = scenes.config2(n=n, n_cams=1)
    cam = cams[0]
    procs = cpu_procs()
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
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
              f"preprocess of all {n} Gaussians for camera 0, then {procs} blocks of 4 random "
              f"pixels blended against every visible Gaussian in parallel over {procs} host "
              f"processes; frames/s extrapolated linearly to 1920x1080 (the reference blend is "
              f"exactly O(V*P))")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / max(args.steps, 1),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded configs[2] distributions)", "impl": "reference",
            "config": headline_config(world, args.cams),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "port",
                             "cpu_model": cpu_model(), "sample": sample,
                             "s_per_px_one_core": float(np.median([d["s_per_px_one_core"] for d in details])),
                             "preprocess_s": float(np.median([d["t_prep"] for d in details]))},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
class Ctx:
    """Per-process state shared by the workloads of one bench run."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist
        self.args = args
        self.rank, self.world, self.local = dist_env()
        # SGS_BENCH_SHARED_GPU=1: functional check of the multi-rank control
        # flow on a one-GPU box (every rank on cuda:0, gloo collectives); its
        # numbers are not measurements and the line says so
        self.shared = os.environ.get("SGS_BENCH_SHARED_GPU") == "1" and self.world > 1
        if self.shared:
            self.local = 0
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        if self.world > 1 and not dist.is_initialized():
            if self.shared:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=self.dev)
        self.peaks, self.peak_src = measured_peaks()
        self.n_sm = torch.cuda.get_device_properties(self.dev).multi_processor_count
        self.sm_mhz = float(self.peaks.get("sm_max_mhz", 1965.0))
        self.hbm = float(self.peaks.get("hbm_gbs", 6549.1))

    def barrier(self):
        import torch.distributed as dist
        if self.world > 1:
            dist.barrier()

    def max_over_ranks(self, *vals):
        import torch
        import torch.distributed as dist
        t = torch.tensor([float(v) for v in vals], device=self.dev, dtype=torch.float64)
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(v) for v in t]

    def sum_over_ranks(self, *vals):
        import torch
        import torch.distributed as dist
        t = torch.tensor([float(v) for v in vals], device=self.dev, dtype=torch.float64)
        if self.world > 1:
            dist.all_reduce(t)
        return [float(v) for v in t]

    def close(self):
        import torch.distributed as dist
        if self.world > 1 and dist.is_initialized():
            dist.destroy_process_group()


def fwd_pair_peak(ctx) -> float:
    # nominal 18 FP32 instructions + 1 EX2 per pair evaluation
    return ctx.n_sm * ctx.sm_mhz * 1e6 * min(128.0 / 18.0, 16.0)


def bwd_pair_peak(ctx) -> float:
    # the backward's nominal cost is 2.5x the forward's 18 FP32
    # instructions per (pixel, kept record) pair, i.e. 45
    return ctx.n_sm * ctx.sm_mhz * 1e6 * 128.0 / 45.0


def run_dropin(scene, cams) -> dict:
    """The reference-signature path a drop-in user calls per view:
    render._render_params (render.py:393-408) with the reference's float64
    SceneParams in and a float64 (H, W, 3) image out -- the scene crosses the
    link on every call, as the signature requires (no cache can prove a
    caller's arrays unchanged without reading them).  Wall clock per call
    (the call is synchronous: it returns host memory)."""
    import time

    import torch

    from paper_2509_07021_b200 import render as R
    from paper_2509_07021_b200 import scenes
    p = R.SceneParams(**{f: getattr(scene, f).astype(np.float64) for f in scenes.FIELDS},
                      lobe_mask=scene.lobe_mask)
    R._render_params(p, cams[0], (0.0, 0.0, 0.0))  # workspaces sized
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for cam in cams:
        img = R._render_params(p, cam, (0.0, 0.0, 0.0))
    dt = time.perf_counter() - t0
    assert img.dtype == np.float64
    h2d = sum(int(getattr(p, f).size) * 4 for f in scenes.FIELDS) + int(p.lobe_mask.size) * 4
    return {"value": len(cams) / dt, "unit": UNIT, "views": len(cams),
            "h2d_bytes_per_view": h2d, "d2h_bytes_per_view": int(img.size) * 4,
            "api": "render._render_params (float64 SceneParams in, float64 image out, one call per view, "
                   "scene uploaded every call), wall clock"}


def run_headline(ctx, timed_clocks: bool = True) -> dict:
    """configs[2]: the 64-camera batch, sharded over the ranks."""
    import torch

    from paper_2509_07021_b200 import _ffi, scenes
    from paper_2509_07021_b200.batch import BatchRenderer, PinnedScene
    from paper_2509_07021_b200.camera import to_sgs
    from paper_2509_07021_b200.postprocess import measured_render_vram
    from paper_2509_07021_b200.rasterizer import GaussianTensors, Rasterizer
    from paper_2509_07021_b200.sharding import shard_views
    import ctypes as C

    args, dev = ctx.args, ctx.dev
    n = args.n or 1_000_000
    scene, cams64 = scenes.config2(n=n, n_cams=args.cams)
    mine = shard_views(len(cams64), ctx.rank, ctx.world)
    my_cams = [cams64[v] for v in mine]
    V = len(my_cams)
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
                rast.forward(g, cam, check=True, track=False)
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
    ws = rast.workspace(g, my_cams[0])
    _ffi.call("sgs_vram_model", C.byref(g.c_params()), C.byref(to_sgs(my_cams[0])), 16,
              C.byref(ws.desc), C.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    vs = ws.stats()
    model3s = 40 * vs["vram3s_visible"] + 12 * vs["vram3s_entries"]
    frame_vram = measured_render_vram(g, my_cams[0], rast=rast)
    inflight_bytes = sum(w.nbytes for w in rast._shared.values())

    # ---- timed region (device time, CUDA events on the launching stream).
    # The views of a step are spread round-robin over `streams` so one view's
    # latency-bound binning overlaps another view's raster.
    stream = torch.cuda.current_stream(dev)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out_bufs = [(torch.empty((c.height, c.width, 3), device=dev),
                 torch.empty((c.height, c.width), device=dev)) for c in my_cams]
    ovf = torch.zeros((V, 2), dtype=torch.int64, device=dev)

    def step_renders():
        for k, cam in enumerate(my_cams):
            with torch.cuda.stream(streams[k % len(streams)]):
                if args.no_graphs:
                    rast.forward(g, cam, check=False, out=(*out_bufs[k], None), track=False) \
                        .record_overflow(ovf[k])
                else:  # one CUDA-graph launch per view (captured on first use)
                    ovf[k].copy_(rast.graph_forward(g, cam, out_bufs[k]))

    for s in streams[1:]:
        s.wait_stream(stream)
    step_renders()  # captures the graphs outside the timed region
    for s in streams[1:]:
        stream.wait_stream(s)
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(ctx.local) if timed_clocks else None
    ctx.barrier()
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
    ctx.barrier()
    clk = clocks.stop() if clocks else None
    t_ms = start.elapsed_time(stop)
    assert int(ovf[:, 0].max()) == 0, "a timed view overflowed its tile-entry capacity"

    # ---- dominant-kernel timing for the roofline: the same renders on ONE
    # stream, CUDA events bracketing each raster launch on its stream
    n_ev = min(args.steps, 3) * V
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(n_ev)]
    e = 0
    for _ in range(min(args.steps, 3)):
        for k, cam in enumerate(my_cams):
            rast.forward(g, cam, check=False, out=(*out_bufs[k], None), track=False, _events=ev[e])
            e += 1
    torch.cuda.synchronize(dev)
    raster_ms = [a[0].elapsed_time(a[1]) for a in ev]
    prep_ms = [a[2].elapsed_time(a[3]) for a in ev]
    bin_ms = [a[3].elapsed_time(a[0]) for a in ev]   # sgs_bin: depth sort, scan, emission, tile sort

    # ---- e2e through the host-buffer batch API
    pinned = PinnedScene(scene)
    br = BatchRenderer(rast, device=dev, streams=args.streams)
    for _ in range(br.slots):  # every slot's buffers allocated before the timed calls
        br.render_views(pinned, my_cams, wait=False)
    br.finish()
    ctx.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        # every step uploads the whole scene and reads back every image; the
        # next step's upload overlaps this step's renders (double-buffered)
        br.render_views(pinned, my_cams, wait=False)
    br.finish()  # every image read back and overflow-checked
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ctx.barrier()
    t_e2e = e0.elapsed_time(e1)
    assert br.rerendered == 0, "e2e views re-rendered after an overflow inside the timed region"
    # release the pinned host buffers now (cudaFreeHost synchronises the
    # device; a later garbage collection would stall another workload's
    # event-timed region)
    pinned = None
    br = None
    import gc
    gc.collect()
    torch.cuda.synchronize(dev)

    dropin = run_dropin(scene, my_cams[:min(V, 16)]) if V else None

    # the e2e path's own roofline: pinned host <-> device copy bandwidth,
    # measured here (both directions at once, as the batch API overlaps them)
    link = measure_link(dev)
    t_ms, t_e2e = ctx.max_over_ranks(t_ms, t_e2e)
    frames = len(cams64) * args.steps
    value = frames / (t_ms / 1e3)
    e2e = frames / (t_e2e / 1e3)
    raster_mean = float(np.mean(raster_ms))
    achieved = pairs_per_view / (raster_mean / 1e3)
    peak_pairs = fwd_pair_peak(ctx)
    E = float(np.mean([s_["n_entries"] for s_ in stats]))
    Es = float(np.mean([s_["n_bin_entries"] for s_ in stats]))
    n_emit = float(np.mean([s_["n_emitting"] for s_ in stats]))
    N = float(n)

    def stage(ms_list, nbytes, what):
        ms = float(np.mean(ms_list))
        gbs = nbytes / (ms / 1e3) / 1e9
        return {"ms_per_view": ms, "algorithmic_bytes": int(nbytes), "GB_per_s": gbs,
                "frac_of_hbm": gbs / ctx.hbm, "bytes_model": what}
    # algorithmic bytes per view: preprocess reads the 152 B SoA
    # row and writes 20 B of keys/rects/counts for every primitive plus 80 B
    # of records for every emitting one; binning = depth sort (copy 8 +
    # histogram 4 + 4 passes x 16 B per primitive), offsets scan (24 B),
    # emission reads (76 B per primitive) and writes 8 B per super-tile entry,
    # and the super-tile sort (histogram 4 + pass 12 B per entry)
    if args.sort_mode == 0:
        bin_bytes, bin_model = N * (8 + 4 + 64 + 24 + 76) + Es * (8 + 16), \
            "176 B per primitive + 24 B per super-tile entry"
    else:
        # the same primitive depth sort, then 64-bit tile entries in depth order
        # sorted on the 13 tile bits of a 1080p frame (2 passes)
        bin_bytes, bin_model = N * (8 + 4 + 64 + 24 + 76) + E * (12 + 8 + 2 * 24), \
            "176 B per primitive + 68 B per tile entry (emission 12 B, histogram 8 B, 2 passes x 24 B)"
    stages = {
        "preprocess": stage(prep_ms, N * (152 + 20) + n_emit * 80,
                            "152 B read + 20 B written per primitive + 80 B records per emitting"),
        "binning": stage(bin_ms, bin_bytes, bin_model),
    }
    traffic = profiled_traffic("raster_fwd_kernel")
    return {
        "value": value, "t_ms": t_ms, "e2e": e2e, "frames": frames, "mine": V, "dropin": dropin,
        "mpix_per_s": value * 1920 * 1080 / 1e6,
        "vram": {"peak_dynamic_bytes_per_frame": int(frame_vram["peak_dynamic_bytes"]),
                 "workspace_bytes_per_frame": int(frame_vram["workspace_bytes"]),
                 "workspace_bytes_in_flight": int(inflight_bytes),
                 "reference_model_3sigma_bytes": int(model3s),
                 "static_scene_bytes": int(static_bytes),
                 "tile_entries_per_view": E},
        "roofline": {"bound": "fp32_issue", "kernel": "raster_fwd_kernel",
                     "achieved": achieved / 1e9, "peak": peak_pairs / 1e9, "unit": "Gpair/s",
                     "frac": achieved / peak_pairs, "traffic": traffic,
                     "note": f"pairs/view={pairs_per_view:.4g} (GPU counter); peak = {ctx.n_sm} SMs x "
                             f"{ctx.sm_mhz:.0f} MHz ({ctx.peak_src} sm_max) x 128/18 pairs/clk/SM; "
                             f"DRAM traffic {(traffic or 0) / (raster_mean / 1e3) / 1e9:.0f} GB/s: not "
                             f"memory-bound",
                     "raster_ms_per_view": raster_mean},
        "e2e_bytes": (int(pinned_bytes(scene)), int(sum(c.width * c.height * 12 + 16 for c in my_cams))),
        "link": link,
        "stages": stages, "super_tile_entries_per_view": Es,
        "clocks": clk, "gpu_launches": int(args.steps * V * (KERNELS_PER_FRAME if args.sort_mode == 0 else 12)),
        "scene": scene, "cams": cams64,
    }


def measure_link(dev, nbytes: int = 1 << 30) -> dict:
    """Pinned host <-> device copy bandwidth (GB/s): D2H alone, H2D alone,
    and both at once on two streams (CUDA events, best of 3)."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d2 = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    out = {}
    for name in ("d2h", "h2d", "both"):
        best = 0.0
        for _ in range(3):
            torch.cuda.synchronize(dev)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s1)
            s2.wait_event(a)
            if name in ("d2h", "both"):
                with torch.cuda.stream(s1):
                    h.copy_(d, non_blocking=True)
            if name in ("h2d", "both"):
                with torch.cuda.stream(s2):
                    d2.copy_(h2, non_blocking=True)
            s1.wait_stream(s2)
            b.record(s1)
            torch.cuda.synchronize(dev)
            moved = nbytes * (2 if name == "both" else 1)
            best = max(best, moved / (a.elapsed_time(b) / 1e3) / 1e9)
        out[name + "_GBs"] = best
    return out


def pinned_bytes(scene) -> int:
    from paper_2509_07021_b200.batch import HOST_FIELDS
    n = sum(np.asarray(getattr(scene, f)).size * 4 for f in HOST_FIELDS)
    pm = getattr(scene, "prim_mask", None)
    return n + (0 if pm is None else np.asarray(pm).size * 4)


def run_cfg1(ctx) -> dict:
    """configs[1]: 200k Gaussians with soft-pruning masks (prim Bernoulli(0.6),
    K ~ U{0..3} lobes), one 1280x720 view; frames/s and the measured peak
    dynamic render VRAM next to the reference model 40 vis + 12 E
    (postprocess.py:101-137).  Every rank renders the frame (replicas)."""
    import torch
    import ctypes as C

    from paper_2509_07021_b200 import _ffi, scenes
    from paper_2509_07021_b200.camera import to_sgs
    from paper_2509_07021_b200.postprocess import measured_render_vram
    from paper_2509_07021_b200.rasterizer import GaussianTensors, Rasterizer
    args, dev = ctx.args, ctx.dev
    scene, (cam,) = scenes.config1()
    rast = Rasterizer(device=dev)
    g = GaussianTensors.from_arrays(scene, device=dev)
    for _ in range(max(args.warmup, 3)):
        rast.forward(g, cam, check=True, track=False)
    out = (torch.empty((cam.height, cam.width, 3), device=dev), torch.empty((cam.height, cam.width), device=dev))
    ovf = rast.graph_forward(g, cam, out)
    stream = torch.cuda.current_stream(dev)
    reps = 8
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    ctx.barrier()
    e0.record(stream)
    for _ in range(args.steps * reps):
        rast.graph_forward(g, cam, out)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    assert int(ovf[0]) == 0
    t_ms = ctx.max_over_ranks(e0.elapsed_time(e1))[0]
    vram = measured_render_vram(g, cam, rast=rast)
    ws = rast.workspace(g, cam, private=True, capacity=1)
    _ffi.call("sgs_vram_model", C.byref(g.c_params()), C.byref(to_sgs(cam)), 16, C.byref(ws.desc),
              C.c_void_p(stream.cuda_stream))
    vs = ws.stats()
    frames = args.steps * reps * ctx.world
    return {"metric": "frames/s (configs[1]: 200k Gaussians, soft masks, 1280x720)",
            "value": frames / (t_ms / 1e3), "unit": "frames/s", "scaling": "weak (replicas)",
            "ms_per_frame": t_ms / (args.steps * reps),
            "vram": {"measured_peak_dynamic_bytes": int(vram["peak_dynamic_bytes"]),
                     "workspace_bytes": int(vram["workspace_bytes"]),
                     "output_bytes": int(vram["output_bytes"]),
                     "reference_model_bytes": int(40 * vs["vram3s_visible"] + 12 * vs["vram3s_entries"]),
                     "reference_model": "40 B x visible + 12 B x 3-sigma tile entries (postprocess.py:136)",
                     "visible": int(vram["visible"]), "emitting": int(vram["emitting"]),
                     "tile_entries": int(vram["tile_entries"])},
            "launch": "one CUDA graph per frame", "frames": frames}


# -------------------------------------------------------- configs[3] training
def run_cfg3(ctx) -> dict:
    """configs[3]: 500k Gaussians, 8 views 1280x720 per step, forward + fused
    L1/SSIM loss + backward per view, mask gradients through the sigmoid,
    gradients all-reduced (NCCL) over ranks.  Views are split over the ranks
    (strong scaling: the 8-view step is fixed).  The backward raster (K6) is
    timed alone per view for its roofline: pairs = kept (pixel, record)
    pairs, i.e. the sum of the forward's per-pixel contributor counts."""
    import torch

    from paper_2509_07021_b200 import scenes
    from paper_2509_07021_b200.loss import image_loss
    from paper_2509_07021_b200.render import LossConfig
    from paper_2509_07021_b200.train import SoftPruneTrainer
    import torch.distributed as dist
    args, dev = ctx.args, ctx.dev
    group = dist.group.WORLD if ctx.world > 1 else None
    n = args.n if (args.n and args.workload == "train") else 500_000
    scene, cams = scenes.config3(n=n)
    targets = [torch.from_numpy(scenes.target_image(0, c.height, c.width, v)).to(dev)
               for v, c in enumerate(cams)]
    tr = SoftPruneTrainer(scene, scene.extra["prim_logit"], scene.extra["lobe_logit"], device=dev,
                          group=group)
    for _ in range(max(args.warmup, 3)):
        tr.step(cams, targets, ctx.rank, ctx.world, apply=True, graph=not args.no_graphs)  # sized, captured
    torch.cuda.synchronize(dev)
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(ctx.local) if args.workload == "train" else None
    ctx.barrier()
    torch.cuda.synchronize(dev)
    e0.record(stream)
    for _ in range(args.steps):
        tr.step(cams, targets, ctx.rank, ctx.world, apply=True, sync=False,
                graph=not args.no_graphs)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    clk = clocks.stop() if clocks else None
    t_ms = e0.elapsed_time(e1)
    # per-phase device time of each view on one stream; K6 alone for the roofline
    g = tr.gaussians()
    rast = tr.rast
    phases = {"forward": [], "loss": [], "backward_raster": [], "backward_params": []}
    pairs = []
    for cam in cams:  # size every view's workspace first: no host sync inside the timed phases
        rast.forward(g, cam, check=True)
    torch.cuda.synchronize(dev)
    for v, cam in enumerate(cams):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        # the GPU sleeps while the host enqueues the view's four phases, so
        # host-side call overhead never shows up inside an event interval
        torch.cuda._sleep(20_000_000)
        ev[0].record(stream)
        fr = rast.forward(g, cam, check=False)
        ev[1].record(stream)
        _, dimg, _ = image_loss(fr.img, targets[v], LossConfig())
        ev[2].record(stream)
        g2 = rast.backward_raster(g, fr, dimg)
        ev[3].record(stream)
        rast.backward_params(g, fr.cam, g2, mask_grads=True)
        ev[4].record(stream)
        torch.cuda.synchronize(dev)
        pairs.append(int(fr.ncontrib.to(torch.int64).sum()))
        for k, name in enumerate(phases):
            phases[name].append(ev[k].elapsed_time(ev[k + 1]))
    t_ms = ctx.max_over_ranks(t_ms)[0]
    views = len(cams) * args.steps
    k6_ms = float(np.mean(phases["backward_raster"]))
    achieved = float(np.mean(pairs)) / (k6_ms / 1e3)
    peak = bwd_pair_peak(ctx)
    return {"metric": "training views/s (configs[3]: fwd + L1/SSIM + bwd + mask grads + allreduce)",
            "value": views / (t_ms / 1e3), "unit": "views/s", "steps": args.steps,
            "ms_per_step": t_ms / args.steps, "scaling": "strong", "dtype": "f32",
            "config": {"workload": f"configs[3]: {n} Gaussians, 3 lobes, 8 views 1280x720, soft masks "
                                   "(sigmoid logits), lambda_ssim 0.2, mask sparsity penalty",
                       "parallelism": f"views split over {ctx.world} ranks, NCCL gradient allreduce"},
            "phase_ms_per_view": {k: float(np.mean(v)) for k, v in phases.items()},
            "roofline_backward": {
                "bound": "fp32_issue", "kernel": "raster_bwd_kernel", "achieved": achieved / 1e9,
                "peak": peak / 1e9, "unit": "Gpair/s", "frac": achieved / peak,
                "traffic": profiled_traffic("raster_bwd_kernel"),
                "pairs_per_view": float(np.mean(pairs)), "ms_per_view": k6_ms,
                "note": f"pairs = sum over pixels of the kept contributor count; peak = {ctx.n_sm} SMs x "
                        f"{ctx.sm_mhz:.0f} MHz x 128/45 (SURVEY §8(d): 2.5x the forward's 18 FP32 "
                        f"instructions per pair), K6 timed alone with CUDA events"},
            "clocks": clk, "gpu_launches": int(args.steps * len(cams) * 16 // max(ctx.world, 1))}


# ------------------------------------------------------------ configs[4] stress
def run_cfg4(ctx) -> dict:
    """configs[4]: 5M Gaussians, one 3840x2160 frame split into horizontal
    tile strips balanced by a per-row cost estimate; rank r renders strip r
    (Gaussians replicated, no collective).  One GPU renders all strips."""
    import torch
    import torch.distributed as dist

    from paper_2509_07021_b200 import scenes
    from paper_2509_07021_b200._ffi import CapacityError
    from paper_2509_07021_b200.rasterizer import GaussianTensors, Rasterizer
    from paper_2509_07021_b200.sharding import (balanced_strips, refine_row_costs, row_costs_from_rects,
                                                row_costs_measured)
    args, dev = ctx.args, ctx.dev
    n = args.n if (args.n and args.workload == "stress") else 5_000_000
    scene, (cam,) = scenes.config4(n=n)
    rast = Rasterizer(device=dev)
    g = GaussianTensors.from_arrays(scene, device=dev)
    tiles_y = (cam.height + 15) // 16
    # strip planning from one measured full frame: raster cost per tile row
    # from the kept pairs (contributor counts), binning cost from the tile
    # entries (sharding.row_costs_measured)
    _, rect, tt = rast.preprocess_only(g, cam)
    entry_rows = row_costs_from_rects(rect.cpu().numpy().view(np.uint32), tt.cpu().numpy().view(np.uint32),
                                      tiles_y)
    img = torch.empty((cam.height, cam.width, 3), device=dev)
    T = torch.empty((cam.height, cam.width), device=dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    full = rast.forward(g, cam, check=True, _events=ev)
    full = rast.forward(g, cam, check=True, _events=ev)
    torch.cuda.synchronize(dev)
    cost = row_costs_measured(full.ncontrib.cpu().numpy(), entry_rows, ev[0].elapsed_time(ev[1]),
                              ev[3].elapsed_time(ev[0]))
    full = None
    per_rank = 1
    while True:
        strips = balanced_strips(cost, ctx.world * per_rank)[ctx.rank * per_rank:(ctx.rank + 1) * per_rank]
        ok = 1.0
        try:
            for y0, y1 in strips:
                rast.forward(g, cam, check=True, tile_rows=(y0, y1), out=(img, T, None), track=False)
        except CapacityError:
            ok = 0.0
        if ctx.world > 1:  # every rank must use the same strip partition
            f = torch.tensor([ok], device=dev)
            dist.all_reduce(f, op=dist.ReduceOp.MIN)
            ok = float(f[0])
        if ok:
            break
        per_rank *= 2

    def strip_ms(y0, y1) -> float:
        for _ in range(2):
            rast.forward(g, cam, check=True, tile_rows=(y0, y1), out=(img, T, None), track=False)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rast.forward(g, cam, check=False, tile_rows=(y0, y1), out=(img, T, None), track=False)
        e1.record()
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1)

    # re-plan twice from the measured strip times (sharding.refine_row_costs):
    # every strip also projects and depth-sorts each primitive overlapping it,
    # which a per-row model cannot see (profiles/predict_strips.py)
    n_strips = ctx.world * per_rank
    if n_strips > 1:
        for _ in range(2):
            plan = balanced_strips(cost, n_strips)
            t = torch.zeros(n_strips, dtype=torch.float64, device=dev)
            for j in range(ctx.rank * per_rank, (ctx.rank + 1) * per_rank):
                t[j] = strip_ms(*plan[j])
            if ctx.world > 1:
                dist.all_reduce(t)
            cost = refine_row_costs(cost, plan, t.cpu().numpy())
        strips = balanced_strips(cost, n_strips)[ctx.rank * per_rank:(ctx.rank + 1) * per_rank]
        for y0, y1 in strips:  # size the refined strips' workspaces
            rast.forward(g, cam, check=True, tile_rows=(y0, y1), out=(img, T, None), track=False)

    def frame():
        for y0, y1 in strips:
            rast.forward(g, cam, check=False, tile_rows=(y0, y1), out=(img, T, None), track=False)

    for _ in range(max(args.warmup, 3)):
        frame()
    torch.cuda.synchronize(dev)
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(ctx.local) if args.workload == "stress" else None
    ctx.barrier()
    torch.cuda.synchronize(dev)
    e0.record(stream)
    for _ in range(args.steps):
        frame()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    clk = clocks.stop() if clocks else None
    t_ms = ctx.max_over_ranks(e0.elapsed_time(e1))[0]
    ent = 0
    for y0, y1 in strips:
        st = rast.forward(g, cam, check=True, tile_rows=(y0, y1), out=(img, T, None), track=False).stats()
        assert not st["overflow"]
        ent += st["n_entries"]
    ent = int(ctx.sum_over_ranks(ent)[0])
    return {"metric": "frames/s (configs[4]: 5M Gaussians, 3840x2160, tile strips)",
            "value": args.steps / (t_ms / 1e3), "unit": "frames/s", "steps": args.steps,
            "ms_per_step": t_ms / args.steps, "scaling": "strong", "dtype": "f32",
            "config": {"workload": f"configs[4]: {n} Gaussians, 3840x2160, FoV 60, radius 2.5",
                       "strips_rank0": [list(s_) for s_ in strips], "ranks": ctx.world},
            "tile_entries_per_frame": ent, "clocks": clk,
            "gpu_launches": int(args.steps * len(strips) * KERNELS_PER_FRAME)}


def run_key64(ctx, scene, cams) -> dict:
    """The north_star's literal binning: 64-bit (tile << 32 | depth bits) keys
    radix-sorted by the onesweep (SGS_SORT_KEY64), configs[2] camera batch of
    this rank, one stream, host launches; per-view binning bytes vs HBM.  The
    keys are emitted in the float64 depth order (the primitives' depth sort,
    as in the default mode), so the LSD sort runs over the tile digits only."""
    import torch

    from paper_2509_07021_b200 import _ffi
    from paper_2509_07021_b200.rasterizer import GaussianTensors, Rasterizer
    from paper_2509_07021_b200.sharding import shard_views
    args, dev = ctx.args, ctx.dev
    my_cams = [cams[v] for v in shard_views(len(cams), ctx.rank, ctx.world)][:8]
    rast = Rasterizer(sort_mode=_ffi.SORT_KEY64, device=dev)
    g = GaussianTensors.from_arrays(scene, device=dev)
    stats = [rast.forward(g, c, check=True, track=False).stats() for c in my_cams]
    out = [(torch.empty((c.height, c.width, 3), device=dev), torch.empty((c.height, c.width), device=dev), None)
           for c in my_cams]
    stream = torch.cuda.current_stream(dev)
    reps = max(2, args.steps // 4)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(reps * len(my_cams))]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    e0.record(stream)
    k = 0
    for _ in range(reps):
        for j, c in enumerate(my_cams):
            rast.forward(g, c, check=False, out=out[j], track=False, _events=ev[k])
            k += 1
    e1.record(stream)
    torch.cuda.synchronize(dev)
    t_ms = ctx.max_over_ranks(e0.elapsed_time(e1))[0]
    bin_ms = float(np.mean([a[3].elapsed_time(a[0]) for a in ev]))
    E = float(np.mean([s_["n_entries"] for s_ in stats]))
    N = float(g.n)
    tiles = ((cams[0].width + 15) // 16) * ((cams[0].height + 15) // 16)
    passes = (max(1, int(np.ceil(np.log2(tiles)))) + 7) // 8
    # depth sort + tie fix-up + scan + emission reads per primitive (176 B, as
    # the default mode); per tile entry the emission writes 12 B, the tile sort
    # reads 8 B for its histogram and moves 24 B per pass
    nbytes = N * 176 + E * (12 + 8 + passes * 24)
    frames = reps * len(my_cams) * ctx.world
    return {"metric": f"frames/s (configs[2], SGS_SORT_KEY64: 64-bit tile|depth keys emitted in depth order, "
                      f"{passes} onesweep passes over the tile bits)",
            "value": frames / (t_ms / 1e3), "unit": "frames/s", "streams": 1, "launch": "host launches",
            "binning": {"ms_per_view": bin_ms, "algorithmic_bytes": int(nbytes),
                        "GB_per_s": nbytes / (bin_ms / 1e3) / 1e9,
                        "frac_of_hbm": nbytes / (bin_ms / 1e3) / 1e9 / ctx.hbm,
                        "bytes_model": f"176 B per primitive + {12 + 8 + passes * 24} B per tile entry "
                                       f"(emission 12 B, histogram 8 B, {passes} passes x 24 B)"},
            "tile_entries_per_view": E}


def e2e_roofline(h, h2d, d2h, steps) -> dict:
    """The batch API moves every image D2H (fp32 RGB, 24.9 MB at 1080p) and
    the scene H2D each step; the copies overlap the renders, so the step is
    bounded by the link: max(D2H bytes / D2H bandwidth, device step time)."""
    link = h["link"]
    t_link = d2h / (link["d2h_GBs"] * 1e9)
    t_dev = h["t_ms"] / 1e3 / steps
    bound = max(t_link, t_dev)
    achieved_ms = h["frames"] / h["e2e"] / steps * 1e3
    return {"bound": "pcie_d2h" if t_link >= t_dev else "device",
            "link_GBs": link, "d2h_GB_per_step": d2h / 1e9,
            "bound_ms_per_step": bound * 1e3, "achieved_ms_per_step": achieved_ms,
            "frac": bound * 1e3 / achieved_ms}


def torch_sync(ctx):
    import torch
    torch.cuda.synchronize(ctx.dev)


def run_ours(args):
    """Our arm: the configs[2] headline (+ the sub-workloads with --workload all)."""
    import gc
    # No automatic garbage collection inside the timed regions: a full
    # collection pauses the host for milliseconds, longer than the GPU's
    # queued work, and showed up as gaps of up to 8 ms inside the per-phase
    # event intervals.  Collections run explicitly between workloads.
    gc.collect()
    gc.disable()
    ctx = Ctx(args)
    if args.workload in ("train", "stress", "cfg1"):
        fn = {"train": run_cfg3, "stress": run_cfg4, "cfg1": lambda c: run_cfg1(c)}[args.workload]
        res = fn(ctx)
        if ctx.rank == 0:
            line = dict(res)
            line.update({"n_gpus": ctx.world, "warmup": args.warmup, "higher_is_better": True,
                         "vs_baseline": None, "data": "synthetic (seeded BASELINE configs distributions)"})
            if ctx.shared:
                line["functional_check_only"] = SHARED_NOTE
            print(json.dumps(line), flush=True)
        ctx.close()
        return
    h = run_headline(ctx)
    workloads = {}
    if args.workload == "all":
        for name, fn in (("cfg1", run_cfg1), ("cfg3", run_cfg3), ("cfg4", run_cfg4),
                         ("cfg2_key64", lambda c: run_key64(c, h["scene"], h["cams"]))):
            gc.collect()
            torch_sync(ctx)
            workloads[name] = fn(ctx)
    if ctx.rank == 0:
        h2d, d2h = h["e2e_bytes"]
        line = {
            "metric": METRIC, "value": h["value"], "unit": UNIT, "n_gpus": ctx.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": h["t_ms"] / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded BASELINE configs[2] distributions, random-init scene)",
            "config": headline_config(ctx.world, args.cams),
            "setup": {"streams_per_gpu": args.streams,
                      "launch": "host launches" if args.no_graphs else "one CUDA graph per view",
                      "sort_mode": ["depth_first", "key64"][args.sort_mode]},
            "mpix_per_s": h["mpix_per_s"], "vram": h["vram"], "roofline": h["roofline"],
            "e2e": {"value": h["e2e"], "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "batch.BatchRenderer.render_views (pinned host scene in, host images out, "
                           "overflow-checked)",
                    "roofline": e2e_roofline(h, h2d, d2h, args.steps)},
            "e2e_dropin": h["dropin"],
            "stages": h["stages"], "super_tile_entries_per_view": h["super_tile_entries_per_view"],
            "gpu_launches": h["gpu_launches"], "clocks": h["clocks"],
        }
        if ctx.shared:
            line["functional_check_only"] = SHARED_NOTE
        if workloads:
            line["workloads"] = workloads
            line["gpu_launches"] += sum(int(w.get("gpu_launches", 0)) for w in workloads.values())
        if not args.no_cpu_baseline and ctx.world == 1:
            procs = cpu_procs()
            rate, d = cpu_reference_rate(h["scene"], h["cams"][0], n_jobs=2 * procs, procs=procs)
            line["cpu_baseline"] = {
                "value": rate, "unit": UNIT, "cores": procs, "kind": "port", "cpu_model": cpu_model(),
                "sample": (f"camera 0: preprocess of all Gaussians + {2 * procs} blocks of 4 random "
                           f"pixels (dense f64 reference restatement, oracle/ref_dense.py) over "
                           f"{procs} processes; extrapolated to 1920x1080"),
                "s_per_px_one_core": d["s_per_px_one_core"], "preprocess_s": d["t_prep"],
                "cfg0_full_frame": cfg0_full_frame_cpu(procs)}
        print(json.dumps(line), flush=True)
    ctx.close()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
