"""bench.py keeps the driver's JSON-line contract: the reference arm on the
host (CPU) and our arm on a B200 (gpu marker)."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"], timeout=600)
    assert BASE_KEYS <= d.keys()
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert {"value", "unit", "cores", "kind", "sample"} <= d["cpu_baseline"].keys()
    assert d["cpu_baseline"]["kind"] in ("port", "reference")
    assert d["cpu_baseline"]["cpu_model"]
    sys.path.insert(0, str(ROOT))
    import bench
    assert d["config"] == bench.headline_config(1)   # the driver compares the arms' configs


@pytest.mark.gpu
def test_our_arm_line():
    d = _run(["--steps", "2", "--warmup", "3", "--cams", "4", "--workload", "all", "--no-cpu-baseline"],
             timeout=1200)
    assert BASE_KEYS <= d.keys()
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= d["roofline"].keys()
    assert 0 < d["roofline"]["frac"] < 2
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= d["e2e"].keys()
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["e2e_dropin"]["value"] > 0 and d["e2e_dropin"]["views"] >= 1  # render._render_params path
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= d["clocks"].keys()
    assert "workload" in d["config"]
    w = d["workloads"]
    assert {"cfg1", "cfg3", "cfg4", "cfg2_key64"} <= w.keys()
    assert all(w[k]["value"] > 0 for k in w)
    assert w["cfg1"]["vram"]["measured_peak_dynamic_bytes"] > 0
    assert 0 < w["cfg3"]["roofline_backward"]["frac"] < 2


def _run_two_ranks(args, timeout, env_extra):
    import os
    env = dict(os.environ, **env_extra)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", str(ROOT / "bench.py"), "--gpus", "2", *args]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]   # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.gpu
def test_two_rank_control_flow_on_one_gpu():
    """The torchrun path of our arm (view shards, barriers, max-over-ranks
    timing, the trainer's bucketed all-reduce) with both ranks sharing the
    one GPU over gloo (SGS_BENCH_SHARED_GPU): a functional check, marked as
    such in the line -- the driver's multi-GPU runs use NCCL, one GPU each."""
    d = _run_two_ranks(["--steps", "1", "--warmup", "3", "--cams", "4", "--gaussians", "100000", "--workload", "render",
                        "--no-cpu-baseline"], timeout=900, env_extra={"SGS_BENCH_SHARED_GPU": "1"})
    assert d["n_gpus"] == 2 and d["value"] > 0 and "functional_check_only" in d
    assert d["e2e"]["value"] > 0
    t = _run_two_ranks(["--steps", "1", "--warmup", "3", "--gaussians", "50000", "--workload", "train"], timeout=900,
                       env_extra={"SGS_BENCH_SHARED_GPU": "1"})
    assert t["n_gpus"] == 2 and t["value"] > 0 and "functional_check_only" in t
