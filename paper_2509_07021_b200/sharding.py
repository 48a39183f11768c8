"""Multi-GPU partitioning of the render path.

One process per GPU (torchrun / torch.distributed, NCCL over NVLink for the
data path).  Gaussians are replicated on every rank.

* View sharding (configs[2]): cameras are independent; rank r renders views
  r, r + G, r + 2G, ...  No collective.
* Tile strips (configs[4]): the frame's tile rows are split into G
  contiguous strips balanced by a per-row cost estimate from a cheap
  first pass; every rank preprocesses all N but emits keys only for its
  strip (sgs_camera.tile_y0/1).  No collective (optional gather for output).
* Data-parallel training (configs[3]): each rank runs forward + backward on
  its views; the parameter gradients are flattened into one bucket and
  all-reduced (SUM) -- the only collective on the path.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_views(n_views: int, rank: int, world: int) -> list[int]:
    """Round-robin view assignment (every view exactly once)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid rank/world")
    return list(range(rank, n_views, world))


def balanced_strips(row_cost, world: int) -> list[tuple[int, int]]:
    """Split tile rows [0, R) into `world` contiguous strips with roughly equal
    total cost (greedy prefix split on the cumulative cost).  Every strip is
    non-empty when R >= world."""
    cost = np.asarray(row_cost, dtype=np.float64)
    R = cost.size
    if world < 1:
        raise ValueError("world must be >= 1")
    if R == 0:
        return [(0, 0)] * world
    cum = np.concatenate([[0.0], np.cumsum(np.maximum(cost, 0.0) + 1e-9)])
    total = cum[-1]
    bounds = [0]
    for k in range(1, world):
        target = total * k / world
        b = int(np.searchsorted(cum, target, side="left"))
        lo = bounds[-1] + 1 if R - bounds[-1] > world - k else bounds[-1]
        hi = R - (world - k) if R >= world else R
        bounds.append(int(min(max(b, lo), max(hi, lo))))
    bounds.append(R)
    return [(bounds[i], bounds[i + 1]) for i in range(world)]


def row_costs_from_rects(rects: np.ndarray, tiles_touched: np.ndarray, tiles_y: int) -> np.ndarray:
    """Per-tile-row entry estimate from the preprocess rectangles (uniform
    spread of each primitive's tile count over its rows)."""
    cost = np.zeros(tiles_y, np.float64)
    r = np.asarray(rects, dtype=np.uint32).reshape(-1, 2)
    tt = np.asarray(tiles_touched, dtype=np.float64)
    live = tt > 0
    ty0 = (r[live, 1] & 0xFFFF).astype(np.int64)
    ty1 = (r[live, 1] >> 16).astype(np.int64)
    per = tt[live] / (ty1 - ty0 + 1)
    diff = np.zeros(tiles_y + 1)
    np.add.at(diff, ty0, per)
    np.add.at(diff, ty1 + 1, -per)
    cost += np.cumsum(diff)[:tiles_y]
    return cost


class GradBucket:
    """Flatten a dict of gradient tensors into one contiguous buffer (one
    NCCL all-reduce per step) and scatter it back."""

    def __init__(self, shapes: dict, device, dtype=torch.float32):
        self.keys = list(shapes)
        self.shapes = {k: tuple(shapes[k]) for k in self.keys}
        self.sizes = {k: int(np.prod(self.shapes[k])) for k in self.keys}
        self.offsets = {}
        off = 0
        for k in self.keys:
            self.offsets[k] = off
            off += (self.sizes[k] + 3) // 4 * 4  # 16-byte aligned views (float4 rows)
        self.numel = off
        self.flat = torch.zeros(off, device=device, dtype=dtype)

    def zero(self):
        self.flat.zero_()

    def view(self, k) -> torch.Tensor:
        o = self.offsets[k]
        return self.flat[o:o + self.sizes[k]].view(self.shapes[k])

    def add_(self, grads: dict):
        for k in self.keys:
            if k in grads and grads[k] is not None:
                self.view(k).add_(grads[k].to(self.flat.dtype))

    def allreduce_(self, group=None, average_over: float | None = None):
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=group)
        if average_over:
            self.flat.div_(average_over)
        return self

    def as_dict(self) -> dict:
        return {k: self.view(k) for k in self.keys}
