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


def row_costs_measured(ncontrib, entry_rows, raster_ms: float, bin_ms: float, tile: int = 16) -> np.ndarray:
    """Per-tile-row cost (ms) of one frame from a measured render: raster
    time spread over the rows in proportion to the kept (pixel, record)
    pairs (the forward's per-pixel contributor counts, summed per row) and
    binning time in proportion to the tile entries (``entry_rows``, e.g.
    row_costs_from_rects).  Tile entries alone mis-predict the raster: dense
    central rows terminate early (configs[4]: 0.23 ms for a central eighth
    of the frame against 1.0 ms for an edge eighth with as many entries)."""
    nc = np.asarray(ncontrib, dtype=np.float64)
    rows = -(-nc.shape[0] // tile)
    pad = np.zeros((rows * tile,) + nc.shape[1:])
    pad[:nc.shape[0]] = nc
    pairs = pad.reshape(rows, -1).sum(axis=1)
    ent = np.asarray(entry_rows, dtype=np.float64)[:rows]
    cost = np.zeros(rows)
    if pairs.sum() > 0:
        cost += raster_ms * pairs / pairs.sum()
    if ent.sum() > 0:
        cost += bin_ms * ent / ent.sum()
    return cost


def refine_row_costs(row_cost, strips, strip_ms) -> np.ndarray:
    """One refinement step of a strip plan from measured strip times: the
    rows of each strip are rescaled so they sum to that strip's measured
    time (which includes what a per-row model misses -- each strip projects
    and depth-sorts every primitive overlapping it), keeping the within-strip
    shape.  balanced_strips on the result re-plans."""
    cost = np.asarray(row_cost, dtype=np.float64).copy()
    for (y0, y1), t in zip(strips, strip_ms):
        s = cost[y0:y1].sum()
        if y1 > y0:
            cost[y0:y1] = cost[y0:y1] * (t / s) if s > 0 else t / (y1 - y0)
    return cost


class GradBucket:
    """Flatten a dict of gradient tensors into one contiguous buffer and
    scatter it back.

    ``chunks == 1``: field-major (every field contiguous; one all-reduce).
    ``chunks > 1`` (``n`` = the shared leading dimension, the primitive
    count): chunk-major -- primitive range c holds every field's rows of that
    range contiguously -- so chunk c can be all-reduced as soon as the
    parameter backward of its rows is done, while later chunks are still
    being accumulated (the overlapped, bucketed reduction of SURVEY §8(e)).
    Every field row block starts on a 16-byte boundary (float4 rows)."""

    def __init__(self, shapes: dict, device, dtype=torch.float32, chunks: int = 1, n: int | None = None):
        self.keys = list(shapes)
        self.shapes = {k: tuple(shapes[k]) for k in self.keys}
        self.sizes = {k: int(np.prod(self.shapes[k])) for k in self.keys}
        self.chunks = max(1, int(chunks))
        if self.chunks > 1:
            n = int(n if n is not None else self.shapes[self.keys[0]][0])
            if any(self.shapes[k][0] != n for k in self.keys):
                raise ValueError("chunked buckets need a common leading dimension")
            per = -(-n // self.chunks)
            per = (per + 3) // 4 * 4
            self.bounds = [(min(c * per, n), min((c + 1) * per, n)) for c in range(self.chunks)]
        else:
            self.bounds = [(0, None)]
        self.offsets = {}
        self.chunk_off = []
        off = 0
        for c, (p0, p1) in enumerate(self.bounds):
            self.chunk_off.append(off)
            for k in self.keys:
                rows = self.shapes[k][0] if self.chunks == 1 else p1 - p0
                size = self.sizes[k] if self.chunks == 1 else rows * int(np.prod(self.shapes[k][1:]))
                self.offsets[(k, c)] = (off, size)
                off += (size + 3) // 4 * 4
        self.chunk_off.append(off)
        self.numel = off
        self.flat = torch.zeros(off, device=device, dtype=dtype)

    def zero(self):
        self.flat.zero_()

    def chunk_view(self, k, c: int = 0) -> torch.Tensor:
        o, size = self.offsets[(k, c)]
        if self.chunks == 1:
            return self.flat[o:o + size].view(self.shapes[k])
        p0, p1 = self.bounds[c]
        return self.flat[o:o + size].view((p1 - p0,) + self.shapes[k][1:])

    def chunk_flat(self, c: int) -> torch.Tensor:
        return self.flat[self.chunk_off[c]:self.chunk_off[c + 1]]

    def view(self, k) -> torch.Tensor:
        if self.chunks != 1:
            raise ValueError("a chunked bucket has no single view per field; use chunk_view / as_dict")
        return self.chunk_view(k, 0)

    def add_(self, grads: dict):
        for k in self.keys:
            if k in grads and grads[k] is not None:
                for c, (p0, p1) in enumerate(self.bounds):
                    src = grads[k] if self.chunks == 1 else grads[k][p0:p1]
                    self.chunk_view(k, c).add_(src.to(self.flat.dtype))

    def allreduce_(self, group=None, average_over: float | None = None):
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=group)
        if average_over:
            self.flat.div_(average_over)
        return self

    def as_dict(self) -> dict:
        if self.chunks == 1:
            return {k: self.chunk_view(k, 0) for k in self.keys}
        return {k: torch.cat([self.chunk_view(k, c) for c in range(self.chunks)]) for k in self.keys}
