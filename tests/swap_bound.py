"""Depth-swap bound: does sorting by the
fp32 depth key (float bits of z, ties by lower index) instead of the
reference's float64 z (render.py:262, 307: ``argsort(z, kind="stable")``)
change any pixel?

The reference computes z in float64 from the float64 camera; the build
computes it from the float32-rounded camera and keeps 32 bits.  Two
primitives closer in depth than that rounding can therefore come out in the
opposite order.  Swapping two adjacent layers a, b at a pixel changes its
colour by exactly T alpha_a alpha_b (c_a - c_b) (T = transmittance in front
of them), and by nothing when the pixel terminated in front of them
(render.py:378-388 keeps only the prefix with T_next >= 1e-4).

``swap_bound`` finds every pair that is inverted relative to the float64
order (within a window of 8 reference positions), keeps those whose tile
rectangles overlap, bounds alpha_a alpha_b |c_a - c_b| over pixel windows
around the pair (Appendix B: around each mean and their midpoint) and, for
the pixels where that bound exceeds ``floor``, evaluates T in front of the
pair from every emitting primitive ahead of it.  Inputs are the renderer's
own per-primitive outputs (Rasterizer.export_projected, or the CPU
restatement's preprocess -- bit-identical), so the analysis describes the
order the GPU actually used.  Test infrastructure only.
"""

from __future__ import annotations

import numpy as np

LOG2E = 1.4426950408889634
T_CUT = 1e-4


def f64_depth(position, cam) -> np.ndarray:
    """z exactly as the reference forms it: p.position @ W.T + t (render.py:262)."""
    W = np.asarray(cam.rotation, dtype=np.float64).reshape(3, 3)
    t = np.asarray(cam.translation, dtype=np.float64).reshape(3)
    return (np.asarray(position, dtype=np.float64) @ W.T + t)[:, 2]


def _alpha(rec, px, py):
    """alpha of records (k, 16) at pixel centres (px, py) (broadcast), from the
    eigen form the rasterizer evaluates: p = log2 o - t1^2 - t2^2."""
    mx, my, lo = rec[:, 0:1], rec[:, 1:2], rec[:, 2:3]
    e1, e2, e3, e4 = (rec[:, 8 + k:9 + k] for k in range(4))
    dx, dy = px[None, :] - mx, py[None, :] - my
    t1 = e1 * dx + e2 * dy
    t2 = e3 * dy - e4 * dx
    return np.minimum(np.exp2(lo - t1 * t1 - t2 * t2), 0.99)


def swap_bound(z64, depth_bits, rect, tiles_touched, records, width, height, window=8, floor=1e-6,
               half=3, max_eval=10**7, depth_res=None):
    """Returns a dict of counts and the largest swap effect found.  The order
    analysed is the float32 key order with ties by index or, with
    ``depth_res``, ties by the float64 residual first (the build's order)."""
    emit = np.flatnonzero(np.asarray(tiles_touched) > 0)
    out = {"emitting": int(emit.size), "inverted_pairs": 0, "overlapping_pairs": 0,
           "pairs_above_floor": 0, "pixels_evaluated": 0, "max_bound": 0.0, "max_effect": 0.0,
           "max_effect_T": None}
    if emit.size < 2:
        return out
    z64 = np.asarray(z64, np.float64)
    db = np.asarray(depth_bits).view(np.uint32).astype(np.int64)
    ref = emit[np.argsort(z64[emit], kind="stable")]
    if depth_res is None:
        gpu = emit[np.lexsort((emit, db[emit]))]      # float bits, ties by lower index
    else:                                             # float bits, then the float64 residual, then index
        gpu = emit[np.lexsort((emit, np.asarray(depth_res)[emit], db[emit]))]
    rank = np.empty(int(emit.max()) + 1, np.int64)
    rank[gpu] = np.arange(gpu.size)
    r32 = np.asarray(rect).view(np.uint32)
    tx0, tx1 = (r32[:, 0] & 0xffff).astype(np.int64), (r32[:, 0] >> 16).astype(np.int64)
    ty0, ty1 = (r32[:, 1] & 0xffff).astype(np.int64), (r32[:, 1] >> 16).astype(np.int64)
    rec = np.asarray(records, np.float64)
    pairs = []
    for k in range(1, window + 1):
        a, b = ref[:-k], ref[k:]           # a in front of b in the reference order
        inv = rank[a] > rank[b]
        if not inv.any():
            continue
        a, b = a[inv], b[inv]
        out["inverted_pairs"] += int(a.size)
        ov = (np.maximum(tx0[a], tx0[b]) <= np.minimum(tx1[a], tx1[b])) & \
             (np.maximum(ty0[a], ty0[b]) <= np.minimum(ty1[a], ty1[b]))
        pairs.append(np.stack([a[ov], b[ov]], 1))
    pairs = np.concatenate(pairs) if pairs else np.zeros((0, 2), np.int64)
    out["overlapping_pairs"] = int(len(pairs))
    if not len(pairs):
        return out
    off = np.arange(-half, half + 1, dtype=np.float64)
    wx, wy = np.meshgrid(off, off)
    wx, wy = wx.ravel(), wy.ravel()
    evals = 0
    for a, b in pairs:
        ca, cb = rec[a, 12:15], rec[b, 12:15]
        dc = float(np.abs(ca - cb).max())
        if dc == 0.0:
            continue
        centres = [(rec[a, 0], rec[a, 1]), (rec[b, 0], rec[b, 1]),
                   (0.5 * (rec[a, 0] + rec[b, 0]), 0.5 * (rec[a, 1] + rec[b, 1]))]
        px = np.concatenate([np.floor(cx) + 0.5 + wx for cx, _ in centres])
        py = np.concatenate([np.floor(cy) + 0.5 + wy for _, cy in centres])
        on = (px > 0) & (px < width) & (py > 0) & (py < height)
        px, py = px[on], py[on]
        if px.size == 0:
            continue
        aa = _alpha(rec[[a]], px, py)[0]
        ab = _alpha(rec[[b]], px, py)[0]
        bound = aa * ab * dc
        out["max_bound"] = max(out["max_bound"], float(bound.max()))
        hot = bound > floor
        if not hot.any():
            continue
        out["pairs_above_floor"] += 1
        first = min(rank[a], rank[b])
        ahead = gpu[:first]
        hx, hy, hb = px[hot], py[hot], bound[hot]
        tiles = (hx // 16).astype(np.int64) + 100000 * (hy // 16).astype(np.int64)
        for tkey in np.unique(tiles):
            if evals >= max_eval:
                out["truncated"] = True
                break
            sel = tiles == tkey
            tx, ty = int(tkey % 100000), int(tkey // 100000)
            cand = ahead[(tx0[ahead] <= tx) & (tx1[ahead] >= tx) & (ty0[ahead] <= ty) & (ty1[ahead] >= ty)]
            evals += int(sel.sum())
            if cand.size:
                al = _alpha(rec[cand], hx[sel], hy[sel])            # (k, p) in GPU order
                T = np.cumprod(1.0 - al, axis=0)
                alive = T.min(axis=0) >= T_CUT                      # not terminated in front of the pair
                Tb = T[-1]
            else:
                alive = np.ones(int(sel.sum()), bool)
                Tb = np.ones(int(sel.sum()))
            eff = np.where(alive, Tb * hb[sel], 0.0)
            j = int(np.argmax(eff))
            if eff[j] > out["max_effect"]:
                out["max_effect"], out["max_effect_T"] = float(eff[j]), float(Tb[j])
    out["pixels_evaluated"] = evals
    return out
