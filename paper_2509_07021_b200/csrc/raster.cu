// raster.cu -- K5 forward and K6 backward tile rasterizers.
//
// Forward semantics (render.py:355-408, _chunk_blend / _render_params): per
// pixel, front to back over the depth-ordered primitives,
//   alpha = min(o * exp(-q/2), 0.99);  T_{i+1} = T_i (1 - alpha)
// primitive i is composited iff T_{i+1} >= 1e-4 (the kept set is a prefix),
// img = sum_i alpha_i T_i c_i + T_bg bg with T_bg the last kept transmittance.
// No alpha < 1/255 skip.  Pairs outside the opacity-aware support (q > qmax,
// i.e. o G < 1e-7) are skipped; see sgs_geom.h.
//
// One CTA per 16x16 tile, one pixel per thread.  Batches of 256 records of
// the tile's list are staged in shared memory (coalesced gather by sorted
// value), then every warp walks the batch in lock step; a warp leaves the
// batch once all of its pixels have terminated, the CTA leaves the tile once
// all 256 have (__syncthreads_count).
//
// Backward (render.py:535-573) walks each tile's list back to front from the
// last primitive any pixel kept, recovering T_i = T_{i+1} / (1 - alpha_i) and
// the suffix sum S_i = sum_{j>i} w_j (c_j . g) + T_bg (bg . g) exactly as the
// reference's reverse cumsum does, so
//   dL/dalpha_i = (T_i (c_i . g) - S_i / (1 - alpha_i)) [a_i < 0.99]
// Per-primitive partials are reduced across the warp with shuffles, across
// warps in shared memory, and flushed to HBM with one atomic per value per
// (primitive, tile).
#include "common.cuh"

namespace sgs {

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <bool kImportance, bool kCount>
__global__ void __launch_bounds__(256) raster_fwd_kernel(const uint2* __restrict__ ranges,
                                                         const uint32_t* __restrict__ vals,
                                                         const float4* __restrict__ rec_geo,
                                                         const float4* __restrict__ rec_con,
                                                         const float4* __restrict__ rec_col, SgsCam cam, float3 bg,
                                                         float* __restrict__ out_img, float* __restrict__ out_T,
                                                         uint32_t* __restrict__ out_nc,
                                                         float* __restrict__ weight_sums,
                                                         unsigned long long* __restrict__ pair_count) {
  __shared__ float4 s_geo[256];
  __shared__ float4 s_con[256];
  __shared__ float4 s_col[256];
  __shared__ uint32_t s_id[kImportance ? 256 : 1];

  const int tile = blockIdx.x + cam.tile_y0 * cam.tiles_x;
  const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
  const int t = threadIdx.x, lane = t & 31;
  const int px = tx * SGS_TILE + (t & 15), py = ty * SGS_TILE + (t >> 4);
  const bool inside = px < cam.width && py < cam.height;
  const float fx = (float)px + 0.5f, fy = (float)py + 0.5f;
  const uint2 rg = ranges[tile];
  const uint32_t start = rg.x, end = rg.y > rg.x ? rg.y : rg.x;

  float T = 1.0f, C0 = 0.0f, C1 = 0.0f, C2 = 0.0f;
  uint32_t nc = 0, reached = 0;
  bool done = !inside;

  for (uint32_t b = start; b < end; b += 256) {
    if (__syncthreads_count(done) == 256) break;
    const uint32_t j = b + t;
    if (j < end) {
      const uint32_t g = vals[j];
      s_geo[t] = rec_geo[g];
      s_con[t] = rec_con[g];
      s_col[t] = rec_col[g];
      if (kImportance) s_id[t] = g;
    }
    __syncthreads();
    const int nb = (int)min(256u, end - b);
    for (int k = 0; k < nb; ++k) {
      if (__all_sync(0xffffffffu, done)) break;
      const float4 G = s_geo[k];
      const float4 K = s_con[k];
      const float dx = fx - G.x, dy = fy - G.y;
      const float p = dx * (K.x * dx + K.y * dy) + K.z * dy * dy;
      float w = 0.0f;
      if (kCount && !done) ++reached;
      if (!done && p >= G.w) {
        const float a = G.z * ex2_approx(p);
        const float alpha = fminf(a, SGS_ALPHA_MAX);
        const float Tn = T * (a < SGS_ALPHA_MAX ? 1.0f - a : SGS_ONE_MINUS_ALPHA_MAX);
        if (Tn < SGS_T_KEEP) {
          done = true;
        } else {
          const float4 c = s_col[k];
          w = alpha * T;
          C0 += w * c.x;
          C1 += w * c.y;
          C2 += w * c.z;
          T = Tn;
          nc = b - start + k + 1;
        }
      }
      if (kImportance) {
        float ws = warp_sum(w);
        if (lane == 0 && ws != 0.0f) atomicAdd(&weight_sums[s_id[k]], ws);
      }
    }
  }
  if (kCount) {
    unsigned long long r = reached;
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    if (lane == 0 && r) atomicAdd(pair_count, r);
  }
  if (inside) {
    const size_t pix = (size_t)py * cam.width + px;
    out_img[3 * pix + 0] = C0 + T * bg.x;
    out_img[3 * pix + 1] = C1 + T * bg.y;
    out_img[3 * pix + 2] = C2 + T * bg.z;
    out_T[pix] = T;
    out_nc[pix] = nc;
  }
}

constexpr int kGrad = 9;

__global__ void __launch_bounds__(256) raster_bwd_kernel(const uint2* __restrict__ ranges,
                                                         const uint32_t* __restrict__ vals,
                                                         const float4* __restrict__ rec_geo,
                                                         const float4* __restrict__ rec_con,
                                                         const float4* __restrict__ rec_col, SgsCam cam, float3 bg,
                                                         const float* __restrict__ final_T,
                                                         const uint32_t* __restrict__ ncontrib,
                                                         const float* __restrict__ dimg, float* __restrict__ grad2d) {
  __shared__ float4 s_geo[256];
  __shared__ float4 s_con[256];
  __shared__ float4 s_col[256];
  __shared__ uint32_t s_id[256];
  __shared__ float s_acc[256][kGrad];
  __shared__ uint32_t s_max_nc;

  const int tile = blockIdx.x + cam.tile_y0 * cam.tiles_x;
  const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int px = tx * SGS_TILE + (t & 15), py = ty * SGS_TILE + (t >> 4);
  const bool inside = px < cam.width && py < cam.height;
  const float fx = (float)px + 0.5f, fy = (float)py + 0.5f;
  const uint2 rg = ranges[tile];
  const uint32_t start = rg.x;

  float T = 1.0f, g0 = 0.0f, g1 = 0.0f, g2 = 0.0f, S = 0.0f;
  uint32_t nc = 0;
  if (t == 0) s_max_nc = 0;
  __syncthreads();
  if (inside) {
    const size_t pix = (size_t)py * cam.width + px;
    T = final_T[pix];
    nc = ncontrib[pix];
    g0 = dimg[3 * pix + 0];
    g1 = dimg[3 * pix + 1];
    g2 = dimg[3 * pix + 2];
    S = T * (g0 * bg.x + g1 * bg.y + g2 * bg.z);
    atomicMax(&s_max_nc, nc);
  }
  __syncthreads();
  const uint32_t stop = start + s_max_nc;  // one past the last entry any pixel kept
  const uint32_t my_end = start + nc;

  for (uint32_t hi = stop; hi > start;) {
    const uint32_t lo = hi - start > 256 ? hi - 256 : start;
    const int nb = (int)(hi - lo);
    __syncthreads();  // previous batch fully flushed
    if (t < nb) {
      const uint32_t g = vals[lo + t];
      s_geo[t] = rec_geo[g];
      s_con[t] = rec_con[g];
      s_col[t] = rec_col[g];
      s_id[t] = g;
    }
    for (int c = 0; c < kGrad; ++c) s_acc[t][c] = 0.0f;
    __syncthreads();
    for (int k = nb - 1; k >= 0; --k) {
      const uint32_t idx = lo + k;
      if (__all_sync(0xffffffffu, idx >= my_end)) continue;
      const float4 G = s_geo[k];
      const float4 K = s_con[k];
      const float dx = fx - G.x, dy = fy - G.y;
      const float p = dx * (K.x * dx + K.y * dy) + K.z * dy * dy;
      bool active = idx < my_end && p >= G.w;
      float v[kGrad];
#pragma unroll
      for (int c = 0; c < kGrad; ++c) v[c] = 0.0f;
      if (active) {
        const float4 col = s_col[k];
        const float Gv = ex2_approx(p);
        const float a = G.z * Gv;
        const float alpha = fminf(a, SGS_ALPHA_MAX);
        const float om = a < SGS_ALPHA_MAX ? 1.0f - a : SGS_ONE_MINUS_ALPHA_MAX;
        const float Ti = T / om;
        const float w = alpha * Ti;
        const float cg = col.x * g0 + col.y * g1 + col.z * g2;
        const float dalpha = (a < SGS_ALPHA_MAX) ? (Ti * cg - S / om) : 0.0f;
        S += w * cg;
        T = Ti;
        const float dq = -0.5f * G.z * Gv * dalpha;
        v[0] = w * g0;
        v[1] = w * g1;
        v[2] = w * g2;
        v[3] = dq;
        v[4] = dq * dx;
        v[5] = dq * dy;
        v[6] = dq * dx * dx;
        v[7] = dq * dx * dy;
        v[8] = dq * dy * dy;
      }
      if (__any_sync(0xffffffffu, active)) {
#pragma unroll
        for (int c = 0; c < kGrad; ++c) v[c] = warp_sum(v[c]);
        if (lane < kGrad) {
          float mine = v[0];
#pragma unroll
          for (int c = 1; c < kGrad; ++c)
            if (lane == c) mine = v[c];
          atomicAdd(&s_acc[k][lane], mine);
        }
      }
    }
    __syncthreads();
    if (t < nb) {
      float* dst = grad2d + (size_t)s_id[t] * kGrad;
#pragma unroll
      for (int c = 0; c < kGrad; ++c) {
        const float x = s_acc[t][c];
        if (x != 0.0f) atomicAdd(dst + c, x);
      }
    }
    hi = lo;
  }
  (void)warp;
}

int launch_raster_fwd(const SgsCam& cam, float3 bg, const sgs_workspace* ws, const Layout& lo, const uint32_t* vals,
                      float* img, float* T, uint32_t* nc, float* weight_sums, unsigned long long* pairs,
                      cudaStream_t st) {
  const int grid = (cam.tile_y1 - cam.tile_y0) * cam.tiles_x;
  const uint2* ranges = at<uint2>(ws, lo.ranges);
  const float4* g = at<float4>(ws, lo.rec_geo);
  const float4* k = at<float4>(ws, lo.rec_con);
  const float4* c = at<float4>(ws, lo.rec_col);
  if (weight_sums && pairs)
    raster_fwd_kernel<true, true><<<grid, 256, 0, st>>>(ranges, vals, g, k, c, cam, bg, img, T, nc, weight_sums, pairs);
  else if (weight_sums)
    raster_fwd_kernel<true, false><<<grid, 256, 0, st>>>(ranges, vals, g, k, c, cam, bg, img, T, nc, weight_sums,
                                                         nullptr);
  else if (pairs)
    raster_fwd_kernel<false, true><<<grid, 256, 0, st>>>(ranges, vals, g, k, c, cam, bg, img, T, nc, nullptr, pairs);
  else
    raster_fwd_kernel<false, false><<<grid, 256, 0, st>>>(ranges, vals, g, k, c, cam, bg, img, T, nc, nullptr,
                                                          nullptr);
  SGS_LAUNCH_CHECK("raster_fwd_kernel");
  return SGS_OK;
}

int launch_raster_bwd(const SgsCam& cam, float3 bg, const sgs_workspace* ws, const Layout& lo, const uint32_t* vals,
                      const float* T, const uint32_t* nc, const float* dimg, float* grad2d, cudaStream_t st) {
  const int grid = (cam.tile_y1 - cam.tile_y0) * cam.tiles_x;
  SGS_CUDA(cudaMemsetAsync(grad2d, 0, (size_t)lo.n * kGrad * sizeof(float), st));
  raster_bwd_kernel<<<grid, 256, 0, st>>>(at<uint2>(ws, lo.ranges), vals, at<float4>(ws, lo.rec_geo),
                                          at<float4>(ws, lo.rec_con), at<float4>(ws, lo.rec_col), cam, bg, T, nc,
                                          dimg, grad2d);
  SGS_LAUNCH_CHECK("raster_bwd_kernel");
  return SGS_OK;
}

}  // namespace sgs
