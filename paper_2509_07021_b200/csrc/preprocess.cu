// preprocess.cu -- K1: per-primitive projection, culling, support rectangle,
// exact ellipse-tile counts and SG color.  Replaces _prepare
// (/root/reference/pkg/src/sgsplat/render.py:259-317) minus the argsort, and
// the reference VRAM model's 3-sigma counts (postprocess.py:118-135).
//
// One thread per primitive, grid-stride over N.  The arithmetic lives in
// sgs_geom.h so the CPU restatement (oracle/) reproduces every bit that feeds
// a tile key.  HBM-bound: ~156 B read + 60 B written per primitive.
#include "common.cuh"

namespace sgs {

constexpr int kPreSlots = 256;  // (primitive, super row) union slots per warp

__device__ __forceinline__ void warp_count(unsigned long long* ctr, bool pred) {
  unsigned m = __ballot_sync(0xffffffffu, pred);
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(ctr, (unsigned long long)__popc(m));
}

// The exact tile counts are the expensive part: one ellipse-row span (two
// quadratic roots) per tile row the support rectangle covers, and the row
// count varies 1..>10 across a warp.  They are computed warp-cooperatively:
// the warp's primitives' tile rows are flattened into one list and processed
// 32 at a time, lane = tile row; each row's tile count is summed into its
// primitive's shared-memory slot and its super-tile columns are merged into
// the (primitive, super row) slot, from which each primitive then sums its
// super-tile count.  The spans are sgs_row_span -- the definition the
// emission and the CPU restatement use -- so the counts agree bit for bit.
// Warps whose rectangles are tall use super-row items instead (four rows per
// lane; rows outside the rectangle evaluated and masked), which need fewer
// item iterations when little is masked.
template <int kL>
#ifndef SGS_PRE_CTAS
#define SGS_PRE_CTAS 3
#endif
#ifndef SGS_PRE_REG_CTAS
#define SGS_PRE_REG_CTAS SGS_PRE_CTAS
#endif
__global__ void __launch_bounds__(256, SGS_PRE_REG_CTAS) preprocess_kernel(sgs_params P, SgsCam cam, float4* __restrict__ rec_geo,
                                                         float4* __restrict__ rec_con, float4* __restrict__ rec_col,
                                                         float4* __restrict__ rec_span,
                                                         float4* __restrict__ rec_eig,
                                                         uint32_t* __restrict__ depth_key,
                                                         float* __restrict__ depth_res, uint2* __restrict__ rect,
                                                         uint32_t* __restrict__ tiles_touched,
                                                         uint32_t* __restrict__ super_touched,
                                                         uint32_t* __restrict__ depth_hist,
                                                         uint32_t* __restrict__ row_off, uint16_t* __restrict__ row_spans,
                                                         uint32_t row_cap, Counters* ctr) {
  __shared__ uint32_t s_cnt[8][32], s_sup[8][32];
  // per warp: (primitive, super row) slots of the super-tile column union
  __shared__ int s_lo[8][kPreSlots], s_hi[8][kPreSlots];
  __shared__ uint32_t s_hist[4][256];  // depth-key digit counts of this CTA's primitives
  if (depth_hist) {
    for (int j = threadIdx.x; j < 4 * 256; j += blockDim.x) (&s_hist[0][0])[j] = 0;
    __syncthreads();
  }
  const int64_t n = P.n;
  const int L = kL > 0 ? kL : P.n_lobes;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool window = cam.tile_y0 > 0 || cam.tile_y1 < cam.tiles_y;  // strip render
  if (depth_hist && !window && blockIdx.x == 0 && threadIdx.x == 0) ctr->n_depth = (uint32_t)n;
  // iterate whole warps so the ballots and the cooperative row loop see converged warps
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const int64_t i = base + threadIdx.x;
    const bool live = i < n;
    bool visible = false;
    SgsProj pr;
    pr.emits = 0;
    pr.tx0 = pr.ty0 = 0;
    pr.tx1 = pr.ty1 = -1;
    float pos[3] = {0.0f, 0.0f, 0.0f};
    float g[4], k[4];
    SgsSpan sp;
    sp.valid = 0;
    if (live) {
      pos[0] = P.position[3 * i];
      pos[1] = P.position[3 * i + 1];
      pos[2] = P.position[3 * i + 2];
      float4 q4 = reinterpret_cast<const float4*>(P.quat)[i];
      float quat[4] = {q4.x, q4.y, q4.z, q4.w};
      float ls[3] = {P.log_scale[3 * i], P.log_scale[3 * i + 1], P.log_scale[3 * i + 2]};
      float pm = P.prim_mask ? P.prim_mask[i] : 1.0f;
      sgs_project(pos, quat, ls, P.opacity[i], pm, &cam, &pr);
      visible = pr.visible;
      if (pr.emits) {
        sgs_pack_geo(&pr, g, k);
        sp = sgs_span(g, k);
      }
    }
    // tile-row items (no masked rows) unless the warp's rectangles are tall
    // enough that four-row super-row items waste little (<= 20 % masked rows)
    // and need fewer item iterations
    uint32_t my_off, cnt, nsup;
    bool tile_rows;
    {
      const uint32_t rows_w = __reduce_add_sync(0xffffffffu, pr.emits ? (uint32_t)(pr.ty1 - pr.ty0 + 1) : 0u);
      const uint32_t srows_w =
          __reduce_add_sync(0xffffffffu, pr.emits ? (uint32_t)(pr.ty1 / SGS_SUPER - pr.ty0 / SGS_SUPER + 1) : 0u);
      tile_rows = 4ull * SGS_SUPER * srows_w > 5ull * rows_w;
    }
    if (tile_rows) {
      // ---- exact counts, one tile row per lane (the rows of the warp's
      // primitives flattened: no masked rows, full lanes); each row's span is
      // stored, and its super-tile columns are merged into its (primitive,
      // super row) slot with shared-memory min / max
      const uint32_t nrows_all = pr.emits ? (uint32_t)(pr.ty1 - pr.ty0 + 1) : 0u;
      const uint32_t nsr = pr.emits ? (uint32_t)(pr.ty1 / SGS_SUPER - pr.ty0 / SGS_SUPER + 1) : 0u;
      const uint32_t sincl = warp_incl_scan(nsr, lane);
      const uint32_t sbase = sincl - nsr;
      const bool slots_ok = __shfl_sync(0xffffffffu, sincl, 31) <= (uint32_t)kPreSlots;  // warp-uniform
      s_cnt[warp][lane] = 0;
      if (slots_ok)
        for (uint32_t j = lane; j < (uint32_t)kPreSlots; j += 32) {
          s_lo[warp][j] = 0x7fffffff;
          s_hi[warp][j] = -1;
        }
      __syncwarp();
      const uint32_t incl = warp_incl_scan(nrows_all, lane);
      const uint32_t start = incl - nrows_all;
      const uint32_t R = __shfl_sync(0xffffffffu, incl, 31);
      // row-span store: one u16 (first column - tx0 | count << 8) per tile row of
      // the support rectangle, space handed out per warp; primitives that do not
      // fit (store full, or wider than 255 tiles) are re-solved by the emission
      my_off = kNoRows;
      if (row_spans) {
        const uint32_t nrows = pr.tx1 - pr.tx0 < 255 ? nrows_all : 0u;
        const uint32_t rincl = warp_incl_scan(nrows, lane);
        const uint32_t rtot = __shfl_sync(0xffffffffu, rincl, 31);
        uint32_t rbase = 0;
        if (lane == 31 && rtot) rbase = atomicAdd(&ctr->row_alloc, rtot);
        rbase = __shfl_sync(0xffffffffu, rbase, 31);
        if (nrows && (uint64_t)rbase + rincl <= row_cap) my_off = rbase + rincl - nrows;
      }
      for (uint32_t k0 = 0; k0 < R; k0 += 32) {
        const uint32_t kk = k0 + lane;
        const int owner = lane_search(start, kk < R ? kk : R - 1);
        const SgsSpan os = shfl_span(sp, owner);
        const int otx0 = __shfl_sync(0xffffffffu, pr.tx0, owner);
        const int oty0 = __shfl_sync(0xffffffffu, pr.ty0, owner);
        const int otx1 = __shfl_sync(0xffffffffu, pr.tx1, owner);
        const uint32_t ostart = __shfl_sync(0xffffffffu, start, owner);
        const uint32_t ooff = __shfl_sync(0xffffffffu, my_off, owner);
        const uint32_t osb = __shfl_sync(0xffffffffu, sbase, owner);
        if (kk < R) {
          const int ty = oty0 + (int)(kk - ostart);
          int f;
          const int c = sgs_row_span(&os, &cam, ty, otx0, otx1, &f);
          if (c) {
            atomicAdd(&s_cnt[warp][owner], (uint32_t)c);
            if (slots_ok) {
              const uint32_t slot = osb + (uint32_t)(ty / SGS_SUPER - oty0 / SGS_SUPER);
              atomicMin(&s_lo[warp][slot], f / SGS_SUPER);
              atomicMax(&s_hi[warp][slot], (f + c - 1) / SGS_SUPER);
            }
          }
          if (ooff != kNoRows)
            row_spans[ooff + (kk - ostart)] = (uint16_t)(c > 0 ? (((f - otx0) & 0xff) | (c << 8)) : 0);
        }
      }
      __syncwarp();
      cnt = s_cnt[warp][lane];
      nsup = 0;
      if (cnt) {
        if (slots_ok) {
          for (uint32_t j = 0; j < nsr; ++j) {
            const int lo = s_lo[warp][sbase + j], hi = s_hi[warp][sbase + j];
            if (hi >= lo) nsup += (uint32_t)(hi - lo + 1);
          }
        } else {
          // more super rows in this warp than slots: each primitive reads its
          // stored row spans back (the __syncwarp above orders the stores), or
          // re-solves them when they were not stored
          for (int sr = pr.ty0 / SGS_SUPER; sr <= pr.ty1 / SGS_SUPER; ++sr) {
            if (my_off != kNoRows) {
              int lo = 0x7fffffff, hi = -1;
  #pragma unroll
              for (int q = 0; q < SGS_SUPER; ++q) {
                const int ty = sr * SGS_SUPER + q;
                if (ty < pr.ty0 || ty > pr.ty1) continue;
                const uint32_t e = row_spans[my_off + (uint32_t)(ty - pr.ty0)];
                const int c = (int)(e >> 8);
                if (c > 0) {
                  const int f = pr.tx0 + (int)(e & 0xffu);
                  lo = min(lo, f / SGS_SUPER);
                  hi = max(hi, (f + c - 1) / SGS_SUPER);
                }
              }
              if (hi >= lo) nsup += (uint32_t)(hi - lo + 1);
            } else {
              int rf[SGS_SUPER], rc[SGS_SUPER], fsc;
              nsup += (uint32_t)sgs_super_row_spans(&sp, &cam, pr.tx0, pr.ty0, pr.tx1, pr.ty1, sr, rf, rc, &fsc);
            }
          }
        }
      }
    } else {
      // ---- exact counts, one super-tile row per lane
      const uint32_t nitems = pr.emits ? (uint32_t)(pr.ty1 / SGS_SUPER - pr.ty0 / SGS_SUPER + 1) : 0u;
      s_cnt[warp][lane] = 0;
      s_sup[warp][lane] = 0;
      __syncwarp();
      const uint32_t incl = warp_incl_scan(nitems, lane);
      const uint32_t start = incl - nitems;
      const uint32_t R = __shfl_sync(0xffffffffu, incl, 31);
      // row-span store: one u16 (first column - tx0 | count << 8) per tile row of
      // the support rectangle, space handed out per warp; primitives that do not
      // fit (store full, or wider than 255 tiles) are re-solved by the emission
      my_off = kNoRows;
      if (row_spans) {
        const uint32_t nrows = pr.emits && pr.tx1 - pr.tx0 < 255 ? (uint32_t)(pr.ty1 - pr.ty0 + 1) : 0u;
        const uint32_t rincl = warp_incl_scan(nrows, lane);
        const uint32_t rtot = __shfl_sync(0xffffffffu, rincl, 31);
        uint32_t rbase = 0;
        if (lane == 31 && rtot) rbase = atomicAdd(&ctr->row_alloc, rtot);
        rbase = __shfl_sync(0xffffffffu, rbase, 31);
        if (nrows && (uint64_t)rbase + rincl <= row_cap) my_off = rbase + rincl - nrows;
      }
      for (uint32_t k0 = 0; k0 < R; k0 += 32) {
        const uint32_t kk = k0 + lane;
        const int owner = lane_search(start, kk < R ? kk : R - 1);
        const SgsSpan os = shfl_span(sp, owner);
        const int otx0 = __shfl_sync(0xffffffffu, pr.tx0, owner);
        const int oty0 = __shfl_sync(0xffffffffu, pr.ty0, owner);
        const int otx1 = __shfl_sync(0xffffffffu, pr.tx1, owner);
        const int oty1 = __shfl_sync(0xffffffffu, pr.ty1, owner);
        const uint32_t ostart = __shfl_sync(0xffffffffu, start, owner);
        const uint32_t ooff = __shfl_sync(0xffffffffu, my_off, owner);
        if (kk < R) {
          const int sr = oty0 / SGS_SUPER + (int)(kk - ostart);
          int rf[SGS_SUPER], rc[SGS_SUPER], fsc;
          const int nsc = sgs_super_row_spans(&os, &cam, otx0, oty0, otx1, oty1, sr, rf, rc, &fsc);
          const uint32_t nt = (uint32_t)(rc[0] + rc[1] + rc[2] + rc[3]);
          if (nt) atomicAdd(&s_cnt[warp][owner], nt);
          if (nsc) atomicAdd(&s_sup[warp][owner], (uint32_t)nsc);
          if (ooff != kNoRows) {
  #pragma unroll
            for (int j = 0; j < SGS_SUPER; ++j) {
              const int ty = sr * SGS_SUPER + j;
              if (ty >= oty0 && ty <= oty1)
                row_spans[ooff + (uint32_t)(ty - oty0)] =
                    (uint16_t)(rc[j] > 0 ? (((rf[j] - otx0) & 0xff) | (rc[j] << 8)) : 0);
            }
          }
        }
      }
      __syncwarp();
      cnt = s_cnt[warp][lane];
      nsup = s_sup[warp][lane];
    }
    const bool emitting = cnt > 0;
    if (live) {
      tiles_touched[i] = cnt;
      super_touched[i] = nsup;
      if (row_off) row_off[i] = cnt ? my_off : kNoRows;
      const uint32_t dk = emitting ? sgs_float_to_bits(pr.depth) : 0x7fffffffu;
      depth_key[i] = dk;
      depth_res[i] = emitting ? pr.depth_res : 0.0f;
      if (depth_hist && emitting) {
#pragma unroll
        for (int d = 0; d < 4; ++d) atomicAdd(&s_hist[d][(dk >> (8 * d)) & 0xffu], 1u);
      }
      rect[i] = make_uint2((uint32_t)(pr.tx0 & 0xffff) | ((uint32_t)(pr.tx1 & 0xffff) << 16),
                           (uint32_t)(pr.ty0 & 0xffff) | ((uint32_t)(pr.ty1 & 0xffff) << 16));
      if (emitting) {
        float diffuse[3] = {P.diffuse[3 * i], P.diffuse[3 * i + 1], P.diffuse[3 * i + 2]};
        float axis[3 * SGS_MAX_LOBES], sharp[SGS_MAX_LOBES], amp[3 * SGS_MAX_LOBES], lm[SGS_MAX_LOBES];
#pragma unroll
        for (int l = 0; l < (kL > 0 ? kL : SGS_MAX_LOBES); ++l) {
          if (kL == 0 && l >= L) break;
          sharp[l] = P.sharpness[i * L + l];
          lm[l] = P.lobe_mask[i * L + l];
#pragma unroll
          for (int kk = 0; kk < 3; ++kk) {
            axis[3 * l + kk] = P.axis_raw[(i * L + l) * 3 + kk];
            amp[3 * l + kk] = P.amplitude[(i * L + l) * 3 + kk];
          }
        }
        float c_pre[3], c[3];
        sgs_color(pos, diffuse, axis, sharp, amp, lm, L, &cam, c_pre, c);
        float span2[3];
        sgs_span_cache(&sp, &k[3], span2);
        rec_geo[i] = make_float4(g[0], g[1], g[2], g[3]);
        rec_con[i] = make_float4(k[0], k[1], k[2], k[3]);
        rec_span[i] = make_float4(span2[0], span2[1], span2[2], 0.0f);
        float e4[4];
        sgs_pack_eig(&pr, e4);
        rec_eig[i] = make_float4(e4[0], e4[1], e4[2], e4[3]);
        rec_col[i] = make_float4(c[0], c[1], c[2], 0.0f);
      }
    }
    if (depth_hist && !window) {
      // full frames sort every primitive: the not-emitting key 0x7fffffff
      // counted once per warp (32 lanes on the same four shared counters
      // would serialise).  Strip renders sort only the emitting primitives
      // (compacted by compact_depth_keys), so they are not counted there.
      const uint32_t m = __ballot_sync(0xffffffffu, live && !emitting);
      if (lane == 0 && m) {
        const uint32_t c = (uint32_t)__popc(m);
        atomicAdd(&s_hist[0][0xffu], c);
        atomicAdd(&s_hist[1][0xffu], c);
        atomicAdd(&s_hist[2][0xffu], c);
        atomicAdd(&s_hist[3][0x7fu], c);
      }
    }
    warp_count(&ctr->n_visible, visible);
    warp_count(&ctr->n_emitting, emitting);
    unsigned long long e = cnt;
    for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
    if (lane == 0 && e) atomicAdd(&ctr->n_entries, e);
  }
  if (depth_hist) {
    __syncthreads();
    for (int j = threadIdx.x; j < 4 * 256; j += blockDim.x) {
      const uint32_t v = (&s_hist[0][0])[j];
      if (v) atomicAdd(&depth_hist[j], v);
    }
  }
}

// Reference VRAM model: 3-sigma per-axis AABB, strict on-image test, floor /
// clip tile rectangle (postprocess.py:118-135), in fp32 on the same
// projection as the renderer.
__global__ void __launch_bounds__(256) vram3s_kernel(sgs_params P, SgsCam cam, int tile_px, Counters* ctr) {
  const int64_t n = P.n;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int tiles_x = (cam.width + tile_px - 1) / tile_px, tiles_y = (cam.height + tile_px - 1) / tile_px;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const int64_t i = base + threadIdx.x;
    bool on = false;
    unsigned long long ent = 0;
    if (i < n) {
      float pos[3] = {P.position[3 * i], P.position[3 * i + 1], P.position[3 * i + 2]};
      float4 q4 = reinterpret_cast<const float4*>(P.quat)[i];
      float quat[4] = {q4.x, q4.y, q4.z, q4.w};
      float ls[3] = {P.log_scale[3 * i], P.log_scale[3 * i + 1], P.log_scale[3 * i + 2]};
      SgsProj pr;
      sgs_project(pos, quat, ls, 1.0f, 1.0f, &cam, &pr);
      if (pr.visible) {
        float rx = F_MUL(3.0f, F_SQRT(pr.cov00)), ry = F_MUL(3.0f, F_SQRT(pr.cov11));
        float x0 = F_SUB(pr.mx, rx), x1 = F_ADD(pr.mx, rx), y0 = F_SUB(pr.my, ry), y1 = F_ADD(pr.my, ry);
        on = x1 > 0.0f && x0 < (float)cam.width && y1 > 0.0f && y0 < (float)cam.height;
        if (on) {
          float t = (float)tile_px;
          int tx0 = (int)fminf(fmaxf(F_FLOOR(F_DIV(x0, t)), 0.0f), (float)(tiles_x - 1));
          int tx1 = (int)fminf(fmaxf(F_FLOOR(F_DIV(x1, t)), 0.0f), (float)(tiles_x - 1));
          int ty0 = (int)fminf(fmaxf(F_FLOOR(F_DIV(y0, t)), 0.0f), (float)(tiles_y - 1));
          int ty1 = (int)fminf(fmaxf(F_FLOOR(F_DIV(y1, t)), 0.0f), (float)(tiles_y - 1));
          ent = (unsigned long long)(tx1 - tx0 + 1) * (unsigned long long)(ty1 - ty0 + 1);
        }
      }
    }
    warp_count(&ctr->vram3s_visible, on);
    for (int o = 16; o > 0; o >>= 1) ent += __shfl_xor_sync(0xffffffffu, ent, o);
    if ((threadIdx.x & 31) == 0 && ent) atomicAdd(&ctr->vram3s_entries, ent);
  }
}

// Per-primitive projection record for the host API's _prepare / project
// (render.py:259-330): [visible, depth, mean2d(2), cov2d 00/01/11, conic
// 00/01/11, color_pre(3), color(3)], 16 floats, every primitive.
__global__ void __launch_bounds__(256) project_records_kernel(sgs_params P, SgsCam cam, float* __restrict__ out) {
  const int64_t n = P.n;
  const int L = P.n_lobes;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float pos[3] = {P.position[3 * i], P.position[3 * i + 1], P.position[3 * i + 2]};
    float4 q4 = reinterpret_cast<const float4*>(P.quat)[i];
    float quat[4] = {q4.x, q4.y, q4.z, q4.w};
    float ls[3] = {P.log_scale[3 * i], P.log_scale[3 * i + 1], P.log_scale[3 * i + 2]};
    SgsProj pr;
    sgs_project(pos, quat, ls, P.opacity[i], P.prim_mask ? P.prim_mask[i] : 1.0f, &cam, &pr);
    float* o = out + 16 * i;
    for (int k = 0; k < 16; ++k) o[k] = 0.0f;
    o[0] = pr.visible ? 1.0f : 0.0f;
    o[1] = pr.depth;
    if (!pr.visible) continue;
    o[2] = pr.mx;
    o[3] = pr.my;
    o[4] = pr.cov00;
    o[5] = pr.cov01;
    o[6] = pr.cov11;
    o[7] = pr.con00;
    o[8] = pr.con01;
    o[9] = pr.con11;
    float diffuse[3] = {P.diffuse[3 * i], P.diffuse[3 * i + 1], P.diffuse[3 * i + 2]};
    float c_pre[3], c[3];
    sgs_color(pos, diffuse, P.axis_raw + (size_t)i * L * 3, P.sharpness + (size_t)i * L,
              P.amplitude + (size_t)i * L * 3, P.lobe_mask + (size_t)i * L, L, &cam, c_pre, c);
    for (int k = 0; k < 3; ++k) {
      o[10 + k] = c_pre[k];
      o[13 + k] = c[k];
    }
  }
}

int launch_project_records(const sgs_params& P, const SgsCam& cam, float* out, cudaStream_t st) {
  int grid = persistent_grid((uint64_t)P.n, 256, 8);
  project_records_kernel<<<grid, 256, 0, st>>>(P, cam, out);
  SGS_LAUNCH_CHECK("project_records_kernel");
  return SGS_OK;
}

int launch_preprocess(const sgs_params& P, const SgsCam& cam, const sgs_workspace* ws, const Layout& lo,
                      cudaStream_t st) {
  Counters* ctr = at<Counters>(ws, lo.counters);
  int grid = persistent_grid((uint64_t)P.n, 256, SGS_PRE_CTAS);  // one wave of resident CTAs
#define SGS_PRE(KL)                                                                                             \
  preprocess_kernel<KL><<<grid, 256, 0, st>>>(P, cam, at<float4>(ws, lo.rec_geo), at<float4>(ws, lo.rec_con),    \
                                              at<float4>(ws, lo.rec_col), at<float4>(ws, lo.rec_span),           \
                                              at<float4>(ws, lo.rec_eig), at<uint32_t>(ws, lo.depth_key),        \
                                              at<float>(ws, lo.depth_res),                                        \
                                              at<uint2>(ws, lo.rect), at<uint32_t>(ws, lo.tiles_touched),        \
                                              at<uint32_t>(ws, lo.super_touched),                                 \
                                              at<uint32_t>(ws, lo.hist) + kDepthHistOff,                         \
                                              lo.row_cap ? at<uint32_t>(ws, lo.row_off) : nullptr,                 \
                                              lo.row_cap ? at<uint16_t>(ws, lo.row_spans) : nullptr,               \
                                              (uint32_t)lo.row_cap, ctr)
  if (P.n_lobes == 3)
    SGS_PRE(3);
  else
    SGS_PRE(0);
#undef SGS_PRE
  SGS_LAUNCH_CHECK("preprocess_kernel");
  return SGS_OK;
}

int launch_vram3s(const sgs_params& P, const SgsCam& cam, int tile_px, Counters* ctr, cudaStream_t st) {
  int grid = persistent_grid((uint64_t)P.n, 256, 8);
  vram3s_kernel<<<grid, 256, 0, st>>>(P, cam, tile_px, ctr);
  SGS_LAUNCH_CHECK("vram3s_kernel");
  return SGS_OK;
}

}  // namespace sgs
