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
// One CTA per 16x16 tile.  The tile's primitive list is read from its cell's
// sorted list -- the super-tile list in depth-first mode, filtered to this
// tile by the tile's bit of the exact 16-bit membership mask each entry carries, or the
// tile's own list in 64-bit-key mode -- in batches that are compacted
// (stable) into shared memory.  The per-tile list index of a staged entry is
// its rank among the tile's hits, identical in both modes.
//
// Backward (render.py:535-573) walks each tile's list back to front from the
// last entry any pixel kept (the forward records that candidate position per
// tile), recovering T_i = T_{i+1} / (1 - alpha_i) and the suffix sum
// S_i = sum_{j>i} w_j (c_j . g) + T_bg (bg . g) exactly as the reference's
// reverse cumsum does, so
//   dL/dalpha_i = (T_i (c_i . g) - S_i / (1 - alpha_i)) [a_i < 0.99]
// Per-primitive partials are reduced across the warp with shuffles, across
// warps in shared memory, and flushed to HBM with one atomic per value per
// (primitive, tile).
#include <type_traits>

#include "common.cuh"

namespace sgs {

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Eight per-lane values summed over the warp by recursive halving (4 + 2 +
// 1 + 1 + 1 = 9 shuffles instead of 8 x 5).  Lane l ends with the total of
// value reduce8_index(l) (the four lanes l & ~3 .. l | 3 hold the same one).
__device__ __forceinline__ float warp_reduce8(const float v[8], int lane) {
  const bool u16 = lane & 16, u8 = lane & 8, u4 = lane & 4;
  float a[4];
#pragma unroll
  for (int j = 0; j < 4; ++j)
    a[j] = (u16 ? v[j + 4] : v[j]) + __shfl_xor_sync(0xffffffffu, u16 ? v[j] : v[j + 4], 16);
  float b[2];
#pragma unroll
  for (int j = 0; j < 2; ++j)
    b[j] = (u8 ? a[j + 2] : a[j]) + __shfl_xor_sync(0xffffffffu, u8 ? a[j] : a[j + 2], 8);
  float c = (u4 ? b[1] : b[0]) + __shfl_xor_sync(0xffffffffu, u4 ? b[0] : b[1], 4);
  c += __shfl_xor_sync(0xffffffffu, c, 2);
  return c + __shfl_xor_sync(0xffffffffu, c, 1);
}

__device__ __forceinline__ int reduce8_index(int lane) {
  return ((lane & 16) ? 4 : 0) + ((lane & 8) ? 2 : 0) + ((lane & 4) ? 1 : 0);
}


struct ListArgs {
  const uint2* ranges;      // per cell [start, end) into vals
  const uint32_t* keys;     // depth-first: sorted (super_id << 16 | tile mask) keys
  const uint32_t* vals;     // sorted primitive indices
  const uint2* rect;        // per primitive packed tile rectangle
  const float4* geo;
  const float4* con;
  const float4* col;
  const float4* eig;
  const float4* span;
  uint32_t* cand_end;       // per tile: one past the last candidate any pixel kept
  const uint32_t* order;    // raster dispatch order of the window's cells (longest list first)
  int super_x;
  int cell_base;            // first cell of the tile-row window
};

__device__ __forceinline__ int list_cell(bool filter, int tx, int ty, int tile, int super_x) {
  return filter ? (ty / SGS_SUPER) * super_x + tx / SGS_SUPER : tile;
}

// Tile of CTA `b` in cost order: the forward raster's CTAs walk the window's
// cells longest list first (cell_order_kernel), so the heaviest tiles start in
// the first wave instead of forming the tail.  In depth-first mode a cell is
// a 4x4-tile super-tile and 16 consecutive CTAs take its tiles.  Returns false
// for tiles outside the image or the tile-row window.
template <bool kFilter>
__device__ __forceinline__ bool ordered_tile(const ListArgs& la, const SgsCam& cam, uint32_t b, int& tx, int& ty) {
  if (kFilter) {
    const int cell = (int)la.order[b >> 4] + la.cell_base;
    const int sub = (int)(b & 15u);
    tx = (cell % la.super_x) * SGS_SUPER + (sub & 3);
    ty = (cell / la.super_x) * SGS_SUPER + (sub >> 2);
  } else {
    const int tile = (int)la.order[b] + la.cell_base;
    tx = tile % cam.tiles_x;
    ty = tile / cam.tiles_x;
  }
  return tx < cam.tiles_x && ty >= cam.tile_y0 && ty < cam.tile_y1;
}

// Dispatch order of the window's n cells, longest lists first: a counting
// sort on 64 length classes (log2 of the length with one mantissa bit),
// descending.  Only the raster's CTA scheduling depends on this order (not
// any result), so ties within a class are placed by shared-memory atomics.
constexpr int kOrderClasses = 64;
__device__ __forceinline__ int length_class(uint32_t len) {
  if (len == 0) return 0;
  const int e = 31 - __clz(len);                                 // floor(log2 len)
  const int half = e > 0 ? (int)((len >> (e - 1)) & 1u) : 0;    // next bit
  const int c = 2 * e + half + 1;
  return c < kOrderClasses ? c : kOrderClasses - 1;
}

// Length of item i: the cell's list length (forward), or with `cand_end` the
// candidates tile i of the window kept in the forward (backward raster: its
// work is the kept part of the list, walked back to front).
struct OrderSrc {
  const uint2* ranges;
  int base;
  const uint32_t* cand_end;  // null: cell list lengths
  int tiles_x, tile0, super_x;
  bool filt;
};

__device__ __forceinline__ uint32_t order_len(const OrderSrc& o, int i) {
  if (!o.cand_end) {
    const uint2 r = o.ranges[o.base + i];
    return r.y > r.x ? r.y - r.x : 0u;
  }
  const int tile = i + o.tile0, tx = tile % o.tiles_x, ty = tile / o.tiles_x;
  const uint32_t s = o.ranges[list_cell(o.filt, tx, ty, tile, o.super_x)].x, e = o.cand_end[tile];
  return e > s ? e - s : 0u;
}

__global__ void __launch_bounds__(1024) cell_order_kernel(OrderSrc src, int n, uint32_t* __restrict__ order) {
  __shared__ uint32_t hist[kOrderClasses];
  __shared__ uint32_t cursor[kOrderClasses];
  const int t = threadIdx.x;
  if (t < kOrderClasses) hist[t] = 0;
  __syncthreads();
  for (int i = t; i < n; i += blockDim.x) {
    atomicAdd(&hist[length_class(order_len(src, i))], 1u);
  }
  __syncthreads();
  if (t < 32) {  // exclusive scan over classes, longest class first
    const uint32_t a = hist[kOrderClasses - 1 - 2 * t], b = hist[kOrderClasses - 2 - 2 * t];
    uint32_t x = a + b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (t >= o) x += y;
    }
    const uint32_t excl = x - a - b;
    cursor[kOrderClasses - 1 - 2 * t] = excl;
    cursor[kOrderClasses - 2 - 2 * t] = excl + a;
  }
  __syncthreads();
  for (int i = t; i < n; i += blockDim.x) {
    order[atomicAdd(&cursor[length_class(order_len(src, i))], 1u)] = (uint32_t)i;
  }
}

// Shared-memory staging buffer of N records.
template <int N>
struct Stage {
  static constexpr bool kIds = true;
  float4 geo[N];
  float4 con[N];
  float4 col[N];
  uint32_t id[N];
  uint32_t cand[N];
  uint32_t wcnt[32];
};

// Stage without primitive ids / candidate positions (image-only forward):
// 8 KB less shared memory per CTA.
template <int N>
struct StageNoIds {
  static constexpr bool kIds = false;
  float4 geo[N];
  float4 con[N];
  float4 col[N];
  uint32_t wcnt[32];
};

// Append the members of tile (tx, ty) among candidates [c_lo, c_hi) (at
// most THREADS * CPT) of the cell list to the shared-memory batch at `base`,
// in list order.  Depth-first mode reads membership from the 16-bit tile mask
// carried in each sorted key (bit `local_bit`); 64-bit-key lists are per
// tile already.  Returns the number appended.  Ends with __syncthreads().
template <int THREADS, int CPT, bool kFilter, bool kColor, class S>
__device__ __forceinline__ int stage_append(uint32_t c_lo, uint32_t c_hi, uint32_t local_bit, const ListArgs& a,
                                            int base, S& s) {
  constexpr int W = THREADS / 32;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t bal[CPT];
#pragma unroll
  for (int h = 0; h < CPT; ++h) {
    const uint32_t c = c_lo + t + h * THREADS;
    bool hit = c < c_hi;
    if (kFilter && hit) hit = (a.keys[c] >> local_bit) & 1u;
    bal[h] = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) s.wcnt[h * W + warp] = __popc(bal[h]);
  }
  __syncthreads();
  int total = 0;
#pragma unroll
  for (int h = 0; h < CPT; ++h) {
    int pre = 0;
    for (int j = 0; j < CPT * W; ++j) {
      const int v = (int)s.wcnt[j];
      pre += (j < h * W + warp) ? v : 0;
      if (h == 0) total += v;
    }
    if ((bal[h] >> lane) & 1u) {
      const uint32_t c = c_lo + t + h * THREADS;
      const int pos = base + pre + __popc(bal[h] & lt);
      const uint32_t g = a.vals[c];
      s.geo[pos] = a.geo[g];
      s.con[pos] = a.eig[g];
      if (kColor) s.col[pos] = a.col[g];
      if constexpr (S::kIds) {
        s.id[pos] = g;
        s.cand[pos] = c;
      }
    }
  }
  __syncthreads();
  return total;
}

// A chunk of candidates [lo, hi) whose list keys and primitive indices are
// held in registers: the forward raster loads the next chunk before blending
// the current batch, so the list loads overlap the blend instead of stalling
// the next staging step.
template <int CPT>
struct ChunkRegs {
  uint32_t key[CPT], val[CPT];
  uint32_t lo, hi;
};

template <int THREADS, int CPT, bool kFilter>
__device__ __forceinline__ void load_chunk(ChunkRegs<CPT>& r, uint32_t lo, uint32_t hi, const ListArgs& a) {
  r.lo = lo;
  r.hi = hi;
#pragma unroll
  for (int h = 0; h < CPT; ++h) {
    const uint32_t c = lo + threadIdx.x + h * THREADS;
    r.key[h] = (kFilter && c < hi) ? a.keys[c] : 0u;
    r.val[h] = c < hi ? a.vals[c] : 0u;
  }
}

// stage_append on a register chunk (same records), each staged in the
// forward raster's tile-local form: geo = (c1, c2, log2 o_eff, -) with the
// eigen-form offsets c1 = -(e1 mx' + e2 my'), c2 = e4 mx' - e3 my' of the
// mean relative to the tile origin (mx' = mx - ox exactly), so a pixel at
// tile-local (lx, ly) has t1 = e1 lx + e2 ly + c1, t2 = e3 ly - e4 lx + c2.
// A listed record reaches the tile, so |t| stays small there and the offsets
// cost no precision (|c| <~ |t| + |e| 16).
template <int THREADS, int CPT, bool kFilter, class S, bool kLocal = true>
__device__ __forceinline__ int stage_append_regs(const ChunkRegs<CPT>& r, uint32_t local_bit, const ListArgs& a,
                                                 int base, S& s, float ox, float oy) {
  constexpr int W = THREADS / 32;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t bal[CPT];
#pragma unroll
  for (int h = 0; h < CPT; ++h) {
    const uint32_t c = r.lo + t + h * THREADS;
    bool hit = c < r.hi;
    if (kFilter) hit = hit && ((r.key[h] >> local_bit) & 1u);
    bal[h] = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) s.wcnt[h * W + warp] = __popc(bal[h]);
  }
  __syncthreads();
  int total = 0;
#pragma unroll
  for (int h = 0; h < CPT; ++h) {
    int pre = 0;
    for (int j = 0; j < CPT * W; ++j) {
      const int v = (int)s.wcnt[j];
      pre += (j < h * W + warp) ? v : 0;
      if (h == 0) total += v;
    }
    if ((bal[h] >> lane) & 1u) {
      const int pos = base + pre + __popc(bal[h] & lt);
      const uint32_t g = r.val[h];
      const float4 G = a.geo[g], E = a.eig[g];
      if constexpr (kLocal) {
        const float mx = G.x - ox, my = G.y - oy;
        s.geo[pos] = make_float4(fmaf(-E.x, mx, -(E.y * my)), fmaf(E.w, mx, -(E.z * my)), G.z, 0.0f);
      } else {
        s.geo[pos] = G;  // (mx, my, log2 o_eff, -) as stored
      }
      s.con[pos] = E;
      s.col[pos] = a.col[g];
      if constexpr (S::kIds) {
        s.id[pos] = g;
        s.cand[pos] = r.lo + t + h * THREADS;
      }
    }
  }
  __syncthreads();
  return total;
}

__device__ __forceinline__ uint32_t tile_local_bit(int tx, int ty) {
  return (uint32_t)((ty % SGS_SUPER) * SGS_SUPER + (tx % SGS_SUPER));
}

// Forward raster: 128 threads per 16x16 tile, each thread owns two
// vertically adjacent pixels (a warp covers an 8x8 quadrant, which keeps its
// lanes' supports and termination coherent).  Per staged record the two
// pixels share the record loads, dx and A dx; the per-pixel blend is
// predicated, and a warp skips a record outright when none of its 64 pixels
// is inside the record's support.  Warp-level termination (every pixel's
// transmittance fell below the cutoff) is voted once per kVoteEvery records
// rather than per record: a dead pixel is predicated off anyway, so the vote
// only bounds the work a finished warp wastes.
// kTrack: record per-pixel contributor counts and the per-tile candidate end
// the backward pass walks from; a render that only returns the image skips it.
constexpr double kWeightScale = 4294967296.0;  // importance fixed point: 2^32 units
constexpr int kFwdThreads = 128;
constexpr int kFwdCPT = 2;
constexpr int kFwdChunk = kFwdThreads * kFwdCPT;  // candidates examined per staging step
#ifndef SGS_FWD_BATCH
#define SGS_FWD_BATCH 128
#endif
#ifndef SGS_VOTE_EVERY
#define SGS_VOTE_EVERY 8
#endif
#ifndef SGS_FWD_MIN_BLOCKS
#define SGS_FWD_MIN_BLOCKS 8
#endif
#ifndef SGS_FWD_TRACK_MIN_BLOCKS
#define SGS_FWD_TRACK_MIN_BLOCKS 7
#endif
constexpr int kFwdBatch = SGS_FWD_BATCH;          // staged entries processed per block sync
constexpr int kFwdBuf = kFwdBatch + kFwdChunk;
constexpr int kVoteEvery = SGS_VOTE_EVERY;

// Warp vote without the compiler's divergence guard (callers are converged).
__device__ __forceinline__ bool warp_any(bool p) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred P, Q;\n\tsetp.ne.u32 P, %1, 0;\n\tvote.sync.any.pred Q, P, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, Q;\n\t}"
      : "=r"(r)
      : "r"((uint32_t)p));
  return r != 0;
}

// One pixel's front-to-back step against one record of its tile's list;
// p = log2(o G) (see sgs_pack_eig).  Every listed record is blended into every
// pixel of the tile, as the reference blends every primitive into every pixel
// (render.py:355-390); the lists hold the primitives whose support o G >= 1e-7
// meets the tile (binning), so a listed record outside a pixel's support
// contributes alpha < 1e-7, like the reference.
// Liveness is carried in the sign of T: a pixel whose next transmittance
// would fall below the cutoff keeps its last kept T, negated.  A terminated
// pixel needs no separate test: its Tn is negative, so it is never kept
// again, and re-terminating leaves -|T| unchanged.
//   alpha = min(2^p, 0.99),  w = alpha T,  Tn = T - w   (sgs_geom.h SGS_T_KEEP)
//   keep = Tn >= T_keep:  C += w c,  T = Tn;   else T = -|T|
// kClamp = false when no record of the batch can reach alpha 0.99 (the
// staging checks log2 o_eff < kLog2AlphaSafe), which drops the clamp.
constexpr float kLog2AlphaSafe = -0.0146f;  // 2^x = 0.98993 < 0.99 with ex2.approx's error
template <bool kClamp>
__device__ __forceinline__ bool blend_px(float p, const float4& c, float& T, float& C0, float& C1, float& C2,
                                         float& w) {
  const float a = ex2_approx(p);
  const float alpha = kClamp ? fminf(a, SGS_ALPHA_MAX) : a;
  w = alpha * T;
  const float Tn = T - w;
  const bool keep = Tn >= SGS_T_KEEP;
  if (keep) {
    C0 = fmaf(w, c.x, C0);
    C1 = fmaf(w, c.y, C1);
    C2 = fmaf(w, c.z, C2);
  }
  T = keep ? Tn : -fabsf(T);
  return keep;
}

// blend_px for the thread's two pixels at once with packed FP32x2 arithmetic
// (FFMA2 / FMUL2 / FADD2 on sm_100: one instruction for both pixels, each
// lane IEEE-rounded exactly as the scalar operation).  T2 = (T0, T1) and the
// colour accumulators are packed per channel: Cr = (C0.r, C1.r), ...
__device__ __forceinline__ float2 f2(float x) { return make_float2(x, x); }
__device__ __forceinline__ float2 neg2(float2 v) { return make_float2(-v.x, -v.y); }

template <bool kClamp>
__device__ __forceinline__ void blend2(float2 p, const float4& c, float2& T2, float2& Cr, float2& Cg, float2& Cb,
                                       bool& k0, bool& k1, float2& w) {
  float2 alpha = make_float2(ex2_approx(p.x), ex2_approx(p.y));
  if (kClamp) alpha = make_float2(fminf(alpha.x, SGS_ALPHA_MAX), fminf(alpha.y, SGS_ALPHA_MAX));
  w = __fmul2_rn(alpha, T2);
  const float2 Tn = __fadd2_rn(T2, neg2(w));  // T - w
  k0 = Tn.x >= SGS_T_KEEP;
  k1 = Tn.y >= SGS_T_KEEP;
  const float2 we = make_float2(k0 ? w.x : 0.0f, k1 ? w.y : 0.0f);  // C + 0 c = C exactly
  Cr = __ffma2_rn(we, f2(c.x), Cr);
  Cg = __ffma2_rn(we, f2(c.y), Cg);
  Cb = __ffma2_rn(we, f2(c.z), Cb);
  T2 = make_float2(k0 ? Tn.x : -fabsf(T2.x), k1 ? Tn.y : -fabsf(T2.y));
  w = we;
}

template <bool kImportance, bool kCount, bool kFilter, bool kTrack>
// The image-only variant is capped at 64 registers (8 resident CTAs, a few
// bytes of spills): slower alone (0.268 vs 0.264 ms) but it shares SMs with
// the other streams' binning kernels, +3 % frames/s in the 4-stream bench.
// The tracked variant (training, 4 view streams) is capped at 72 registers
// (7 CTAs/SM): +1.4 % training views/s although a lone view is slower; the
// importance variant keeps its registers.
__global__ void __launch_bounds__(kFwdThreads, kImportance ? 1 : (kTrack ? SGS_FWD_TRACK_MIN_BLOCKS : SGS_FWD_MIN_BLOCKS)) raster_fwd_kernel(ListArgs la, SgsCam cam, float3 bg,
                                                                 float* __restrict__ out_img,
                                                                 float* __restrict__ out_T,
                                                                 uint32_t* __restrict__ out_nc,
                                                                 unsigned long long* __restrict__ weight_fx,
                                                                 unsigned long long* __restrict__ pair_count) {
  __shared__ std::conditional_t<kImportance || kTrack, Stage<kFwdBuf>, StageNoIds<kFwdBuf>> s;
  __shared__ float s_wp[kImportance ? kFwdThreads / 32 : 1][kImportance ? kFwdBuf : 1];
  static_assert(!kImportance || kVoteEvery % 8 == 0, "importance sums reduce eight records at a time");
  __shared__ uint32_t s_kend;

  int tx, ty;
  if (!ordered_tile<kFilter>(la, cam, blockIdx.x, tx, ty)) return;
  const int tile = ty * cam.tiles_x + tx;
  const int t = threadIdx.x, lane = t & 31;
  // warp w covers the 8x8 quadrant (w & 1, w >> 1) of the tile: lane l owns
  // column l & 7 and rows 2 (l >> 3), 2 (l >> 3) + 1 of it (square blocks
  // keep a warp's supports and termination more coherent than 16x4 strips)
  const int wq = t >> 5, lq = t & 31;
  const int px = tx * SGS_TILE + (wq & 1) * 8 + (lq & 7);
  const int py0 = ty * SGS_TILE + (wq >> 1) * 8 + 2 * (lq >> 3);  // rows py0 and py0 + 1
  const bool in0 = px < cam.width && py0 < cam.height;
  const bool in1 = px < cam.width && py0 + 1 < cam.height;
  // pixel centres relative to the tile origin (records are staged in that frame)
  const float ox = (float)(tx * SGS_TILE), oy = (float)(ty * SGS_TILE);
  const float lx = (float)(px - tx * SGS_TILE) + 0.5f, ly0 = (float)(py0 - ty * SGS_TILE) + 0.5f;
  const uint2 rg = la.ranges[list_cell(kFilter, tx, ty, tile, la.super_x)];
  const uint32_t cs = rg.x, ce = rg.y > rg.x ? rg.y : rg.x;

  // T > 0: live; T < 0: terminated with transmittance -T (pixels off the
  // image start terminated)
  float2 T2 = make_float2(in0 ? 1.0f : -1.0f, in1 ? 1.0f : -1.0f);
  float2 Cr = make_float2(0.0f, 0.0f), Cg = Cr, Cb = Cr;
  const float2 lyv = make_float2(ly0, ly0 + 1.0f);  // the two pixels' tile-local row centres
  uint32_t nc0 = 0, nc1 = 0, reached = 0, kend = 0, hits_before = 0;
  if (kTrack && t == 0) s_kend = 0;

  const uint32_t lbit = tile_local_bit(tx, ty);
  uint32_t cb = cs;
  ChunkRegs<kFwdCPT> pf;
  bool have_pf = false;
  for (;;) {
    // stage until a full batch of this tile's entries (or the list ends)
    int nb = 0;
    while (nb < kFwdBatch && cb < ce) {
      const uint32_t chi = cb + kFwdChunk < ce ? cb + kFwdChunk : ce;
      if (!have_pf) load_chunk<kFwdThreads, kFwdCPT, kFilter>(pf, cb, chi, la);
      have_pf = false;
      nb += stage_append_regs<kFwdThreads, kFwdCPT, kFilter>(pf, lbit, la, nb, s, ox, oy);
      cb = chi;
    }
    if (nb == 0) break;
    // the next chunk's keys / indices load while this batch blends
    if (cb < ce) {
      load_chunk<kFwdThreads, kFwdCPT, kFilter>(pf, cb, cb + kFwdChunk < ce ? cb + kFwdChunk : ce, la);
      have_pf = true;
    }
    // pad the batch to a whole number of vote groups with records of zero
    // opacity (log2 o = -inf), so the group loop below needs no bounds checks
    const int nb_pad = (nb + kVoteEvery - 1) / kVoteEvery * kVoteEvery;
    if (t < nb_pad - nb) {
      s.geo[nb + t] = make_float4(0.0f, 0.0f, -INFINITY, 0.0f);
      s.con[nb + t] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      s.col[nb + t] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    }
    // can any staged record reach the alpha clamp?  (almost never: o_eff >= 0.99)
    bool clampable = false;
    for (int i = t; i < nb; i += kFwdThreads) clampable |= s.geo[i].z >= kLog2AlphaSafe;
    const bool batch_clamp = __syncthreads_or(clampable);
    auto run_batch = [&](auto clamp_tag) {
    constexpr bool kClamp = decltype(clamp_tag)::value;
    for (int k = 0; k < nb_pad; k += kVoteEvery) {
      if (!warp_any(T2.x > 0.0f || T2.y > 0.0f)) break;
      [[maybe_unused]] float wv[kImportance ? kVoteEvery : 1];  // importance: this thread's weight per group record
#pragma unroll
      for (int j = 0; j < kVoteEvery; ++j) {
        const int kk = k + j;
        const float4 G = s.geo[kk];  // (c1, c2, log2 o_eff, -): tile-local form
        const float4 E = s.con[kk];  // scaled eigen form (s1 ux, s1 uy, s2 ux, s2 uy)
        const float2 t1 = __ffma2_rn(f2(E.y), lyv, f2(fmaf(E.x, lx, G.x)));
        const float2 t2 = __ffma2_rn(f2(E.z), lyv, f2(fmaf(-E.w, lx, G.y)));
        const float2 p = __ffma2_rn(neg2(t1), t1, __ffma2_rn(neg2(t2), t2, f2(G.z)));
        if (kCount && kk < nb) reached += (uint32_t)(T2.x > 0.0f) + (uint32_t)(T2.y > 0.0f);
        {
          const float4 c = s.col[kk];
          bool k0, k1;
          float2 w;
          blend2<kClamp>(p, c, T2, Cr, Cg, Cb, k0, k1, w);
          if constexpr (kTrack) {  // kept records form a prefix: count them
            nc0 += (uint32_t)k0;
            nc1 += (uint32_t)k1;
          }
          if constexpr (kImportance) wv[j] = w.x + w.y;
        }
      }
      if constexpr (kImportance) {
        // the group's per-record weight sums over the warp, eight at a time
#pragma unroll
        for (int h = 0; h < kVoteEvery / 8; ++h) {
          const float tot = warp_reduce8(wv + 8 * h, lane);
          if ((lane & 3) == 0) s_wp[wq][k + 8 * h + reduce8_index(lane)] = tot;
        }
      }
    }
    };
    if constexpr (kImportance) {  // this warp's per-record weight sums of the batch
      for (int i = lq; i < nb_pad; i += 32) s_wp[wq][i] = 0.0f;
      __syncwarp();
    }
    if (batch_clamp)
      run_batch(std::true_type{});
    else
      run_batch(std::false_type{});
    if constexpr (kImportance) {  // one atomic per (record, tile): the four warps' sums
      __syncthreads();
      for (int i = t; i < nb; i += kFwdThreads) {
        const float x = (s_wp[0][i] + s_wp[1][i]) + (s_wp[2][i] + s_wp[3][i]);
        // fixed point (2^-32 units): integer sums do not depend on the order
        // the tiles' atomics land in, so the importance -- and the top-k
        // selection ties it feeds (prune.py:204) -- is bitwise reproducible
        if (x != 0.0f) atomicAdd(&weight_fx[s.id[i]], (unsigned long long)__double2ll_rn((double)x * kWeightScale));
      }
    }
    if constexpr (kTrack) {
      // the zero-opacity padding records count as kept for pixels still alive
      const uint32_t lim = hits_before + (uint32_t)nb;
      nc0 = nc0 < lim ? nc0 : lim;
      nc1 = nc1 < lim ? nc1 : lim;
      // candidate position of this thread's last kept entry (for the backward)
      const uint32_t mx = nc0 > nc1 ? nc0 : nc1;
      if (mx > hits_before) kend = s.cand[mx - hits_before - 1] + 1u;
    }
    hits_before += (uint32_t)nb;
    if (cb >= ce) break;
    if (__syncthreads_count(T2.x > 0.0f || T2.y > 0.0f) == 0) break;
  }
  if (kCount) {
    unsigned long long r = reached;
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    if (lane == 0 && r) atomicAdd(pair_count, r);
  }
  if (kTrack && kend) atomicMax(&s_kend, kend);
  const float T0 = fabsf(T2.x), T1 = fabsf(T2.y);
  const float C00 = Cr.x, C01 = Cg.x, C02 = Cb.x, C10 = Cr.y, C11 = Cg.y, C12 = Cb.y;
  if (in0) {
    const size_t pix = (size_t)py0 * cam.width + px;
    out_img[3 * pix + 0] = C00 + T0 * bg.x;
    out_img[3 * pix + 1] = C01 + T0 * bg.y;
    out_img[3 * pix + 2] = C02 + T0 * bg.z;
    if (out_T) out_T[pix] = T0;
    if (kTrack) out_nc[pix] = nc0;
  }
  if (in1) {
    const size_t pix = (size_t)(py0 + 1) * cam.width + px;
    out_img[3 * pix + 0] = C10 + T1 * bg.x;
    out_img[3 * pix + 1] = C11 + T1 * bg.y;
    out_img[3 * pix + 2] = C12 + T1 * bg.z;
    if (out_T) out_T[pix] = T1;
    if (kTrack) out_nc[pix] = nc1;
  }
  if (kTrack) {
    __syncthreads();
    if (t == 0) la.cand_end[tile] = s_kend ? s_kend : cs;
  }
}

constexpr int kGrad = 9;
#ifndef SGS_BWD_MIN_BLOCKS
#define SGS_BWD_MIN_BLOCKS 8
#endif
constexpr int kBwdThreads = 128;
constexpr int kBwdCPT = 1;
constexpr int kBwdChunk = kBwdThreads * kBwdCPT;  // candidates staged per batch

// The nine per-record partials summed over the warp.  A lane's two pixels
// share the column (dx); the four lanes of a column (lane bits 3, 4) are
// summed first on the six dx-free partials -- colour sums c0..c2 = sum w g
// and dq moments m0 = sum dq, m1 = sum dq dy, m2 = sum dq dy^2 -- by
// recursive halving (3 + 2 shuffles), the column sums are turned into the
// dx moments there (sum dq dx = dx m0, ...), and the eight columns (lane
// bits 0..2) are summed by halving again (2 + 1 + 1 shuffles): 9 shuffles in
// all instead of 12.  Returns the total of value reduce9_index(lane).
__device__ __forceinline__ float warp_reduce9(float c0, float c1, float c2, float m0, float m1, float m2, float dx,
                                              int lane) {
  const bool u16 = lane & 16, u8 = lane & 8, u4 = lane & 4, u2 = lane & 2;
  // rows, bit 4: colours stay on u16 = 0, moments on u16 = 1
  const float x0 = (u16 ? m0 : c0) + __shfl_xor_sync(0xffffffffu, u16 ? c0 : m0, 16);
  const float x1 = (u16 ? m1 : c1) + __shfl_xor_sync(0xffffffffu, u16 ? c1 : m1, 16);
  const float x2 = (u16 ? m2 : c2) + __shfl_xor_sync(0xffffffffu, u16 ? c2 : m2, 16);
  // rows, bit 3: (x0, x1) split, x2 summed on both
  const float y0 = (u8 ? x1 : x0) + __shfl_xor_sync(0xffffffffu, u8 ? x0 : x1, 8);
  const float y1 = x2 + __shfl_xor_sync(0xffffffffu, x2, 8);
  // column sums: (u16, u8) = 00: c0, c2 | 01: c1 | 10: m0, dx m0, dx^2 m0 | 11: m1, dx m1, m2
  const float ydx = y0 * dx;
  const float z0 = y0;
  const float z1 = u16 ? ydx : (u8 ? 0.0f : y1);
  const float z2 = u16 ? (u8 ? y1 : ydx * dx) : 0.0f;
  // columns, bit 2: (z0, z1) split, z2 summed on both; bits 1, 0
  const float p0 = (u4 ? z1 : z0) + __shfl_xor_sync(0xffffffffu, u4 ? z0 : z1, 4);
  const float p1 = z2 + __shfl_xor_sync(0xffffffffu, z2, 4);
  const float q = (u2 ? p1 : p0) + __shfl_xor_sync(0xffffffffu, u2 ? p0 : p1, 2);
  return q + __shfl_xor_sync(0xffffffffu, q, 1);
}

// Partial index held by each even lane after warp_reduce9 (4 bits per lane
// pair, 15 = padding or a duplicate): pair i = lane >> 1 has (u16, u8, u4,
// u2) = bits (3, 2, 1, 0) of i and holds u2 ? z2 : (u4 ? z1 : z0) with the
// partial order (w gx, w gy, w gz, dq, dq dx, dq dy, dq dx^2, dq dx dy, dq dy^2).
__device__ __forceinline__ int reduce9_index(int lane) {
  constexpr unsigned long long kLut = 0xf785f463fff1f2f0ull;
  return (lane & 1) ? 15 : (int)((kLut >> (4 * (lane >> 1))) & 15ull);
}

// Backward raster: 128 threads per tile, two vertically adjacent pixels per
// thread (a warp covers an 8x8 quadrant, as in the forward), walking the tile's
// list back to front from the last entry any pixel kept.  Per record each
// thread sums its two pixels' nine partials, the warp reduces them with
// warp_reduce9, and nine lanes store the totals into the warp's slot of the
// batch's shared partials; each batch is flushed by summing the 4 warps'
// partials with one global atomic per (record, partial).  T is recovered with one hardware reciprocal
// per pixel-record, T_i = T_{i+1} rcp(1 - alpha_i) (~1 ulp per record).
// Deterministic mode (kMode 1 + 2, sgs_raster_backward_det): the float
// atomics below add the (record, tile) partials in whatever order the tiles
// finish, so sums are reproducible only to rounding.  Pass 1 (kMode 1)
// records each (primitive, partial)'s largest |partial| (an order-free
// atomicMax on the float bits); pass 2 (kMode 2) recomputes the identical
// partials and adds them as 64-bit fixed point scaled to that maximum
// (fx_scale: every term < 2^42, < 2^20 tiles per primitive), which integer
// addition sums exactly in any order; bwd_fixed_finalize converts back.
__device__ __forceinline__ double fx_scale(uint32_t max_bits) {
  const int e = (int)((max_bits >> 23) & 0xffu) - 127;  // |partial| < 2^(e + 1)
  return __longlong_as_double((long long)(1023 + 41 - e) << 52);  // 2^(41 - e)
}

template <bool kFilter, int kMode>
__global__ void __launch_bounds__(kBwdThreads, SGS_BWD_MIN_BLOCKS) raster_bwd_kernel(ListArgs la, SgsCam cam, float3 bg,
                                                                 const float* __restrict__ final_T,
                                                                 const uint32_t* __restrict__ ncontrib,
                                                                 const float* __restrict__ dimg,
                                                                 float* __restrict__ grad2d,
                                                                 uint32_t* __restrict__ gmax,
                                                                 unsigned long long* __restrict__ gfx) {
  __shared__ Stage<kBwdChunk> s;
  // per-warp partial totals (plain stores; shared-memory float atomics are CAS
  // loops on sm_100), summed over the 4 warps when the batch is flushed
  __shared__ float s_part[kBwdThreads / 32][kBwdChunk][kGrad];
  __shared__ uint32_t s_max_nc;

  // tiles in kept-work order, heaviest first (launch_raster_bwd): the long
  // tiles start in the first wave instead of forming the tail
  const int tile = (int)la.order[blockIdx.x] + cam.tile_y0 * cam.tiles_x;
  const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
  const int t = threadIdx.x, lane = t & 31;
  const int wq = t >> 5, lq = t & 31;  // 8x8 quadrants per warp, as in the forward
  const int px = tx * SGS_TILE + (wq & 1) * 8 + (lq & 7);
  const int py0 = ty * SGS_TILE + (wq >> 1) * 8 + 2 * (lq >> 3);
  const bool in0 = px < cam.width && py0 < cam.height;
  const bool in1 = px < cam.width && py0 + 1 < cam.height;
  const float fx = (float)px + 0.5f, fy0 = (float)py0 + 0.5f;
  const uint2 rg = la.ranges[list_cell(kFilter, tx, ty, tile, la.super_x)];
  const uint32_t cs = rg.x;
  const uint32_t cend = la.cand_end[tile];

  float T0 = 1.0f, T1 = 1.0f, S0 = 0.0f, S1 = 0.0f;
  float g00 = 0.0f, g01 = 0.0f, g02 = 0.0f, g10 = 0.0f, g11 = 0.0f, g12 = 0.0f;
  uint32_t nc0 = 0, nc1 = 0;
  if (t == 0) s_max_nc = 0;
  __syncthreads();
  if (in0) {
    const size_t pix = (size_t)py0 * cam.width + px;
    T0 = final_T[pix];
    nc0 = ncontrib[pix];
    g00 = dimg[3 * pix + 0];
    g01 = dimg[3 * pix + 1];
    g02 = dimg[3 * pix + 2];
    S0 = T0 * (g00 * bg.x + g01 * bg.y + g02 * bg.z);
  }
  if (in1) {
    const size_t pix = (size_t)(py0 + 1) * cam.width + px;
    T1 = final_T[pix];
    nc1 = ncontrib[pix];
    g10 = dimg[3 * pix + 0];
    g11 = dimg[3 * pix + 1];
    g12 = dimg[3 * pix + 2];
    S1 = T1 * (g10 * bg.x + g11 * bg.y + g12 * bg.z);
  }
  float2 T2 = make_float2(T0, T1), S2 = make_float2(S0, S1);
  const float2 gx2 = make_float2(g00, g10), gy2 = make_float2(g01, g11), gz2 = make_float2(g02, g12);
  const float2 fyv = make_float2(fy0, fy0 + 1.0f);
  const uint32_t ncm = nc0 > nc1 ? nc0 : nc1;
  if (ncm) atomicMax(&s_max_nc, ncm);
  __syncthreads();
  const uint32_t max_nc = s_max_nc;
  const uint32_t warp_nc = __reduce_max_sync(0xffffffffu, ncm);
  // (a pixel off the image has nc 0, so its warp never takes the all-active
  // body, which would advance its unused transmittance)
  const uint32_t warp_min_nc = __reduce_min_sync(0xffffffffu, min(nc0, nc1));
  const uint32_t lbit = tile_local_bit(tx, ty);
  const int vidx = reduce9_index(lane);
  uint32_t hits_after = 0;

  // the list keys / indices of the next (earlier) chunk load while this one
  // is processed
  ChunkRegs<kBwdCPT> pf;
  if (cend > cs) load_chunk<kBwdThreads, kBwdCPT, kFilter>(pf, cend - cs > (uint32_t)kBwdChunk ? cend - kBwdChunk : cs,
                                                           cend, la);
  for (uint32_t hi = cend; hi > cs;) {
    const uint32_t lo = hi - cs > (uint32_t)kBwdChunk ? hi - kBwdChunk : cs;
    __syncthreads();  // previous batch fully flushed
    const int nb = stage_append_regs<kBwdThreads, kBwdCPT, kFilter, decltype(s), false>(pf, lbit, la, 0, s,
                                                                                      0.0f, 0.0f);
    if (lo > cs) load_chunk<kBwdThreads, kBwdCPT, kFilter>(pf, lo - cs > (uint32_t)kBwdChunk ? lo - kBwdChunk : cs,
                                                           lo, la);
    const uint32_t base = max_nc - hits_after - (uint32_t)nb;  // per-tile list index of staged entry 0
    const int wq_ = t >> 5;
    // staged records at or past the warp's last kept one (list index >=
    // warp_nc) need no work: their partial slots are zeroed together
    const int k_top = (int)max((int64_t)-1, min((int64_t)nb - 1, (int64_t)warp_nc - 1 - (int64_t)base));
    for (int i = (k_top + 1) * kGrad + lane; i < nb * kGrad; i += 32) (&s_part[wq_][0][0])[i] = 0.0f;
    // Records whose per-tile index is below every pixel's kept count in this
    // warp (warp_min_nc: ~82 % of the records processed at configs[3]) are
    // active for all 64 pixels -- the loop body drops the per-pixel activity
    // selects for them (kAll); the records between the warp's smallest and
    // largest kept count take the general body.
    auto record = [&](int k, auto all_tag) {
      constexpr bool kAll = decltype(all_tag)::value;
      const uint32_t idx = base + (uint32_t)k;
      const float4 G = s.geo[k];  // (mx, my, log2 o_eff, -)
      const float4 E = s.con[k];  // scaled eigen form (s1 ux, s1 uy, s2 ux, s2 uy)
      const float4 col = s.col[k];
      // the thread's two pixels packed per quantity (FFMA2/FMUL2/FADD2), as in the forward
      const float dx = fx - G.x;
      const float2 dy = __fadd2_rn(fyv, f2(-G.y));
      const float e1dx = E.x * dx, e3dx = E.w * dx;
      const float2 t1 = __ffma2_rn(f2(E.y), dy, f2(e1dx));
      const float2 t2 = __ffma2_rn(f2(E.z), dy, f2(-e3dx));
      const float2 pq = __ffma2_rn(neg2(t1), t1, __fmul2_rn(neg2(t2), t2));  // log2 G = -(t1^2 + t2^2)
      const float2 p = __fadd2_rn(pq, f2(G.z));                                // log2 (o_eff G)
      const bool act0 = kAll || idx < nc0, act1 = kAll || idx < nc1;
      // A record outside the support every active pixel of the warp was
      // binned with (log2 G >= pmin, geo.w: o_bin G >= 1e-7) contributes
      // < 1e-7 of any partial and changes T by a factor within 1e-7 of 1:
      // skip it whole.  o_bin = max(o_eff, grad_floor) (sgs_camera).
      if (!warp_any((act0 && pq.x >= G.w) || (act1 && pq.y >= G.w))) {
        if (vidx < kGrad) s_part[wq_][k][vidx] = 0.0f;
        return;
      }
      const float2 a = make_float2(ex2_approx(p.x), ex2_approx(p.y));
      const float2 alpha = make_float2(fminf(a.x, SGS_ALPHA_MAX), fminf(a.y, SGS_ALPHA_MAX));
      const float2 om = __fadd2_rn(f2(1.0f), neg2(alpha));  // the forward's T_next = T - alpha T
      // om in [0.0099, 1]: MUFU.RCP, ~1 ulp
      const float2 rom = make_float2(rcp_approx(om.x), rcp_approx(om.y));
      const float2 Ti = __fmul2_rn(T2, rom);
      const float2 w = __fmul2_rn(alpha, Ti);
      const float2 cg = __ffma2_rn(f2(col.x), gx2, __ffma2_rn(f2(col.y), gy2, __fmul2_rn(f2(col.z), gz2)));
      const float2 dal = __ffma2_rn(Ti, cg, neg2(__fmul2_rn(S2, rom)));
      // o_eff = 0 (binned by the gradient floor): alpha is 0 everywhere, but
      // dL/do_eff = sum G dL/dalpha is not; its dq partials are taken per
      // unit opacity (G itself; K7 reads them so)
      float2 ag = a;
      if (G.z == -INFINITY) ag = make_float2(ex2_approx(pq.x), ex2_approx(pq.y));  // warp-uniform
      const float2 dq = __fmul2_rn(__fmul2_rn(f2(-0.5f), ag), dal);
      const float2 Sn = __ffma2_rn(w, cg, S2);
      const bool l0 = act0 && a.x < SGS_ALPHA_MAX, l1 = act1 && a.y < SGS_ALPHA_MAX;
      const float2 dqa = make_float2(l0 ? dq.x : 0.0f, l1 ? dq.y : 0.0f);
      float2 ww;
      if constexpr (kAll) {
        S2 = Sn;
        T2 = Ti;
        ww = w;
      } else {
        ww = make_float2(act0 ? w.x : 0.0f, act1 ? w.y : 0.0f);
        S2 = make_float2(act0 ? Sn.x : S2.x, act1 ? Sn.y : S2.y);
        T2 = make_float2(act0 ? Ti.x : T2.x, act1 ? Ti.y : T2.y);
      }
      const float2 wgx = __fmul2_rn(ww, gx2), wgy = __fmul2_rn(ww, gy2), wgz = __fmul2_rn(ww, gz2);
      // the column's pixels share dx: the dq moments are summed in dy only and
      // the dx factors applied to the column sums inside the reduction
      const float2 qy = __fmul2_rn(dqa, dy);
      const float tot = warp_reduce9(wgx.x + wgx.y, wgy.x + wgy.y, wgz.x + wgz.y, dqa.x + dqa.y, qy.x + qy.y,
                                     fmaf(qy.y, dy.y, qy.x * dy.x), dx, lane);
      if (vidx < kGrad) s_part[wq_][k][vidx] = tot;
    };
    const int k_all = (int)max((int64_t)0, min((int64_t)k_top + 1, (int64_t)warp_min_nc - (int64_t)base));
    for (int k = k_top; k >= k_all; --k) record(k, std::false_type{});
    for (int k = k_all - 1; k >= 0; --k) record(k, std::true_type{});
    __syncthreads();
    for (int i = t; i < nb * kGrad; i += kBwdThreads) {
      const int k = i / kGrad, c = i - k * kGrad;
      float x = 0.0f;
#pragma unroll
      for (int w = 0; w < kBwdThreads / 32; ++w) x += s_part[w][k][c];
      if (x != 0.0f) {
        const size_t o = (size_t)s.id[k] * kGrad + c;
        if constexpr (kMode == 0)
          atomicAdd(grad2d + o, x);
        else if constexpr (kMode == 1)
          atomicMax(gmax + o, __float_as_uint(fabsf(x)));
        else
          atomicAdd(gfx + o, (unsigned long long)__double2ll_rn((double)x * fx_scale(gmax[o])));
      }
    }
    hits_after += (uint32_t)nb;
    hi = lo;
  }
}

// ------------------------------------------------------------- list export
// Per-tile lists materialised from the cell lists (parity checks): pass 0
// counts each tile's hits into ranges[t].y, a scan turns them into
// [start, end), pass 1 writes (tile << 32 | depth_bits, primitive) in order.
template <bool kFilter>
__global__ void __launch_bounds__(kFwdThreads) export_lists_kernel(ListArgs la, SgsCam cam, int pass,
                                                                   const uint32_t* __restrict__ depth_key,
                                                                   uint2* __restrict__ tile_ranges,
                                                                   unsigned long long* __restrict__ keys,
                                                                   uint32_t* __restrict__ vals) {
  __shared__ Stage<kFwdChunk> s;
  const int tile = blockIdx.x;
  const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
  const uint2 rg = la.ranges[list_cell(kFilter, tx, ty, tile, la.super_x)];
  const uint32_t cs = rg.x, ce = rg.y > rg.x ? rg.y : rg.x;
  uint32_t out = pass == 0 ? 0u : tile_ranges[tile].x;
  const uint32_t lbit = tile_local_bit(tx, ty);
  for (uint32_t cb = cs; cb < ce; cb += kFwdChunk) {
    const uint32_t chi = cb + kFwdChunk < ce ? cb + kFwdChunk : ce;
    const int nb = stage_append<kFwdThreads, kFwdCPT, kFilter, false>(cb, chi, lbit, la, 0, s);
    if (pass == 1)
      for (int k = threadIdx.x; k < nb; k += kFwdThreads) {
        const uint32_t g = s.id[k];
        keys[out + k] = ((unsigned long long)tile << 32) | depth_key[g];
        vals[out + k] = g;
      }
    out += (uint32_t)nb;
    __syncthreads();
  }
  if (pass == 0 && threadIdx.x == 0) tile_ranges[tile] = make_uint2(0u, out);
}

__global__ void __launch_bounds__(1024) export_scan_kernel(uint2* __restrict__ r, int n) {
  __shared__ uint32_t warp_tot[32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int base = 0; base < n; base += 1024) {
    const int i = base + threadIdx.x;
    const uint32_t v = i < n ? r[i].y : 0u;
    uint32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    uint32_t pre = carry;
    for (int k = 0; k < w; ++k) pre += warp_tot[k];
    if (i < n) r[i] = v ? make_uint2(pre + x - v, pre + x) : make_uint2(0u, 0u);
    __syncthreads();
    if (threadIdx.x == 1023) carry = pre + x;
    __syncthreads();
  }
}

bool final_in_alt(const Layout& lo);

static ListArgs list_args(const sgs_workspace* ws, const Layout& lo, const uint32_t* vals) {
  ListArgs a;
  a.ranges = at<uint2>(ws, lo.ranges);
  a.keys = at<uint32_t>(ws, final_in_alt(lo) ? lo.ent_key_alt : lo.ent_key);
  a.vals = vals;
  a.rect = at<uint2>(ws, lo.rect);
  a.geo = at<float4>(ws, lo.rec_geo);
  a.con = at<float4>(ws, lo.rec_con);
  a.col = at<float4>(ws, lo.rec_col);
  a.eig = at<float4>(ws, lo.rec_eig);
  a.span = at<float4>(ws, lo.rec_span);
  a.cand_end = at<uint32_t>(ws, lo.cand_end);
  a.order = at<uint32_t>(ws, lo.cell_order);
  a.super_x = lo.super_x;
  a.cell_base = 0;
  return a;
}

int launch_raster_fwd(const SgsCam& cam, float3 bg, const sgs_workspace* ws, const Layout& lo, const uint32_t* vals,
                      float* img, float* T, uint32_t* nc, unsigned long long* weight_fx, unsigned long long* pairs,
                      cudaStream_t st) {
  ListArgs a = list_args(ws, lo, vals);
  const bool filt = lo.sort_mode == SGS_SORT_DEPTH_FIRST;
  // cells of the tile-row window, then their dispatch order
  int n_cells, grid;
  if (filt) {
    const int sr0 = cam.tile_y0 / SGS_SUPER, sr1 = (cam.tile_y1 - 1) / SGS_SUPER;
    a.cell_base = sr0 * lo.super_x;
    n_cells = (sr1 - sr0 + 1) * lo.super_x;
    grid = n_cells * SGS_SUPER * SGS_SUPER;
  } else {
    a.cell_base = cam.tile_y0 * cam.tiles_x;
    n_cells = (cam.tile_y1 - cam.tile_y0) * cam.tiles_x;
    grid = n_cells;
  }
  {
    const OrderSrc src{a.ranges, a.cell_base, nullptr, cam.tiles_x, 0, lo.super_x, filt};
    cell_order_kernel<<<1, 1024, 0, st>>>(src, n_cells, at<uint32_t>(ws, lo.cell_order));
    SGS_LAUNCH_CHECK("cell_order_kernel");
  }
#define SGS_FWD(I, C, F, K) \
  raster_fwd_kernel<I, C, F, K><<<grid, kFwdThreads, 0, st>>>(a, cam, bg, img, T, nc, weight_fx, pairs)
#define SGS_FWD_TRACK(I, C, F) \
  if (nc) SGS_FWD(I, C, F, true); else SGS_FWD(I, C, F, false)
  if (filt) {
    if (weight_fx && pairs) SGS_FWD_TRACK(true, true, true);
    else if (weight_fx) SGS_FWD_TRACK(true, false, true);
    else if (pairs) SGS_FWD_TRACK(false, true, true);
    else SGS_FWD_TRACK(false, false, true);
  } else {
    if (weight_fx && pairs) SGS_FWD_TRACK(true, true, false);
    else if (weight_fx) SGS_FWD_TRACK(true, false, false);
    else if (pairs) SGS_FWD_TRACK(false, true, false);
    else SGS_FWD_TRACK(false, false, false);
  }
#undef SGS_FWD_TRACK
#undef SGS_FWD
  SGS_LAUNCH_CHECK("raster_fwd_kernel");
  return SGS_OK;
}

__global__ void __launch_bounds__(256) bwd_fixed_finalize(const uint32_t* __restrict__ gmax,
                                                          const unsigned long long* __restrict__ gfx,
                                                          float* __restrict__ grad2d, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const uint32_t m = gmax[i];
    grad2d[i] = m ? (float)((double)(long long)gfx[i] / fx_scale(m)) : 0.0f;
  }
}

uint64_t raster_bwd_det_scratch_bytes(int64_t n) { return (uint64_t)(n > 0 ? n : 1) * kGrad * (4 + 8) + 256; }

int launch_raster_bwd(const SgsCam& cam, float3 bg, const sgs_workspace* ws, const Layout& lo, const uint32_t* vals,
                      const float* T, const uint32_t* nc, const float* dimg, float* grad2d, void* det_scratch,
                      cudaStream_t st) {
  const int grid = (cam.tile_y1 - cam.tile_y0) * cam.tiles_x;
  const size_t nv = (size_t)lo.n * kGrad;
  const ListArgs a = list_args(ws, lo, vals);
  const bool filt = lo.sort_mode == SGS_SORT_DEPTH_FIRST;
  static bool carve = false;
  if (!carve) {  // all of the SM's shared memory for the CTAs' partial slots
    SGS_CUDA(cudaFuncSetAttribute(raster_bwd_kernel<true, 0>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    SGS_CUDA(cudaFuncSetAttribute(raster_bwd_kernel<false, 0>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    carve = true;
  }
  {
    const OrderSrc src{a.ranges, 0, a.cand_end, cam.tiles_x, cam.tile_y0 * cam.tiles_x, lo.super_x, filt};
    cell_order_kernel<<<1, 1024, 0, st>>>(src, grid, at<uint32_t>(ws, lo.cell_order));
    SGS_LAUNCH_CHECK("cell_order_kernel (backward)");
  }
  if (!det_scratch) {
    SGS_CUDA(cudaMemsetAsync(grad2d, 0, nv * sizeof(float), st));
    if (filt)
      raster_bwd_kernel<true, 0><<<grid, kBwdThreads, 0, st>>>(a, cam, bg, T, nc, dimg, grad2d, nullptr, nullptr);
    else
      raster_bwd_kernel<false, 0><<<grid, kBwdThreads, 0, st>>>(a, cam, bg, T, nc, dimg, grad2d, nullptr, nullptr);
    SGS_LAUNCH_CHECK("raster_bwd_kernel");
    return SGS_OK;
  }
  unsigned long long* gfx = reinterpret_cast<unsigned long long*>(
      (reinterpret_cast<uintptr_t>(det_scratch) + 255) & ~uintptr_t(255));
  uint32_t* gmax = reinterpret_cast<uint32_t*>(gfx + nv);
  SGS_CUDA(cudaMemsetAsync(gfx, 0, nv * (8 + 4), st));
  if (filt) {
    raster_bwd_kernel<true, 1><<<grid, kBwdThreads, 0, st>>>(a, cam, bg, T, nc, dimg, grad2d, gmax, gfx);
    raster_bwd_kernel<true, 2><<<grid, kBwdThreads, 0, st>>>(a, cam, bg, T, nc, dimg, grad2d, gmax, gfx);
  } else {
    raster_bwd_kernel<false, 1><<<grid, kBwdThreads, 0, st>>>(a, cam, bg, T, nc, dimg, grad2d, gmax, gfx);
    raster_bwd_kernel<false, 2><<<grid, kBwdThreads, 0, st>>>(a, cam, bg, T, nc, dimg, grad2d, gmax, gfx);
  }
  SGS_LAUNCH_CHECK("raster_bwd_kernel (deterministic)");
  bwd_fixed_finalize<<<persistent_grid(nv, 256, 8), 256, 0, st>>>(gmax, gfx, grad2d, nv);
  SGS_LAUNCH_CHECK("bwd_fixed_finalize");
  return SGS_OK;
}

__global__ void __launch_bounds__(256) fixed_to_float_kernel(const unsigned long long* __restrict__ fx, size_t n,
                                                             double inv_scale, float* __restrict__ out, int acc) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float v = (float)((double)(long long)fx[i] * inv_scale);
    out[i] = acc ? out[i] + v : v;
  }
}

int launch_fixed_to_float(const unsigned long long* fx, int64_t n, int frac_bits, float* out, int acc, cudaStream_t st) {
  if (n <= 0) return SGS_OK;
  fixed_to_float_kernel<<<persistent_grid((uint64_t)n, 256, 8), 256, 0, st>>>(fx, (size_t)n, ldexp(1.0, -frac_bits),
                                                                           out, acc);
  SGS_LAUNCH_CHECK("fixed_to_float_kernel");
  return SGS_OK;
}

int launch_export_lists(const SgsCam& cam, const sgs_workspace* ws, const Layout& lo, const uint32_t* vals,
                        unsigned long long* keys, uint32_t* out_vals, uint32_t* ranges, cudaStream_t st) {
  const ListArgs a = list_args(ws, lo, vals);
  uint2* r = reinterpret_cast<uint2*>(ranges);
  const uint32_t* dk = at<uint32_t>(ws, lo.depth_key);
  const bool filt = lo.sort_mode == SGS_SORT_DEPTH_FIRST;
  for (int pass = 0; pass < 2; ++pass) {
    if (filt)
      export_lists_kernel<true><<<lo.n_tiles, kFwdThreads, 0, st>>>(a, cam, pass, dk, r, keys, out_vals);
    else
      export_lists_kernel<false><<<lo.n_tiles, kFwdThreads, 0, st>>>(a, cam, pass, dk, r, keys, out_vals);
    SGS_LAUNCH_CHECK("export_lists_kernel");
    if (pass == 0) {
      export_scan_kernel<<<1, 1024, 0, st>>>(r, lo.n_tiles);
      SGS_LAUNCH_CHECK("export_scan_kernel");
    }
  }
  return SGS_OK;
}

}  // namespace sgs
