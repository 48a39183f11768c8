// binning.cu -- K2 duplicate-with-keys, K3 sort, K4 tile ranges.
//
// The reference orders primitives with one global stable argsort on depth
// (/root/reference/pkg/src/sgsplat/render.py:307) and blends every pixel
// against every primitive.  The tiled renderer needs, per 16x16 tile, the
// primitives whose support meets the tile in (depth, index) order.  The
// contract is the list of 64-bit keys (tile << 32 | depth_bits) with
// primitive-index values, stably sorted, plus per-tile [start, end) ranges.
//
// Both modes first radix-sort the N primitives on their 31-bit depth keys
// (4 passes over N, not E) and order runs of equal keys by the float64
// residual and index (depth_tie_fixup), then emit entries in that order; a
// stable radix sort on the cell id of a list already in (depth, index) order
// yields exactly the (tile, depth, index) order of the full 64-bit sort.
//   SGS_SORT_KEY64       the entries carry the literal 64-bit key
//                        (tile << 32 | depth_bits); the LSD sort runs over the
//                        tile digits only, the low 32 bits arriving ordered
//                        (2 onesweep passes at 1080p, 24 B/entry/pass);
//   SGS_SORT_DEPTH_FIRST the entries are (super-tile id << 16 | 16-bit tile
//                        mask), about a sixth as many, sorted on the
//                        super-tile id (one 9-bit pass at 1080p); the raster
//                        filters each super-tile list by its tile's mask bit.
#include <algorithm>
#include <utility>

#include "sort.cuh"

namespace sgs {

// ---------------------------------------------------------------- scan (u64)
// offsets[r] = sum_{r' < r} tiles_touched[perm ? perm[r'] : r'] ; totals -> counters.
// One kernel, decoupled look-back: partitions of kScanItems ranks are claimed
// in order from a ticket, each publishes its sum, then its inclusive prefix
// once warp 0 has summed the predecessors' published values 32 at a time.
constexpr int kScanThreads = 256, kScanPer = 8;
constexpr int kScanItems = kScanThreads * kScanPer;  // 2048 ranks per partition
constexpr unsigned long long kScanAgg = 1ull << 62, kScanInc = 2ull << 62, kScanVal = (1ull << 62) - 1;

__device__ __forceinline__ uint32_t scan_load(const uint32_t* tt, const uint32_t* perm, uint32_t r) {
  return tt[perm ? perm[r] : r];
}

__global__ void __launch_bounds__(kScanThreads) scan_onepass(const uint32_t* __restrict__ tt,
                                                            const uint32_t* __restrict__ perm, uint32_t n_max,
                                                            const uint32_t* __restrict__ n_ptr,
                                                            uint32_t cap, unsigned long long* status,
                                                            uint32_t* ticket,
                                                            unsigned long long* __restrict__ offsets,
                                                            Counters* ctr) {
  __shared__ unsigned long long warp_tot[kScanThreads / 32];
  __shared__ unsigned long long s_excl;
  __shared__ uint32_t s_part;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const uint32_t n = n_ptr ? min(*n_ptr, n_max) : n_max;  // ranks: the depth-sorted emitting primitives
  const uint32_t nparts = (n + kScanItems - 1) / kScanItems;
  if (nparts == 0) {  // nothing emits
    if (blockIdx.x == 0 && t == 0) {
      ctr->n_bin = 0;
      ctr->capacity = cap;
      ctr->overflow = 0;
      ctr->n_sort = 0;
    }
    return;
  }
  for (;;) {
    if (t == 0) s_part = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t part = s_part;
    if (part >= nparts) return;
    // each thread owns kScanPer consecutive ranks
    const uint32_t r0 = part * kScanItems + (uint32_t)t * kScanPer;
    uint32_t v[kScanPer];
    unsigned long long sum = 0;
#pragma unroll
    for (int k = 0; k < kScanPer; ++k) {
      v[k] = r0 + k < n ? scan_load(tt, perm, r0 + k) : 0u;
      sum += v[k];
    }
    unsigned long long x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    unsigned long long pre = 0, agg = 0;
#pragma unroll
    for (int k = 0; k < kScanThreads / 32; ++k) {
      pre += k < w ? warp_tot[k] : 0ull;
      agg += warp_tot[k];
    }
    if (w == 0) {
      unsigned long long excl = 0;
      if (part == 0) {
        if (lane == 0) atomicExch(&status[0], kScanInc | agg);
      } else {
        if (lane == 0) atomicExch(&status[part], kScanAgg | agg);
        int64_t p = (int64_t)part - 1;
        for (;;) {
          const int64_t q = p - lane;
          unsigned long long sv = kScanInc + 0ull;
          if (q >= 0) sv = *reinterpret_cast<volatile unsigned long long*>(&status[q]);
          const unsigned long long flag = sv & ~kScanVal;
          const uint32_t inc = __ballot_sync(0xffffffffu, flag == kScanInc);
          const uint32_t empty = __ballot_sync(0xffffffffu, flag == 0);
          // lanes up to and including the nearest inclusive prefix must all be published
          const uint32_t need = inc ? (inc & (0u - inc)) * 2u - 1u : 0xffffffffu;
          if (empty & need) continue;
          unsigned long long part_sum = (need >> lane) & 1u ? (sv & kScanVal) : 0ull;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) part_sum += __shfl_xor_sync(0xffffffffu, part_sum, o);
          excl += part_sum;
          if (inc) break;
          p -= 32;
        }
        if (lane == 0) atomicExch(&status[part], kScanInc | (excl + agg));
      }
      if (lane == 0) s_excl = excl;
    }
    __syncthreads();
    unsigned long long o = s_excl + pre + x - sum;
#pragma unroll
    for (int k = 0; k < kScanPer; ++k) {
      if (r0 + k < n) offsets[r0 + k] = o;
      o += v[k];
    }
    if (part + 1 == nparts && t == kScanThreads - 1) {
      const unsigned long long total = o;  // the last thread ends at the grand total
      ctr->n_bin = total;
      ctr->capacity = cap;
      ctr->overflow = total > cap ? 1ull : 0ull;
      ctr->n_sort = (uint32_t)(total < cap ? total : cap);
    }
    __syncthreads();
  }
}

__global__ void set_count(uint32_t* p, uint32_t v) { *p = v; }

static int launch_scan(const uint32_t* tt, const uint32_t* perm, uint32_t n, const uint32_t* n_ptr, uint32_t cap,
                       unsigned long long* status, unsigned long long* offsets, Counters* ctr, cudaStream_t st) {
  const uint32_t nparts = (n + kScanItems - 1) / kScanItems;  // upper bound when n_ptr is given
  if (nparts == 0) {
    SGS_CUDA(cudaMemsetAsync(&ctr->n_bin, 0, sizeof(ctr->n_bin), st));
    SGS_CUDA(cudaMemsetAsync(&ctr->n_sort, 0, sizeof(ctr->n_sort), st));
    return SGS_OK;
  }
  SGS_CUDA(cudaMemsetAsync(status, 0, (size_t)nparts * 8, st));
  SGS_CUDA(cudaMemsetAsync(&ctr->part_counter[kScanTicket], 0, 4, st));
  scan_onepass<<<persistent_grid(nparts, 1, 8), kScanThreads, 0, st>>>(tt, perm, n, n_ptr, cap, status,
                                                                        &ctr->part_counter[kScanTicket], offsets,
                                                                        ctr);
  SGS_LAUNCH_CHECK("scan_onepass");
  return SGS_OK;
}

// ------------------------------------------------------ float64 depth ties
// The radix sorts order by the float32 depth key (the float64 z rounded,
// sgs_project); equal keys come out in input order, which is the
// preprocess's compaction order (depth-first mode) or primitive order
// (64-bit keys).  The reference orders by its float64 z (render.py:307:
// argsort(z, kind="stable")), so every run of equal keys is re-ordered by
// (float64 residual z64 - key, primitive index) -- sgs_project's depth_res;
// equal residuals go by index like the stable argsort.  Runs are rare and
// short (configs[2]: ~4 % of the primitives, 2-4 long), so the thread at a
// run's first element sorts it.  keys: the sort's final (sorted) keys; vals:
// the sorted primitive indices, fixed in place; `skip`: a key never sorted.
template <typename K>
__global__ void __launch_bounds__(256) depth_tie_fixup(const K* __restrict__ keys, uint32_t* __restrict__ vals,
                                                       const float* __restrict__ res, const uint32_t* n_ptr,
                                                       uint32_t n_cap, K skip) {
  const uint32_t n = min(*n_ptr, n_cap);
  const uint32_t stride = gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  for (uint32_t base = blockIdx.x * blockDim.x; base < n; base += stride) {
    // neighbours by shuffle: one key load per element
    const uint32_t i = base + threadIdx.x;
    const K k = i < n ? keys[i] : skip;
    K up = (K)__shfl_down_sync(0xffffffffu, (unsigned long long)k, 1);
    K dn = (K)__shfl_up_sync(0xffffffffu, (unsigned long long)k, 1);
    if (lane == 31) up = i + 1 < n ? keys[i + 1] : skip;
    if (lane == 0) dn = i > 0 && i < n ? keys[i - 1] : skip;
    const bool start = i + 1 < n && k != skip && up == k && dn != k;
    if (!__any_sync(0xffffffffu, start) || !start) continue;
    uint32_t j = i + 2;
    while (j < n && keys[j] == k) ++j;
    if (j - i == 2) {  // the common case: a pair
      const uint32_t a = vals[i], b = vals[i + 1];
      const float ra = res[a], rb = res[b];
      if (rb < ra || (rb == ra && b < a)) {
        vals[i] = b;
        vals[i + 1] = a;
      }
      continue;
    }
    constexpr int kRegRun = 8;
    if (j - i <= (uint32_t)kRegRun) {
      // short run (nearly all): every load issued at once, sorted in registers
      const int len = (int)(j - i);
      uint32_t v[kRegRun];
      float r[kRegRun];
#pragma unroll
      for (int a = 0; a < kRegRun; ++a) v[a] = a < len ? vals[i + a] : 0xffffffffu;
#pragma unroll
      for (int a = 0; a < kRegRun; ++a) r[a] = a < len ? res[v[a]] : INFINITY;
      // padding (r = inf, v = ~0) sorts after every real element
      // odd-even transposition sort on (residual, primitive index)
#pragma unroll
      for (int round = 0; round < kRegRun; ++round)
#pragma unroll
        for (int a = round & 1; a + 1 < kRegRun; a += 2)
          if (r[a + 1] < r[a] || (r[a + 1] == r[a] && v[a + 1] < v[a])) {
            const float tr = r[a];
            r[a] = r[a + 1];
            r[a + 1] = tr;
            const uint32_t tv = v[a];
            v[a] = v[a + 1];
            v[a + 1] = tv;
          }
#pragma unroll
      for (int a = 0; a < kRegRun; ++a)
        if (a < len) vals[i + a] = v[a];
      continue;
    }
    for (uint32_t a = i + 1; a < j; ++a) {
      const uint32_t v = vals[a];
      const float r = res[v];
      uint32_t b = a;
      while (b > i) {
        const uint32_t u = vals[b - 1];
        const float ru = res[u];
        if (!(ru > r || (ru == r && u > v))) break;
        vals[b] = u;
        --b;
      }
      vals[b] = v;
    }
  }
}

// Strip renders (a tile-row window): most primitives do not emit, and
// sorting their sentinel keys would make every rank sort all N.  Only the
// emitting primitives' (key, index) enter the depth sort: compacted here,
// one counter atomic per warp; their order does not matter (depth_tie_fixup
// orders equal keys by residual and index).  A separate kernel: done inside
// the preprocess, the returned atomic cost the full-frame path 26 %.
__global__ void __launch_bounds__(256) compact_depth_keys(const uint32_t* __restrict__ depth_key, uint32_t n,
                                                          uint32_t* __restrict__ dkey_c, uint32_t* __restrict__ didx_c,
                                                          uint32_t* __restrict__ count) {
  const int lane = threadIdx.x & 31;
  for (uint32_t base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
    const uint32_t i = base + threadIdx.x;
    const uint32_t k = i < n ? depth_key[i] : 0x7fffffffu;
    const bool e = k != 0x7fffffffu;
    const uint32_t m = __ballot_sync(0xffffffffu, e);
    uint32_t b = 0;
    if (lane == 0 && m) b = atomicAdd(count, (uint32_t)__popc(m));
    b = __shfl_sync(0xffffffffu, b, 0);
    if (e) {
      const uint32_t pos = b + __popc(m & ((1u << lane) - 1u));
      dkey_c[pos] = k;
      didx_c[pos] = i;
    }
  }
}

// ------------------------------------------------------------- entry emission
#ifndef SGS_EMIT_CTAS
#define SGS_EMIT_CTAS 4  // grid = SMs x this (one wave at 4 resident CTAs), grid-stride over the ranks
#endif
__device__ __forceinline__ void unpack_rect(uint2 r, int& tx0, int& ty0, int& tx1, int& ty1) {
  tx0 = (int)(r.x & 0xffff);
  tx1 = (int)(int16_t)(r.x >> 16);
  ty0 = (int)(r.y & 0xffff);
  ty1 = (int)(int16_t)(r.y >> 16);
}

template <typename KT>
__device__ __forceinline__ KT make_key(uint32_t tile, uint32_t dbits) {
  if (sizeof(KT) == 8) return (KT)(((unsigned long long)tile << 32) | dbits);
  return (KT)tile;
}

// Emission (K2), warp-cooperative and load-balanced.  A warp takes 32
// consecutive primitives in rank order; their entries form one contiguous
// output range, ordered by (primitive, row, column).  The warp flattens the
// primitives' rows into a list of row items and processes 32 row items at a
// time: lane = row item computes the row's span (one span evaluation per row,
// no redundancy), a warp scan gives each row's output offset, then lane =
// entry writes 32 consecutive entries per store instruction.
// kSuper: rows are super-tile rows and entries are (super-tile, primitive);
// otherwise rows are tile rows and entries (tile, primitive).
template <typename KT, bool kSuper>
__global__ void __launch_bounds__(256) emit_entries(const uint32_t* __restrict__ perm, uint32_t n_max,
                                                    const uint32_t* __restrict__ n_ptr,
                                                    const uint32_t* __restrict__ counts,
                                                    const uint2* __restrict__ rect,
                                                    const float4* __restrict__ rec_geo,
                                                    const float4* __restrict__ rec_con,
                                                    const float4* __restrict__ rec_span,
                                                    const uint32_t* __restrict__ depth_key,
                                                    const unsigned long long* __restrict__ offsets, SgsCam cam,
                                                    int super_x, uint32_t cap,
                                                    const unsigned long long* __restrict__ total_ptr,
                                                    KT* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
                                                    uint32_t* __restrict__ cell_hist,
                                                    const uint32_t* __restrict__ row_off,
                                                    const uint16_t* __restrict__ row_spans,
                                                    uint2* __restrict__ ranges, int n_cells) {
  // the sort after this kernel accumulates [start, end) per cell with
  // atomicMin / atomicMax: start every cell empty (start > end)
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_cells; i += gridDim.x * blockDim.x)
    ranges[i] = make_uint2(0xffffffffu, 0u);
  // cell_hist (single-pass super-tile sort): counts of the 9-bit cell digit
  // of every written entry, accumulated per CTA in shared memory
  __shared__ uint32_t s_hist[512];
  if (cell_hist) {
    for (int j = threadIdx.x; j < 512; j += blockDim.x) s_hist[j] = 0;
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const uint32_t n = n_ptr ? min(*n_ptr, n_max) : n_max;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const unsigned long long total = *total_ptr;
  const unsigned long long lim = total < cap ? total : cap;
  const int row_w = kSuper ? super_x : cam.tiles_x;
  for (uint32_t base = warp * 32; base < n; base += nwarps * 32) {
    unsigned long long out = offsets[base];  // uniform: every lane reads the same word
    if (out >= lim) continue;
    const uint32_t r = base + lane;
    uint32_t g = 0, nrows = 0, roff = kNoRows;
    int tx0 = 0, ty0 = 0, tx1 = -1, ty1 = -1;
    if (r < n) {
      g = perm ? perm[r] : r;
      if (counts[g]) {
        if (kSuper && row_off) roff = row_off[g];
        unpack_rect(rect[g], tx0, ty0, tx1, ty1);
        nrows = kSuper ? (uint32_t)(ty1 / SGS_SUPER - ty0 / SGS_SUPER + 1) : (uint32_t)(ty1 - ty0 + 1);
      }
    }
    const uint32_t rincl = warp_incl_scan(nrows, lane);
    const uint32_t rstart = rincl - nrows;
    const uint32_t R = __shfl_sync(0xffffffffu, rincl, 31);
    for (uint32_t k0 = 0; k0 < R; k0 += 32) {
      const uint32_t k = k0 + lane;
      const int owner = lane_search(rstart, k);
      const uint32_t og = __shfl_sync(0xffffffffu, g, owner);
      const int oty0 = __shfl_sync(0xffffffffu, ty0, owner);
      const int oty1 = __shfl_sync(0xffffffffu, ty1, owner);
      const int otx0 = __shfl_sync(0xffffffffu, tx0, owner);
      const int otx1 = __shfl_sync(0xffffffffu, tx1, owner);
      const uint32_t ors = __shfl_sync(0xffffffffu, rstart, owner);
      const uint32_t ooff = __shfl_sync(0xffffffffu, roff, owner);
      const int row = (kSuper ? oty0 / SGS_SUPER : oty0) + (int)(k - ors);
      uint32_t c = 0;
      int first = 0;
      int rf[SGS_SUPER] = {0, 0, 0, 0}, rc[SGS_SUPER] = {0, 0, 0, 0};
      if (k < R) {
        if (kSuper && ooff != kNoRows) {
          // the preprocess's stored row spans (the values sgs_super_row_spans
          // gives): the four loads are issued together (rows outside the
          // rectangle read a clamped row and are masked), columns are >= 0
          uint32_t e[SGS_SUPER];
#pragma unroll
          for (int q = 0; q < SGS_SUPER; ++q) {
            const int ty = min(max(row * SGS_SUPER + q, oty0), oty1);
            e[q] = row_spans[ooff + (uint32_t)(ty - oty0)];
          }
          int lo = 0x7fffffff, hi = -1;
#pragma unroll
          for (int q = 0; q < SGS_SUPER; ++q) {
            const int ty = row * SGS_SUPER + q;
            const bool in = ty >= oty0 && ty <= oty1;
            rc[q] = in ? (int)(e[q] >> 8) : 0;
            rf[q] = rc[q] > 0 ? otx0 + (int)(e[q] & 0xffu) : 0;
            const int a = (int)((uint32_t)rf[q] >> 2), b = (int)((uint32_t)(rf[q] + rc[q] - 1) >> 2);
            lo = rc[q] > 0 && a < lo ? a : lo;
            hi = rc[q] > 0 && b > hi ? b : hi;
          }
          first = hi >= lo ? lo : 0;
          c = hi >= lo ? (uint32_t)(hi - lo + 1) : 0u;
        } else {
          const float4 g4 = rec_geo[og], c4 = rec_con[og];
          const float4 s2 = rec_span[og];
          const float geo[4] = {g4.x, g4.y, g4.z, g4.w}, con[4] = {c4.x, c4.y, c4.z, c4.w};
          const float span2[3] = {s2.x, s2.y, s2.z};
          const SgsSpan sp = sgs_span_cached(geo, con, span2);
          c = kSuper ? (uint32_t)sgs_super_row_spans(&sp, &cam, otx0, oty0, otx1, oty1, row, rf, rc, &first)
                     : (uint32_t)sgs_row_span(&sp, &cam, row, otx0, otx1, &first);
        }
      }
      const uint32_t cincl = warp_incl_scan(c, lane);
      const uint32_t cexcl = cincl - c;
      const uint32_t Ctot = __shfl_sync(0xffffffffu, cincl, 31);
      for (uint32_t j0 = 0; j0 < Ctot; j0 += 32) {
        const uint32_t j = j0 + lane;
        const int ro = lane_search(cexcl, j);
        const int rfirst = __shfl_sync(0xffffffffu, first, ro);
        const int rrow = __shfl_sync(0xffffffffu, row, ro);
        const uint32_t rex = __shfl_sync(0xffffffffu, cexcl, ro);
        const uint32_t rg = __shfl_sync(0xffffffffu, og, ro);
        int mf[SGS_SUPER], mc[SGS_SUPER];
        if (kSuper) {
#pragma unroll
          for (int q = 0; q < SGS_SUPER; ++q) {
            mf[q] = __shfl_sync(0xffffffffu, rf[q], ro);
            mc[q] = __shfl_sync(0xffffffffu, rc[q], ro);
          }
        }
        if (j < Ctot) {
          const unsigned long long o = out + j;
          if (o < lim) {
            const uint32_t col = (uint32_t)rfirst + (j - rex);
            const uint32_t cell = (uint32_t)(rrow * row_w) + col;
            if (kSuper) {
              keys_out[o] = (KT)((cell << 16) | sgs_super_mask_fast(mf, mc, (int)col));
              if (cell_hist) atomicAdd(&s_hist[cell & 511u], 1u);
            }
            else
              keys_out[o] = make_key<KT>(cell, sizeof(KT) == 8 ? depth_key[rg] : 0u);
            vals_out[o] = rg;
          }
        }
      }
      out += Ctot;
    }
  }
  if (cell_hist) {
    __syncthreads();
    for (int j = threadIdx.x; j < 512; j += blockDim.x)
      if (s_hist[j]) atomicAdd(&cell_hist[j], s_hist[j]);
  }
}

// Final location of the sorted values (which ping-pong buffer).
bool final_in_alt(const Layout& lo) {
  int passes = lo.sort_mode == SGS_SORT_KEY64 ? tile_sort_passes(lo.n_tiles) : super_sort_passes(lo.n_super);
  return (passes & 1) != 0;
}

template <typename KT, int IPT, int RBITS, bool kSuper>
static int bin_entries(const SgsCam& cam, const sgs_workspace* ws, const Layout& lo, const uint32_t* perm,
                       const uint32_t* n_ptr, int key_bits, int tile_shift, cudaStream_t st) {
  // the emission accumulates the histogram when the cell sort is one 9-bit pass
  const bool fused_hist = kSuper && RBITS == 9 && key_bits <= 9;
  Counters* ctr = at<Counters>(ws, lo.counters);
  const uint32_t n = (uint32_t)lo.n;
  const uint32_t cap = (uint32_t)lo.cap;
  KT* k0 = at<KT>(ws, lo.ent_key);
  KT* k1 = at<KT>(ws, lo.ent_key_alt);
  uint32_t* v0 = at<uint32_t>(ws, lo.ent_val);
  uint32_t* v1 = at<uint32_t>(ws, lo.ent_val_alt);
  uint2* ranges = at<uint2>(ws, lo.ranges);
  const int n_cells = kSuper ? lo.n_super : lo.n_tiles;
  // the emission accumulates the cell digit counts (fused_hist): from zero on
  // every sgs_bin, which may be repeated after one sgs_preprocess
  if (fused_hist) SGS_CUDA(cudaMemsetAsync(at<uint32_t>(ws, lo.hist) + kSuperHistOff, 0, 512 * 4, st));
  emit_entries<KT, kSuper><<<persistent_grid(n, 256, SGS_EMIT_CTAS), 256, 0, st>>>(
      perm, n, n_ptr, at<uint32_t>(ws, kSuper ? lo.super_touched : lo.tiles_touched), at<uint2>(ws, lo.rect),
      at<float4>(ws, lo.rec_geo), at<float4>(ws, lo.rec_con), at<float4>(ws, lo.rec_span),
      at<uint32_t>(ws, lo.depth_key),
      at<unsigned long long>(ws, lo.offsets), cam, lo.super_x, cap, &ctr->n_bin, k0, v0,
      fused_hist ? at<uint32_t>(ws, lo.hist) + kSuperHistOff : nullptr,
      lo.row_cap ? at<uint32_t>(ws, lo.row_off) : nullptr, lo.row_cap ? at<uint16_t>(ws, lo.row_spans) : nullptr,
      ranges, n_cells);
  SGS_LAUNCH_CHECK("emit_entries");
  bool alt = false;
  // the cell sort's digit counts live apart from the preprocess's depth
  // histograms (kDepthHistOff), which a repeated sgs_bin reads again
  uint32_t* hist = at<uint32_t>(ws, lo.hist) + kSuperHistOff;
  int rc = radix_sort_pairs<KT, IPT, RBITS>(k0, v0, k1, v1, &ctr->n_sort, cap, key_bits, hist,
                                     at<uint32_t>(ws, lo.status), &ctr->part_counter[8], &alt, st, false,
                                     RsRangeOut{ranges, tile_shift}, tile_shift, true, fused_hist);
  if (rc) return rc;
  // both key forms were emitted in the float64 depth order (ties fixed up
  // before the emission), so the stable sort over the cell digits alone
  // gives (cell, depth, residual, index) order: for 64-bit keys the LSD
  // passes over the already-ordered low 32 depth bits are skipped
  // cells without entries keep (0xffffffff, 0): every consumer reads a range
  // as [start, max(start, end)), i.e. empty
  return rc;
}

int launch_bin(const SgsCam& cam, const sgs_workspace* ws, const Layout& lo, cudaStream_t st) {
  Counters* ctr = at<Counters>(ws, lo.counters);
  const uint32_t n = (uint32_t)lo.n;
  const uint32_t cap = (uint32_t)lo.cap;
  unsigned long long* offsets = at<unsigned long long>(ws, lo.offsets);
  unsigned long long* status64 = at<unsigned long long>(ws, lo.scan_blocks);  // scan look-back status
  uint32_t* ka = at<uint32_t>(ws, lo.dkey_alt);
  uint32_t* kb = at<uint32_t>(ws, lo.dkey_tmp);
  uint32_t* ia = at<uint32_t>(ws, lo.didx);
  uint32_t* ib = at<uint32_t>(ws, lo.didx_alt);
  bool alt = false;
  // Both modes first sort the primitives by depth: 31-bit keys
  // (0x7fffffff = not emitting), 4 passes, the four digit histograms
  // accumulated by the preprocess.  Full frames sort all N primitives
  // (n_depth = N), the first pass reading the preprocess's keys in place;
  // strip renders sort only the emitting ones, compacted first.  Either input
  // is left intact, so sgs_bin may be repeated after one sgs_preprocess.
  const bool window = cam.tile_y0 > 0 || cam.tile_y1 < cam.tiles_y;
  const uint32_t* k_first = at<uint32_t>(ws, lo.depth_key);
  const uint32_t* v_first = nullptr;
  if (window) {
    SGS_CUDA(cudaMemsetAsync(&ctr->n_depth, 0, sizeof(uint32_t), st));
    compact_depth_keys<<<persistent_grid(n, 256, 8), 256, 0, st>>>(at<uint32_t>(ws, lo.depth_key), n,
                                                                 at<uint32_t>(ws, lo.dkey_c),
                                                                 at<uint32_t>(ws, lo.didx_c), &ctr->n_depth);
    SGS_LAUNCH_CHECK("compact_depth_keys");
    k_first = at<uint32_t>(ws, lo.dkey_c);
    v_first = at<uint32_t>(ws, lo.didx_c);
  }
  int rc = radix_sort_pairs<uint32_t, kDepthSortIPT, 8, kDepthSortThreads>(
      ka, ia, kb, ib, &ctr->n_depth, n, 31, at<uint32_t>(ws, lo.hist) + kDepthHistOff,
      at<uint32_t>(ws, lo.status), &ctr->part_counter[0], &alt, st, !window, RsRangeOut{nullptr, 0}, 0, false,
      true, k_first, v_first);
  if (rc) return rc;
  uint32_t* perm = alt ? ib : ia;
  depth_tie_fixup<uint32_t><<<persistent_grid(n, 256, 8), 256, 0, st>>>(
      alt ? kb : ka, perm, at<float>(ws, lo.depth_res), &ctr->n_depth, n, 0x7fffffffu);
  SGS_LAUNCH_CHECK("depth_tie_fixup");
  if (lo.sort_mode == SGS_SORT_DEPTH_FIRST) {
    rc = launch_scan(at<uint32_t>(ws, lo.super_touched), perm, n, &ctr->n_depth, cap, status64, offsets, ctr, st);
    if (rc) return rc;
    // keys (super_id << 16 | 16-bit tile mask), sorted on the super id bits only
    const int sbits = tile_sort_bits(lo.n_super);
    if (sbits <= 9)
      return bin_entries<uint32_t, kTileSortIPT, 9, true>(cam, ws, lo, perm, &ctr->n_depth, sbits, 16, st);
    return bin_entries<uint32_t, kTileSortIPT, 8, true>(cam, ws, lo, perm, &ctr->n_depth, sbits, 16, st);
  }
  // SGS_SORT_KEY64: (tile << 32 | depth bits) keys emitted in depth order,
  // sorted on the tile bits
  rc = launch_scan(at<uint32_t>(ws, lo.tiles_touched), perm, n, &ctr->n_depth, cap, status64, offsets, ctr, st);
  if (rc) return rc;
  return bin_entries<unsigned long long, kKey64SortIPT, 8, false>(cam, ws, lo, perm, &ctr->n_depth,
                                                                  tile_sort_bits(lo.n_tiles), 32, st);
}

// Generic 64-bit pair sort exported through the ABI (for tests / tools).
uint64_t sort_u64_temp_bytes(uint64_t n, int bits) {
  const uint64_t parts = rs_parts<unsigned long long, kKey64SortIPT>(n);
  const int passes = (bits + 7) / 8;
  return align256(n * 8) + align256(n * 4) + 16 * 512 * 4 + 256 + parts * 512 * 4 * passes + 64;
}

int launch_sort_u64(unsigned long long* keys, uint32_t* vals, uint32_t n, int bits, void* temp, uint64_t temp_bytes,
                    cudaStream_t st) {
  const uint64_t need = sort_u64_temp_bytes(n, bits);
  if (temp_bytes < need) {
    set_error("sort temp too small: need %llu", (unsigned long long)need);
    return SGS_E_WORKSPACE;
  }
  char* p = reinterpret_cast<char*>(temp);
  auto* k1 = reinterpret_cast<unsigned long long*>(p);
  p += align256((uint64_t)n * 8);
  auto* v1 = reinterpret_cast<uint32_t*>(p);
  p += align256((uint64_t)n * 4);
  uint32_t* hist = reinterpret_cast<uint32_t*>(p);
  p += 16 * 512 * 4;
  uint32_t* meta = reinterpret_cast<uint32_t*>(p);  // [0] = n, [1..16] tickets
  p += 256;
  uint32_t* status = reinterpret_cast<uint32_t*>(p);
  set_count<<<1, 1, 0, st>>>(meta, n);
  SGS_LAUNCH_CHECK("set_count");
  bool alt = false;
  int rc = radix_sort_pairs<unsigned long long, kKey64SortIPT, 8>(keys, vals, k1, v1, meta, n, bits, hist, status,
                                                               meta + 1, &alt, st);
  if (rc) return rc;
  if (alt) {
    SGS_CUDA(cudaMemcpyAsync(keys, k1, (size_t)n * 8, cudaMemcpyDeviceToDevice, st));
    SGS_CUDA(cudaMemcpyAsync(vals, v1, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
  }
  return SGS_OK;
}

}  // namespace sgs
