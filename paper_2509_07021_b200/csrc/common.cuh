// common.cuh -- error plumbing, workspace carving and camera setup shared by
// every translation unit of libsgs.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/sgs.h"
#include "sgs_geom.h"

namespace sgs {

constexpr int kNumSMs = 148;
constexpr int kRadixThreads = 512;  // = kRsThreads in sort.cuh
#ifndef SGS_TILE_SORT_IPT
#define SGS_TILE_SORT_IPT 8
#endif
#ifndef SGS_DEPTH_SORT_IPT
#define SGS_DEPTH_SORT_IPT 16
#endif
constexpr int kTileSortIPT = SGS_TILE_SORT_IPT;  // items per thread, tile-key onesweep passes (4096 per CTA)
constexpr int kDepthSortIPT = SGS_DEPTH_SORT_IPT;
#ifndef SGS_DEPTH_SORT_THREADS
#define SGS_DEPTH_SORT_THREADS 512
#endif
// 1M depth keys = 123 tiles of 8192: one wave of one CTA per SM (256-thread CTAs,
// which leave room for co-resident rasters, measured no faster)
constexpr int kDepthSortThreads = SGS_DEPTH_SORT_THREADS;
constexpr int kKey64SortIPT = 6;
constexpr int kScanTicket = 15;       // Counters::part_counter slot of the offsets scan
constexpr int kRowSpansPerPrim = 8;   // row-span store capacity, u16 entries per primitive
constexpr uint32_t kNoRows = 0xffffffffu;  // row_off of a primitive whose spans are not stored
constexpr uint32_t kMaxEntries = (1u << 30) - 1;  // look-back status packs 30-bit counts
// Digit histograms accumulated by producer kernels (depth-first mode): the
// preprocess counts the 4 depth-key digits, the emission the 9-bit
// super-tile digit.  Both live in the workspace's hist buffer, zeroed by
// sgs_preprocess.
constexpr int kDepthHistOff = 0;      // 4 x 256 u32
constexpr int kSuperHistOff = 1024;   // 512 u32

void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);

#define SGS_CUDA(call)                                     \
  do {                                                     \
    cudaError_t e__ = (call);                              \
    if (e__ != cudaSuccess) return sgs::cuda_fail(e__, #call); \
  } while (0)

#define SGS_LAUNCH_CHECK(what)                             \
  do {                                                     \
    cudaError_t e__ = cudaGetLastError();                  \
    if (e__ != cudaSuccess) return sgs::cuda_fail(e__, what); \
  } while (0)

// Device-side counters at the head of the workspace.
struct Counters {
  unsigned long long n_visible;
  unsigned long long n_emitting;
  unsigned long long n_entries;      // exact E (may exceed capacity)
  unsigned long long capacity;
  unsigned long long overflow;
  unsigned long long vram3s_visible;
  unsigned long long vram3s_entries;
  unsigned long long n_bin;          // entries the binning sorts (super-tile entries in depth-first mode)
  uint32_t n_sort;                   // min(E, capacity): items the tile sort processes
  uint32_t n_depth;                  // primitives entering the depth sort
  uint32_t part_counter[16];         // onesweep partition tickets, one per pass; [kScanTicket] the offsets scan
  uint32_t row_alloc;                // row-span store: entries handed out by the preprocess
  uint32_t pad1[13];
};

// Carved workspace.  All sub-buffers 256-byte aligned.
struct Layout {
  int64_t n;
  int32_t L, W, H, tiles_x, tiles_y, n_tiles;
  int32_t super_x, super_y, n_super;
  int32_t sort_mode;
  int64_t cap;
  // offsets into the workspace
  uint64_t counters, rec_geo, rec_con, rec_col, rec_span, rec_eig, depth_key, depth_res, rect, tiles_touched,
      super_touched, cand_end;
  uint64_t cell_order, row_off, row_spans;
  uint64_t row_cap;
  uint64_t dkey_alt, dkey_tmp, didx, didx_alt, dkey_c, didx_c, offsets, scan_blocks;
  uint64_t ent_key, ent_key_alt, ent_val, ent_val_alt, ranges;
  uint64_t hist, status;
  uint64_t status_bytes;
  uint64_t total;
};

inline int ceil_log2_u64(uint64_t x) {
  int b = 0;
  while ((1ull << b) < x) ++b;
  return b;
}

inline int tile_sort_bits(int n_tiles) { return n_tiles <= 1 ? 1 : ceil_log2_u64((uint64_t)n_tiles); }

inline int tile_sort_passes(int n_tiles) { return (tile_sort_bits(n_tiles) + 7) / 8; }

// super-tile id sort: one 9-bit pass when the ids fit (1080p: 510 cells), else 8-bit passes
inline int super_sort_passes(int n_super) {
  const int b = tile_sort_bits(n_super);
  return b <= 9 ? 1 : (b + 7) / 8;
}

inline uint64_t align256(uint64_t x) { return (x + 255) & ~uint64_t(255); }

inline int make_layout(const sgs_workspace* ws, Layout* lo) {
  if (!ws || ws->n < 0 || ws->n > (int64_t)0x7fffffff || ws->width < 1 || ws->height < 1 ||
      ws->n_lobes < 0 || ws->n_lobes > SGS_MAX_LOBES || ws->entry_capacity < 0 ||
      ws->entry_capacity > (int64_t)kMaxEntries || (ws->width + 63) / 64 * ((ws->height + 63) / 64) > 65536 ||
      (ws->sort_mode != SGS_SORT_DEPTH_FIRST && ws->sort_mode != SGS_SORT_KEY64)) {
    set_error("invalid workspace descriptor");
    return SGS_E_ARG;
  }
  lo->n = ws->n;
  lo->L = ws->n_lobes;
  lo->W = ws->width;
  lo->H = ws->height;
  lo->tiles_x = (ws->width + SGS_TILE - 1) / SGS_TILE;
  lo->tiles_y = (ws->height + SGS_TILE - 1) / SGS_TILE;
  lo->n_tiles = lo->tiles_x * lo->tiles_y;
  lo->super_x = (lo->tiles_x + SGS_SUPER - 1) / SGS_SUPER;
  lo->super_y = (lo->tiles_y + SGS_SUPER - 1) / SGS_SUPER;
  lo->n_super = lo->super_x * lo->super_y;
  lo->sort_mode = ws->sort_mode;
  lo->cap = ws->entry_capacity;
  const uint64_t n = (uint64_t)ws->n + 1, cap = (uint64_t)ws->entry_capacity + 1;
  const bool k64 = ws->sort_mode == SGS_SORT_KEY64;
  uint64_t off = 0;
  auto take = [&](uint64_t bytes) {
    uint64_t o = off;
    off = align256(off + bytes);
    return o;
  };
  lo->counters = take(sizeof(Counters));
  lo->rec_geo = take(n * 16);
  lo->rec_con = take(n * 16);
  lo->rec_col = take(n * 16);
  lo->rec_span = take(n * 16);
  lo->rec_eig = take(n * 16);
  lo->depth_key = take(n * 4);
  lo->depth_res = take(n * 4);
  lo->rect = take(n * 8);
  lo->tiles_touched = take(n * 4);
  lo->super_touched = take(n * 4);
  // row-span store (depth-first mode): the preprocess's exact tile-row spans,
  // one u16 per row, read back by the emission instead of re-solving them
  lo->row_cap = ws->sort_mode == SGS_SORT_DEPTH_FIRST ? (uint64_t)kRowSpansPerPrim * n : 0;
  if (lo->row_cap > 0xfffffff0ull) lo->row_cap = 0xfffffff0ull;  // u32 offsets
  lo->row_off = take(n * 4);
  lo->row_spans = take(lo->row_cap * 2);
  lo->cand_end = take((uint64_t)lo->n_tiles * 4);
  lo->cell_order = take((uint64_t)(lo->n_tiles > lo->n_super ? lo->n_tiles : lo->n_super) * 4);
  lo->dkey_alt = take(n * 4);
  lo->dkey_tmp = take(n * 4);
  lo->didx = take(n * 4);
  lo->didx_alt = take(n * 4);
  // strip renders: the emitting primitives' (depth key, index), compacted
  // (the depth sort's read-only first-pass input); both sort modes
  lo->dkey_c = take(n * 4);
  lo->didx_c = take(n * 4);
  lo->offsets = take(n * 8);
  lo->scan_blocks = take(((n + 2047) / 2048 + 1) * 8);
  const uint64_t key_bytes = k64 ? 8 : 4;  // depth-first: (super_id << 16 | tile mask)
  lo->ent_key = take(cap * key_bytes);
  lo->ent_key_alt = take(cap * key_bytes);
  lo->ent_val = take(cap * 4);
  lo->ent_val_alt = take(cap * 4);
  lo->ranges = take((uint64_t)lo->n_tiles * 8);
  lo->hist = take(16 * 512 * 4);
  // onesweep look-back status: per pass, per partition, 256 digits of u32
  // both modes sort the primitives by depth first; the entry sort then runs
  // over the cell id digits only (64-bit keys: the tile bits above bit 32)
  int tile_passes = k64 ? tile_sort_passes(lo->n_tiles) : super_sort_passes(lo->n_super);
  int ipt = k64 ? kKey64SortIPT : kTileSortIPT;
  uint64_t parts_tile = (cap + (uint64_t)kRadixThreads * ipt - 1) / ((uint64_t)kRadixThreads * ipt);
  uint64_t parts_depth =
      (n + (uint64_t)kDepthSortThreads * kDepthSortIPT - 1) / ((uint64_t)kDepthSortThreads * kDepthSortIPT);
  uint64_t st_tile = parts_tile * 512 * 4 * (uint64_t)tile_passes;
  uint64_t st_depth = parts_depth * 256 * 4 * 4;
  lo->status_bytes = st_tile > st_depth ? st_tile : st_depth;
  lo->status = take(lo->status_bytes);
  lo->total = off;
  return SGS_OK;
}

template <typename T>
inline T* at(const sgs_workspace* ws, uint64_t off) {
  return reinterpret_cast<T*>(reinterpret_cast<char*>(ws->base) + off);
}

inline int check_ws(const sgs_workspace* ws, Layout* lo) {
  int rc = make_layout(ws, lo);
  if (rc) return rc;
  if (!ws->base || ws->bytes < lo->total) {
    set_error("workspace too small: have %llu bytes, need %llu",
              (unsigned long long)ws->bytes, (unsigned long long)lo->total);
    return SGS_E_WORKSPACE;
  }
  return SGS_OK;
}

inline int make_cam(const sgs_camera* c, const Layout& lo, SgsCam* out) {
  if (!c || !(c->fx > 0.0f) || !(c->fy > 0.0f) || c->width != lo.W || c->height != lo.H) {
    set_error("invalid camera (focal lengths must be positive and size must match workspace)");
    return SGS_E_ARG;
  }
  for (int i = 0; i < 9; ++i) out->R[i] = c->rotation[i];
  for (int i = 0; i < 3; ++i) out->t[i] = c->translation[i];
  // C = -R^T t (render.py:54-57), computed in double and rounded once
  for (int k = 0; k < 3; ++k) {
    double s = 0.0;
    for (int i = 0; i < 3; ++i) s += (double)c->rotation[3 * i + k] * (double)c->translation[i];
    out->C[k] = (float)(-s);
  }
  out->fx = c->fx;
  out->fy = c->fy;
  out->cx = c->cx;
  out->cy = c->cy;
  out->near_z = c->near_z;
  out->width = c->width;
  out->height = c->height;
  out->tiles_x = lo.tiles_x;
  out->tiles_y = lo.tiles_y;
  int y0 = c->tile_y0, y1 = c->tile_y1;
  if (y0 == 0 && y1 == 0) y1 = lo.tiles_y;
  if (y0 < 0 || y1 > lo.tiles_y || y0 >= y1) {
    set_error("invalid tile-row window [%d, %d) for %d tile rows", y0, y1, lo.tiles_y);
    return SGS_E_ARG;
  }
  out->tile_y0 = y0;
  out->tile_y1 = y1;
  if (!(c->lowpass >= 0.0f)) {
    set_error("lowpass must be >= 0");
    return SGS_E_ARG;
  }
  out->lowpass = c->lowpass;
  const bool have64 = c->depth_row[0] != 0.0 || c->depth_row[1] != 0.0 || c->depth_row[2] != 0.0 ||
                      c->depth_row[3] != 0.0;
  for (int k = 0; k < 3; ++k) out->rz[k] = have64 ? c->depth_row[k] : (double)c->rotation[6 + k];
  out->tz = have64 ? c->depth_row[3] : (double)c->translation[2];
  out->near64 = c->near_z64 > 0.0 ? c->near_z64 : (double)c->near_z;
  if (!(c->grad_floor >= 0.0f) || c->grad_floor > 1.0f) {
    set_error("grad_floor must be in [0, 1]");
    return SGS_E_ARG;
  }
  out->grad_floor = c->grad_floor;
  return SGS_OK;
}


// ------------------------------------------------------------ warp helpers
#ifdef __CUDACC__
// Largest lane L with x_L <= k, for x non-decreasing across lanes and x_0 <= k.
__device__ __forceinline__ int lane_search(uint32_t x, uint32_t k) {
  int L = 0;
#pragma unroll
  for (int step = 16; step >= 1; step >>= 1) {
    const int c = L + step;
    if (__shfl_sync(0xffffffffu, x, c & 31) <= k && c < 32) L = c;
  }
  return L;
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  return v;
}


// Broadcast lane `src`'s span record to every lane.
__device__ __forceinline__ SgsSpan shfl_span(const SgsSpan& s, int src) {
  SgsSpan o;
  o.mx = __shfl_sync(0xffffffffu, s.mx, src);
  o.my = __shfl_sync(0xffffffffu, s.my, src);
  o.kb = __shfl_sync(0xffffffffu, s.kb, src);
  o.D = __shfl_sync(0xffffffffu, s.D, src);
  o.Q = __shfl_sync(0xffffffffu, s.Q, src);
  o.kx = __shfl_sync(0xffffffffu, s.kx, src);
  o.xm = __shfl_sync(0xffffffffu, s.xm, src);
  o.ym = __shfl_sync(0xffffffffu, s.ym, src);
  o.i2a = __shfl_sync(0xffffffffu, s.i2a, src);
  o.valid = __shfl_sync(0xffffffffu, s.valid, src);
  return o;
}
#endif

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// persistent grid: a whole number of waves of `per_sm` resident CTAs
inline int persistent_grid(uint64_t work_items, int items_per_cta, int per_sm) {
  uint64_t need = (work_items + items_per_cta - 1) / items_per_cta;
  uint64_t cap = (uint64_t)kNumSMs * per_sm;
  if (need < 1) need = 1;
  return (int)(need < cap ? need : cap);
}

}  // namespace sgs
