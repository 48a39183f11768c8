// binning.cu -- K2 duplicate-with-keys, K3 sort, K4 tile ranges.
//
// The reference orders primitives with one global stable argsort on depth
// (/root/reference/pkg/src/sgsplat/render.py:307) and blends every pixel
// against every primitive.  The tiled renderer needs, per 16x16 tile, the
// primitives whose support meets the tile in (depth, index) order.  The
// contract is the list of 64-bit keys (tile << 32 | depth_bits) with
// primitive-index values, stably sorted, plus per-tile [start, end) ranges.
//
// Two bit-identical ways to produce it:
//   SGS_SORT_KEY64       emit entries in primitive-index order with the full
//                        64-bit key and radix-sort 32 + ceil(log2 T) bits
//                        (6 onesweep passes at 1080p, 24 B/entry/pass);
//   SGS_SORT_DEPTH_FIRST radix-sort the N primitives once on their 31-bit
//                        depth keys (4 passes over N, not E), emit entries in
//                        that (depth, index) order carrying only the tile id,
//                        then stably radix-sort on the tile id alone
//                        (ceil(log2 T / 8) passes: 2 at 1080p and 4K, 16 B per
//                        entry per pass).  A stable sort on tile of a list
//                        already ordered by (depth, index) yields exactly the
//                        (tile, depth, index) order of the 64-bit sort.
#include <algorithm>
#include <utility>

#include "sort.cuh"

namespace sgs {

// ---------------------------------------------------------------- scan (u64)
// offsets[r] = sum_{r' < r} tiles_touched[perm ? perm[r'] : r'] ; totals -> counters
constexpr int kScanItems = 2048;  // per CTA (256 threads x 8)

__device__ __forceinline__ uint32_t scan_load(const uint32_t* tt, const uint32_t* perm, uint32_t r) {
  return tt[perm ? perm[r] : r];
}

__global__ void __launch_bounds__(256) scan_reduce(const uint32_t* __restrict__ tt, const uint32_t* __restrict__ perm,
                                                   uint32_t n, unsigned long long* __restrict__ block_sums) {
  __shared__ unsigned long long warp_sum[8];
  const uint32_t b0 = blockIdx.x * kScanItems;
  unsigned long long s = 0;
  for (int i = threadIdx.x; i < kScanItems; i += 256) {
    uint32_t r = b0 + i;
    if (r < n) s += scan_load(tt, perm, r);
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < 8; ++w) t += warp_sum[w];
    block_sums[blockIdx.x] = t;
  }
}

// single CTA: exclusive scan of block sums; writes E, n_sort, overflow
__global__ void __launch_bounds__(1024) scan_blocks(unsigned long long* block_sums, uint32_t nb, uint32_t cap,
                                                    Counters* ctr) {
  __shared__ unsigned long long warp_tot[32];
  __shared__ unsigned long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (uint32_t base = 0; base < nb; base += 1024) {
    uint32_t i = base + threadIdx.x;
    unsigned long long v = i < nb ? block_sums[i] : 0ull, x = v;
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    unsigned long long pre = carry;
    for (int k = 0; k < w; ++k) pre += warp_tot[k];
    if (i < nb) block_sums[i] = pre + x - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry = pre + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    unsigned long long total = carry;
    ctr->n_entries = total;
    ctr->capacity = cap;
    ctr->overflow = total > cap ? 1ull : 0ull;
    ctr->n_sort = (uint32_t)(total < cap ? total : cap);
  }
}

__global__ void __launch_bounds__(256) scan_down(const uint32_t* __restrict__ tt, const uint32_t* __restrict__ perm,
                                                 uint32_t n, const unsigned long long* __restrict__ block_sums,
                                                 unsigned long long* __restrict__ offsets) {
  __shared__ unsigned long long warp_tot[8];
  const uint32_t b0 = blockIdx.x * kScanItems;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // each thread owns 8 consecutive items
  uint32_t v[8];
  unsigned long long s = 0;
  for (int k = 0; k < 8; ++k) {
    uint32_t r = b0 + threadIdx.x * 8 + k;
    v[k] = r < n ? scan_load(tt, perm, r) : 0u;
    s += v[k];
  }
  unsigned long long x = s;
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  unsigned long long pre = block_sums[blockIdx.x];
  for (int k = 0; k < w; ++k) pre += warp_tot[k];
  pre += x - s;
  for (int k = 0; k < 8; ++k) {
    uint32_t r = b0 + threadIdx.x * 8 + k;
    if (r < n) offsets[r] = pre;
    pre += v[k];
  }
}

static int launch_scan(const uint32_t* tt, const uint32_t* perm, uint32_t n, uint32_t cap,
                       unsigned long long* block_sums,
                       unsigned long long* offsets, Counters* ctr, cudaStream_t st) {
  uint32_t nb = (n + kScanItems - 1) / kScanItems;
  if (nb == 0) nb = 1;
  scan_reduce<<<nb, 256, 0, st>>>(tt, perm, n, block_sums);
  SGS_LAUNCH_CHECK("scan_reduce");
  scan_blocks<<<1, 1024, 0, st>>>(block_sums, nb, cap, ctr);
  SGS_LAUNCH_CHECK("scan_blocks");
  scan_down<<<nb, 256, 0, st>>>(tt, perm, n, block_sums, offsets);
  SGS_LAUNCH_CHECK("scan_down");
  return SGS_OK;
}

// ------------------------------------------------------------- entry emission
__device__ __forceinline__ void unpack_rect(uint2 r, int& tx0, int& ty0, int& tx1, int& ty1) {
  tx0 = (int)(r.x & 0xffff);
  tx1 = (int)(int16_t)(r.x >> 16);
  ty0 = (int)(r.y & 0xffff);
  ty1 = (int)(int16_t)(r.y >> 16);
}

template <bool kKey64>
__global__ void __launch_bounds__(256) emit_entries(const uint32_t* __restrict__ perm, uint32_t n,
                                                    const uint32_t* __restrict__ tt, const uint2* __restrict__ rect,
                                                    const float4* __restrict__ rec_geo,
                                                    const float4* __restrict__ rec_con,
                                                    const uint32_t* __restrict__ depth_key,
                                                    const unsigned long long* __restrict__ offsets, SgsCam cam,
                                                    uint32_t cap, void* __restrict__ keys_out,
                                                    uint32_t* __restrict__ vals_out) {
  for (uint32_t r = blockIdx.x * 256 + threadIdx.x; r < n; r += gridDim.x * 256) {
    const uint32_t g = perm ? perm[r] : r;
    const uint32_t cnt = tt[g];
    if (cnt == 0) continue;
    unsigned long long off = offsets[r];
    if (off >= cap) continue;
    int tx0, ty0, tx1, ty1;
    unpack_rect(rect[g], tx0, ty0, tx1, ty1);
    const float4 g4 = rec_geo[g], c4 = rec_con[g];
    const float geo[4] = {g4.x, g4.y, g4.z, g4.w}, con[4] = {c4.x, c4.y, c4.z, c4.w};
    const unsigned long long dbits = kKey64 ? (unsigned long long)depth_key[g] : 0ull;
    const SgsSpan sp = sgs_span(geo, con);
    for (int ty = ty0; ty <= ty1; ++ty) {
      int first;
      const int cnt_row = sgs_row_span(&sp, &cam, ty, tx0, tx1, &first);
      const uint32_t tile0 = (uint32_t)(ty * cam.tiles_x + first);
      for (int j = 0; j < cnt_row; ++j, ++off) {
        if (off >= cap) break;
        if (kKey64)
          reinterpret_cast<unsigned long long*>(keys_out)[off] = ((unsigned long long)(tile0 + j) << 32) | dbits;
        else
          reinterpret_cast<uint32_t*>(keys_out)[off] = tile0 + j;
        vals_out[off] = g;
      }
    }
  }
}

// ---------------------------------------------------------------- tile ranges
template <typename K>
__device__ __forceinline__ uint32_t tile_of(K k) {
  return (uint32_t)(sizeof(K) == 8 ? (k >> 32) : k);
}

template <typename K>
__global__ void __launch_bounds__(256) tile_ranges(const K* __restrict__ keys, const uint32_t* n_ptr,
                                                   uint2* __restrict__ ranges) {
  const uint32_t n = *n_ptr;
  for (uint32_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += gridDim.x * 256) {
    uint32_t t = tile_of(keys[i]);
    if (i == 0 || tile_of(keys[i - 1]) != t) ranges[t].x = i;
    if (i + 1 == n || tile_of(keys[i + 1]) != t) ranges[t].y = i + 1;
  }
}

__global__ void iota_kernel(uint32_t* __restrict__ v, uint32_t n, Counters* ctr) {
  for (uint32_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += gridDim.x * 256) v[i] = i;
  if (blockIdx.x == 0 && threadIdx.x == 0) ctr->n_depth = n;
}

// Final location of the sorted values (which ping-pong buffer).
bool final_in_alt(const Layout& lo) {
  int passes = lo.sort_mode == SGS_SORT_KEY64 ? (32 + tile_sort_bits(lo.n_tiles) + 7) / 8
                                              : tile_sort_passes(lo.n_tiles);
  return (passes & 1) != 0;
}

int launch_bin(const SgsCam& cam, const sgs_workspace* ws, const Layout& lo, cudaStream_t st) {
  Counters* ctr = at<Counters>(ws, lo.counters);
  const uint32_t n = (uint32_t)lo.n;
  const uint32_t cap = (uint32_t)lo.cap;
  const int sms = device_sm_count();
  uint32_t* tt = at<uint32_t>(ws, lo.tiles_touched);
  uint32_t* hist = at<uint32_t>(ws, lo.hist);
  uint32_t* status = at<uint32_t>(ws, lo.status);
  unsigned long long* offsets = at<unsigned long long>(ws, lo.offsets);
  unsigned long long* block_sums = at<unsigned long long>(ws, lo.scan_blocks);
  uint2* ranges = at<uint2>(ws, lo.ranges);
  SGS_CUDA(cudaMemsetAsync(ranges, 0, (size_t)lo.n_tiles * 8, st));
  const int egrid = persistent_grid(n, 256, 8);

  if (lo.sort_mode == SGS_SORT_DEPTH_FIRST) {
    uint32_t* dkey = at<uint32_t>(ws, lo.depth_key);
    uint32_t* dkey_alt = at<uint32_t>(ws, lo.dkey_alt);
    uint32_t* didx = at<uint32_t>(ws, lo.didx);
    uint32_t* didx_alt = at<uint32_t>(ws, lo.didx_alt);
    iota_kernel<<<persistent_grid(n, 256, 8), 256, 0, st>>>(didx, n, ctr);
    SGS_LAUNCH_CHECK("iota_kernel");
    // depth keys are 31-bit (0x7fffffff = not emitting): 4 passes over N.
    // The depth sort must not clobber the preprocess depth keys (exported
    // and used for the 64-bit key view), so sort a copy.
    SGS_CUDA(cudaMemcpyAsync(dkey_alt, dkey, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
    uint32_t* kbuf0 = dkey_alt;
    uint32_t* kbuf1 = at<uint32_t>(ws, lo.dkey_tmp);
    bool alt = false;
    int rc = radix_sort_pairs<uint32_t, kDepthSortIPT>(kbuf0, didx, kbuf1, didx_alt, &ctr->n_depth, n, 31, hist,
                                                        status, &ctr->part_counter[0], &alt, st);
    if (rc) return rc;
    const uint32_t* perm = alt ? didx_alt : didx;
    rc = launch_scan(tt, perm, n, cap, block_sums, offsets, ctr, st);
    if (rc) return rc;
    uint32_t* k0 = at<uint32_t>(ws, lo.ent_key);
    uint32_t* k1 = at<uint32_t>(ws, lo.ent_key_alt);
    uint32_t* v0 = at<uint32_t>(ws, lo.ent_val);
    uint32_t* v1 = at<uint32_t>(ws, lo.ent_val_alt);
    emit_entries<false><<<egrid, 256, 0, st>>>(perm, n, tt, at<uint2>(ws, lo.rect), at<float4>(ws, lo.rec_geo),
                                               at<float4>(ws, lo.rec_con), dkey, offsets, cam, cap, k0, v0);
    SGS_LAUNCH_CHECK("emit_entries");
    rc = radix_sort_pairs<uint32_t, kTileSortIPT>(k0, v0, k1, v1, &ctr->n_sort, cap, tile_sort_bits(lo.n_tiles), hist,
                                                   status, &ctr->part_counter[4], &alt, st);
    if (rc) return rc;
    const uint32_t* kfinal = alt ? k1 : k0;
    tile_ranges<uint32_t><<<persistent_grid(cap, 256, 8), 256, 0, st>>>(kfinal, &ctr->n_sort, ranges);
    SGS_LAUNCH_CHECK("tile_ranges");
  } else {
    uint32_t* dkey = at<uint32_t>(ws, lo.depth_key);
    int rc = launch_scan(tt, nullptr, n, cap, block_sums, offsets, ctr, st);
    if (rc) return rc;
    auto* k0 = at<unsigned long long>(ws, lo.ent_key);
    auto* k1 = at<unsigned long long>(ws, lo.ent_key_alt);
    uint32_t* v0 = at<uint32_t>(ws, lo.ent_val);
    uint32_t* v1 = at<uint32_t>(ws, lo.ent_val_alt);
    emit_entries<true><<<egrid, 256, 0, st>>>(nullptr, n, tt, at<uint2>(ws, lo.rect), at<float4>(ws, lo.rec_geo),
                                              at<float4>(ws, lo.rec_con), dkey, offsets, cam, cap, k0, v0);
    SGS_LAUNCH_CHECK("emit_entries");
    bool alt = false;
    rc = radix_sort_pairs<unsigned long long, kKey64SortIPT>(k0, v0, k1, v1, &ctr->n_sort, cap,
                                                             32 + tile_sort_bits(lo.n_tiles), hist, status,
                                                             &ctr->part_counter[0], &alt, st);
    if (rc) return rc;
    const unsigned long long* kfinal = alt ? k1 : k0;
    tile_ranges<unsigned long long><<<persistent_grid(cap, 256, 8), 256, 0, st>>>(kfinal, &ctr->n_sort, ranges);
    SGS_LAUNCH_CHECK("tile_ranges");
  }
  (void)sms;
  return SGS_OK;
}

// Export the sorted list as 64-bit keys (either mode).
template <typename K>
__global__ void export_keys(const K* __restrict__ keys, const uint32_t* __restrict__ vals,
                            const uint32_t* __restrict__ depth_key, const uint32_t* n_ptr,
                            unsigned long long* __restrict__ out_keys, uint32_t* __restrict__ out_vals) {
  const uint32_t n = *n_ptr;
  for (uint32_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += gridDim.x * 256) {
    uint32_t v = vals[i];
    unsigned long long k;
    if (sizeof(K) == 8)
      k = (unsigned long long)keys[i];
    else
      k = ((unsigned long long)(uint32_t)keys[i] << 32) | depth_key[v];
    out_keys[i] = k;
    out_vals[i] = v;
  }
}

int launch_export_bins(const sgs_workspace* ws, const Layout& lo, unsigned long long* keys, uint32_t* vals,
                       uint32_t* ranges, cudaStream_t st) {
  Counters* ctr = at<Counters>(ws, lo.counters);
  bool alt = final_in_alt(lo);
  const int grid = persistent_grid((uint64_t)lo.cap, 256, 8);
  const uint32_t* v = at<uint32_t>(ws, alt ? lo.ent_val_alt : lo.ent_val);
  if (keys && vals) {
    if (lo.sort_mode == SGS_SORT_KEY64) {
      export_keys<unsigned long long><<<grid, 256, 0, st>>>(
          at<unsigned long long>(ws, alt ? lo.ent_key_alt : lo.ent_key), v, at<uint32_t>(ws, lo.depth_key),
          &ctr->n_sort, keys, vals);
    } else {
      export_keys<uint32_t><<<grid, 256, 0, st>>>(at<uint32_t>(ws, alt ? lo.ent_key_alt : lo.ent_key), v,
                                                  at<uint32_t>(ws, lo.depth_key), &ctr->n_sort, keys, vals);
    }
    SGS_LAUNCH_CHECK("export_keys");
  }
  if (ranges) SGS_CUDA(cudaMemcpyAsync(ranges, at<uint2>(ws, lo.ranges), (size_t)lo.n_tiles * 8,
                                       cudaMemcpyDeviceToDevice, st));
  return SGS_OK;
}

// Generic 64-bit pair sort exported through the ABI (for tests / tools).
int launch_sort_u64(unsigned long long* keys, uint32_t* vals, uint32_t n, int bits, void* temp, uint64_t temp_bytes,
                    cudaStream_t st) {
  constexpr int kTile = 256 * kKey64SortIPT;
  const uint64_t parts = ((uint64_t)n + kTile - 1) / kTile;
  const int passes = (bits + 7) / 8;
  uint64_t need = align256((uint64_t)n * 12) + 16 * 256 * 4 + 256 + parts * 256 * 4 * passes + 64;
  if (temp_bytes < need) {
    set_error("sort temp too small: need %llu", (unsigned long long)need);
    return SGS_E_WORKSPACE;
  }
  char* p = reinterpret_cast<char*>(temp);
  auto* k1 = reinterpret_cast<unsigned long long*>(p);
  auto* v1 = reinterpret_cast<uint32_t*>(p + (uint64_t)n * 8);
  p += align256((uint64_t)n * 12);
  uint32_t* hist = reinterpret_cast<uint32_t*>(p);
  p += 16 * 256 * 4;
  uint32_t* meta = reinterpret_cast<uint32_t*>(p);  // [0] = n, [1..16] tickets
  p += 256;
  uint32_t* status = reinterpret_cast<uint32_t*>(p);
  SGS_CUDA(cudaMemcpyAsync(meta, &n, 4, cudaMemcpyHostToDevice, st));
  bool alt = false;
  int rc = radix_sort_pairs<unsigned long long, kKey64SortIPT>(keys, vals, k1, v1, meta, n, bits, hist, status,
                                                               meta + 1, &alt, st);
  if (rc) return rc;
  if (alt) {
    SGS_CUDA(cudaMemcpyAsync(keys, k1, (size_t)n * 8, cudaMemcpyDeviceToDevice, st));
    SGS_CUDA(cudaMemcpyAsync(vals, v1, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
  }
  return SGS_OK;
}

uint64_t sort_u64_temp_bytes(uint64_t n, int bits) {
  constexpr int kTile = 256 * kKey64SortIPT;
  const uint64_t parts = (n + kTile - 1) / kTile;
  const int passes = (bits + 7) / 8;
  return align256(n * 12) + 16 * 256 * 4 + 256 + parts * 256 * 4 * passes + 64;
}

}  // namespace sgs
