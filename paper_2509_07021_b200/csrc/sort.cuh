// sort.cuh -- stable LSD radix sort of (key, u32 value) pairs, onesweep style:
// one up-front histogram kernel computes every pass's 256-bin digit counts
// in a single read of the keys, then each 8-bit pass is ONE kernel that
// ranks a tile of keys in shared memory (warp match_any + per-warp digit
// histograms, order-preserving), publishes its per-digit counts, resolves
// its global digit offsets by decoupled look-back over earlier tiles, and
// scatters keys/values through shared memory.
//
// Persistent: the grid is at most the number of co-resident CTAs and tiles
// are claimed in order from an atomic ticket, so look-back always waits on a
// CTA that is running.  Item counts are read from device memory, so a whole
// frame can be enqueued (or graph-captured) without a host round trip.
#pragma once

#include "common.cuh"

namespace sgs {

// status word: [31:30] flag (0 empty, 1 aggregate, 2 inclusive prefix), [29:0] count
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagInc = 2u << 30;
constexpr uint32_t kCountMask = (1u << 30) - 1;

template <typename K>
__device__ __forceinline__ uint32_t rs_digit(K k, int shift) {
  return (uint32_t)(k >> shift) & 0xffu;
}

// Lanes of the warp holding the same 8-bit digit, from 8 ballots (cheaper
// than match.any on sm_100).  Lanes outside `valid` never match.
__device__ __forceinline__ uint32_t match_digit8(uint32_t d, uint32_t valid) {
  uint32_t peers = valid;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const uint32_t bit = (d >> b) & 1u;
    const uint32_t m = __ballot_sync(0xffffffffu, bit);
    peers &= bit ? m : ~m;
  }
  return peers;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Histogram of `num_passes` digits starting at bit `begin_bit`; hist is
// num_passes x 256 u32 and must be zeroed.  n = min(*n_ptr, n_cap).
template <typename K>
__global__ void __launch_bounds__(256) rs_histogram(const K* __restrict__ keys, const uint32_t* n_ptr, uint32_t n_cap,
                                                    int begin_bit, int num_passes, uint32_t* __restrict__ hist) {
  // one private 256-bin histogram per warp and pass (contention stays inside a warp)
  extern __shared__ uint32_t sh[];  // [num_passes][8][256]
  const uint32_t n = min(*n_ptr, n_cap);
  const int w = threadIdx.x >> 5;
  for (int j = threadIdx.x; j < num_passes * 8 * 256; j += 256) sh[j] = 0;
  __syncthreads();
  for (uint32_t i = blockIdx.x * 256u + threadIdx.x; i < n; i += gridDim.x * 256u) {
    K k = keys[i];
#pragma unroll 1
    for (int p = 0; p < num_passes; ++p) atomicAdd(&sh[(p * 8 + w) * 256 + rs_digit(k, begin_bit + 8 * p)], 1u);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < num_passes * 256; j += 256) {
    const int p = j >> 8, d = j & 255;
    uint32_t v = 0;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) v += sh[(p * 8 + ww) * 256 + d];
    if (v) atomicAdd(&hist[j], v);
  }
}

// In-place exclusive scan of each pass's 256 bins (one CTA per pass).
__global__ void __launch_bounds__(256) rs_scan_hist(uint32_t* hist) {
  __shared__ uint32_t warp_tot[8];
  uint32_t* h = hist + blockIdx.x * 256;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  uint32_t v = h[t], x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  uint32_t pre = 0;
  for (int i = 0; i < w; ++i) pre += warp_tot[i];
  h[t] = pre + x - v;
}

template <typename K, int IPT>
struct RsSmem {
  static constexpr int kTile = 256 * IPT;
  uint32_t warp_hist[8][256];
  uint32_t digit_start[256];
  uint32_t global_base[256];
  uint32_t warp_tot[8];
  uint32_t part;
  K keys[kTile];
  uint32_t vals[kTile];
};

// One 8-bit pass.  status: nparts x 256 u32, zeroed; ticket zeroed.
template <typename K, int IPT>
__global__ void __launch_bounds__(256) rs_onesweep(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                   K* __restrict__ kout, uint32_t* __restrict__ vout,
                                                   const uint32_t* n_ptr, uint32_t n_cap, int shift,
                                                   const uint32_t* __restrict__ pass_base, uint32_t* status,
                                                   uint32_t* ticket) {
  using S = RsSmem<K, IPT>;
  constexpr int kTile = S::kTile;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S& s = *reinterpret_cast<S*>(smem_raw);
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const uint32_t n = min(*n_ptr, n_cap);
  const uint32_t nparts = (n + kTile - 1) / kTile;
  const uint32_t lt = lanemask_lt();

  for (;;) {
    if (t == 0) s.part = atomicAdd(ticket, 1u);
    for (int j = t; j < 8 * 256; j += 256) (&s.warp_hist[0][0])[j] = 0;
    __syncthreads();
    const uint32_t part = s.part;
    if (part >= nparts) return;

    // ---- load (warp-striped) and rank within the warp, order-preserving
    const uint32_t base = part * kTile + w * 32 * IPT;
    K keys[IPT];
    uint32_t vals[IPT], rank[IPT];
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      uint32_t idx = base + i * 32 + lane;
      bool valid = idx < n;
      keys[i] = valid ? kin[idx] : K(0);
      vals[i] = valid ? vin[idx] : 0u;
    }
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      uint32_t idx = base + i * 32 + lane;
      bool valid = idx < n;
      uint32_t d = rs_digit(keys[i], shift);
      uint32_t peers = match_digit8(d, __ballot_sync(0xffffffffu, valid));
      uint32_t before = valid ? s.warp_hist[w][d] : 0u;
      __syncwarp();
      if (valid && (peers & lt) == 0) s.warp_hist[w][d] = before + __popc(peers);
      __syncwarp();
      rank[i] = before + __popc(peers & lt);
    }
    __syncthreads();

    // ---- per digit: scan over warps, publish, look back
    uint32_t run = 0;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) {
      uint32_t c = s.warp_hist[ww][t];
      s.warp_hist[ww][t] = run;
      run += c;
    }
    uint32_t* my_status = status + (size_t)part * 256 + t;
    if (part == 0) {
      atomicExch(my_status, kFlagInc | run);
    } else {
      atomicExch(my_status, kFlagAgg | run);
    }
    // block exclusive scan of run over digits -> digit_start
    {
      uint32_t x = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) s.warp_tot[w] = x;
      __syncthreads();
      uint32_t pre = 0;
      for (int i = 0; i < w; ++i) pre += s.warp_tot[i];
      s.digit_start[t] = pre + x - run;
    }
    uint32_t excl = 0;
    if (part > 0) {
      int64_t p = (int64_t)part - 1;
      for (;;) {
        uint32_t v = *reinterpret_cast<volatile uint32_t*>(status + (size_t)p * 256 + t);
        uint32_t flag = v & ~kCountMask;
        if (flag == 0) continue;
        excl += v & kCountMask;
        if (flag == kFlagInc) break;
        --p;
      }
      atomicExch(my_status, kFlagInc | (excl + run));
    }
    s.global_base[t] = pass_base[t] + excl;
    __syncthreads();

    // ---- scatter into shared memory in local sorted order
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      uint32_t idx = base + i * 32 + lane;
      if (idx < n) {
        uint32_t d = rs_digit(keys[i], shift);
        uint32_t pos = s.digit_start[d] + s.warp_hist[w][d] + rank[i];
        s.keys[pos] = keys[i];
        s.vals[pos] = vals[i];
      }
    }
    __syncthreads();
    const uint32_t cnt = min((uint32_t)kTile, n - part * kTile);
    for (uint32_t j = t; j < cnt; j += 256) {
      K k = s.keys[j];
      uint32_t d = rs_digit(k, shift);
      uint32_t g = s.global_base[d] + j - s.digit_start[d];
      kout[g] = k;
      vout[g] = s.vals[j];
    }
    __syncthreads();
  }
}

int resident_ctas_per_sm(const void* kernel, int threads, size_t smem);
int device_sm_count();

// Sort `n_cap`-bounded pairs (count in *n_ptr on the device) over bits
// [0, bits).  Ping-pongs between (k0, v0) and (k1, v1); returns in *result_in_alt
// whether the sorted data ends in (k1, v1).  hist: 16*256 u32; status: parts*256*passes u32;
// tickets: >= passes u32; all three zeroed by this function.
template <typename K, int IPT>
int radix_sort_pairs(K* k0, uint32_t* v0, K* k1, uint32_t* v1, const uint32_t* n_ptr, uint32_t n_cap, int bits,
                     uint32_t* hist, uint32_t* status, uint32_t* tickets, bool* result_in_alt, cudaStream_t st) {
  const int passes = (bits + 7) / 8;
  constexpr int kTile = 256 * IPT;
  const uint64_t parts = ((uint64_t)n_cap + kTile - 1) / kTile;
  *result_in_alt = false;
  if (n_cap == 0 || passes == 0) return SGS_OK;
  SGS_CUDA(cudaMemsetAsync(hist, 0, (size_t)passes * 256 * 4, st));
  SGS_CUDA(cudaMemsetAsync(status, 0, (size_t)parts * 256 * 4 * passes, st));
  SGS_CUDA(cudaMemsetAsync(tickets, 0, (size_t)passes * 4, st));
  const int sms = device_sm_count();
  int hgrid = (int)std::min<uint64_t>((n_cap + 256 * 32 - 1) / (256 * 32), (uint64_t)sms * 4);
  if (hgrid < 1) hgrid = 1;
  const size_t hsmem = (size_t)passes * 8 * 256 * 4;
  if (hsmem > 48 * 1024) {
    SGS_CUDA(cudaFuncSetAttribute(rs_histogram<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsmem));
  }
  rs_histogram<K><<<hgrid, 256, hsmem, st>>>(k0, n_ptr, n_cap, 0, passes, hist);
  SGS_LAUNCH_CHECK("rs_histogram");
  rs_scan_hist<<<passes, 256, 0, st>>>(hist);
  SGS_LAUNCH_CHECK("rs_scan_hist");
  const size_t smem = sizeof(RsSmem<K, IPT>);
  static bool attr_set = false;
  if (!attr_set) {
    SGS_CUDA(cudaFuncSetAttribute(rs_onesweep<K, IPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_set = true;
  }
  const int per_sm = resident_ctas_per_sm((const void*)rs_onesweep<K, IPT>, 256, smem);
  if (per_sm < 1) {
    set_error("onesweep kernel cannot be resident");
    return SGS_E_CUDA;
  }
  const int grid = (int)std::min<uint64_t>(parts, (uint64_t)sms * per_sm);
  K* ka = k0;
  K* kb = k1;
  uint32_t* va = v0;
  uint32_t* vb = v1;
  for (int p = 0; p < passes; ++p) {
    rs_onesweep<K, IPT><<<grid, 256, smem, st>>>(ka, va, kb, vb, n_ptr, n_cap, 8 * p, hist + 256 * p,
                                                  status + (size_t)parts * 256 * p, tickets + p);
    SGS_LAUNCH_CHECK("rs_onesweep");
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  *result_in_alt = (passes & 1) != 0;
  return SGS_OK;
}

}  // namespace sgs
