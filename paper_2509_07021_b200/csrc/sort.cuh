// sort.cuh -- stable LSD radix sort of (key, u32 value) pairs, onesweep style:
// one up-front histogram kernel computes every pass's digit counts in a
// single (vectorised) read of the keys, then each pass is ONE kernel that
// ranks a tile of keys in shared memory (warp ballot-match + per-warp digit
// counters, order-preserving), publishes its per-digit counts, resolves its
// global digit offsets by decoupled look-back over earlier tiles, and
// scatters keys / values through shared memory so the global writes are runs
// of consecutive addresses.  Digits are RBITS wide (8 or 9 bits: a 9-bit key
// range -- the super-tile ids of a 1080p frame -- sorts in a single pass).
//
// Persistent: the grid is at most the number of co-resident CTAs and tiles
// are claimed in order from an atomic ticket, so look-back only ever waits on
// a CTA that is running.  Item counts are read from device memory, so a whole
// frame can be enqueued (or graph-captured) without a host round trip.
//
// The final pass of a tile-key sort can also emit the per-cell [start, end)
// ranges: a cell's entries form one contiguous run inside each CTA's
// shared-memory order, so each run contributes one atomicMin / atomicMax
// (K4 fused into K3).
#pragma once

#include <algorithm>
#include <utility>

#include "common.cuh"

namespace sgs {

// status word: [31:30] flag (0 empty, 1 aggregate, 2 inclusive prefix), [29:0] count
enum : uint32_t { kFlagAgg = 1u << 30, kFlagInc = 2u << 30, kCountMask = (1u << 30) - 1 };

constexpr int kRsThreads = 512;  // default CTA size: 16 warps

constexpr int kRsMaxRadix = 512;
#ifndef SGS_RS_LOOKBACK
#define SGS_RS_LOOKBACK 8
#endif
constexpr int kLookback = SGS_RS_LOOKBACK;  // predecessors examined per look-back step

template <typename K, int RBITS>
__device__ __forceinline__ uint32_t rs_digit(K k, int shift) {
  return (uint32_t)(k >> shift) & ((1u << RBITS) - 1u);
}

// Lanes of the warp holding the same RBITS-bit digit, from RBITS ballots.
// Lanes outside `valid` never match.
template <int RBITS>
__device__ __forceinline__ uint32_t match_digit(uint32_t d, uint32_t valid) {
  uint32_t peers = valid;
#pragma unroll
  for (int b = 0; b < RBITS; ++b) {
    // per bit: the bit as a predicate, its ballot, peers &= bit ? m : ~m.
    // Written this way ptxas moves all the digit's bits into predicates with
    // one R2P and needs ~3 instructions per bit (~5 from the C++ form):
    // configs[2] binning 0.230 -> 0.220 ms, configs[4] 3.67 -> 3.48 ms
    uint32_t r;
    asm("{\n\t.reg .pred p;\n\t.reg .b32 m, x;\n\t"
        "setp.ne.u32 p, %2, 0;\n\t"
        "vote.sync.ballot.b32 m, p, 0xffffffff;\n\t"
        "selp.b32 x, 0, 0xffffffff, p;\n\t"
        "xor.b32 m, m, x;\n\t"
        "and.b32 %0, %1, m;\n\t}"
        : "=r"(r)
        : "r"(peers), "r"(d & (1u << b)));
    peers = r;
  }
  return peers;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Histogram of `num_passes` RBITS-bit digits starting at begin_bit; hist is
// num_passes x 2^RBITS u32 and must be zeroed.  n = min(*n_ptr, n_cap).
template <typename K, int RBITS>
__global__ void __launch_bounds__(256) rs_histogram(const K* __restrict__ keys, const uint32_t* n_ptr, uint32_t n_cap,
                                                    int begin_bit, int num_passes, uint32_t* __restrict__ hist) {
  constexpr int R = 1 << RBITS;
  extern __shared__ uint32_t sh[];  // [num_passes][8 warps][R]
  constexpr int V = 16 / sizeof(K);
  const uint32_t n = min(*n_ptr, n_cap);
  const int w = threadIdx.x >> 5;
  for (int j = threadIdx.x; j < num_passes * 8 * R; j += 256) sh[j] = 0;
  __syncthreads();
  const uint32_t nvec = n / V;
  const uint4* kv = reinterpret_cast<const uint4*>(keys);
  for (uint32_t i = blockIdx.x * 256u + threadIdx.x; i < nvec; i += gridDim.x * 256u) {
    uint4 raw = kv[i];
    const K* ks = reinterpret_cast<const K*>(&raw);
#pragma unroll
    for (int v = 0; v < V; ++v)
      for (int p = 0; p < num_passes; ++p)
        atomicAdd(&sh[(p * 8 + w) * R + rs_digit<K, RBITS>(ks[v], begin_bit + RBITS * p)], 1u);
  }
  for (uint32_t i = nvec * V + blockIdx.x * 256u + threadIdx.x; i < n; i += gridDim.x * 256u) {
    K k = keys[i];
    for (int p = 0; p < num_passes; ++p)
      atomicAdd(&sh[(p * 8 + w) * R + rs_digit<K, RBITS>(k, begin_bit + RBITS * p)], 1u);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < num_passes * R; j += 256) {
    const int p = j / R, d = j % R;
    uint32_t v = 0;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) v += sh[(p * 8 + ww) * R + d];
    if (v) atomicAdd(&hist[j], v);
  }
}

template <typename K, int IPT, int RBITS, int NT = kRsThreads>
struct RsSmem {
  static constexpr int kTile = NT * IPT;
  static constexpr int R = 1 << RBITS;
  static constexpr int kWarps = NT / 32;
  uint32_t warp_hist[kWarps][R];
  uint32_t digit_start[R];
  uint32_t global_base[R];
  uint32_t pass_base[R];  // exclusive scan of the pass's digit counts
  uint32_t warp_tot[kWarps];
  uint32_t part;
  uint32_t vals[kTile];
  K keys[kTile];
};

struct RsRangeOut {
  uint2* ranges;   // per-cell [start, end), pre-set to (0xffffffff, 0); null = none
  int tile_shift;  // cell id = key >> tile_shift
};

// One pass.  pass_count: the pass's digit counts (every CTA scans them);
// status: nparts x 2^RBITS u32, zeroed; ticket zeroed.
// vin == nullptr means values are the item indices (first pass of an argsort).
// kout == nullptr skips the key writes.
// Two resident CTAs per SM (64 registers): one CTA's look-back and scatter
// overlap the other's loads and ranking, and the four view streams' rasters
// find room beside the sorts.  The 16-item depth sort spills 28 bytes at 64
// registers and is still faster in the four-stream headline (configs[2]
// 2036 -> 2070 frames/s with the 8-item cell sort; configs[4] 8.08 -> 7.91 ms).
#ifndef SGS_RS_MIN_BLOCKS
#define SGS_RS_MIN_BLOCKS(ipt) 2
#endif
template <typename K, int IPT, int RBITS, int NT = kRsThreads>
__global__ void __launch_bounds__(NT, SGS_RS_MIN_BLOCKS(IPT)) rs_onesweep(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                          K* __restrict__ kout, uint32_t* __restrict__ vout,
                                                          const uint32_t* n_ptr, uint32_t n_cap, int shift,
                                                          const uint32_t* __restrict__ pass_count, uint32_t* status,
                                                          uint32_t* ticket, RsRangeOut rout) {
  static_assert((1 << RBITS) <= NT, "one thread per digit");
  using S = RsSmem<K, IPT, RBITS, NT>;
  constexpr int kRsWarps = S::kWarps;
  constexpr int kTile = S::kTile;
  constexpr int R = S::R;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S& s = *reinterpret_cast<S*>(smem_raw);
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const uint32_t n = min(*n_ptr, n_cap);
  const uint32_t nparts = (n + kTile - 1) / kTile;
  const uint32_t lt = lanemask_lt();

  // each CTA scans the pass's digit counts itself (no separate scan kernel)
  {
    const uint32_t c = t < R ? pass_count[t] : 0u;
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s.warp_tot[w] = x;
    __syncthreads();
    uint32_t pre = 0;
    for (int i = 0; i < w; ++i) pre += s.warp_tot[i];
    if (t < R) s.pass_base[t] = pre + x - c;
    __syncthreads();
  }

  for (;;) {
    if (t == 0) s.part = atomicAdd(ticket, 1u);
    for (int j = t; j < kRsWarps * R; j += NT) (&s.warp_hist[0][0])[j] = 0;
    __syncthreads();
    const uint32_t part = s.part;
    if (part >= nparts) return;

    // ---- load keys + values (warp-striped), rank within the warp, order-preserving
    const uint32_t base = part * kTile + w * 32 * IPT;
    K keys[IPT];
    uint32_t vals[IPT];
    uint16_t rank[IPT];
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const uint32_t idx = base + i * 32 + lane;
      const bool valid = idx < n;
      keys[i] = valid ? kin[idx] : K(0);
      vals[i] = valid ? (vin ? vin[idx] : idx) : 0u;
    }
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const uint32_t idx = base + i * 32 + lane;
      const bool valid = idx < n;
      const uint32_t d = rs_digit<K, RBITS>(keys[i], shift);
      const uint32_t peers = match_digit<RBITS>(d, __ballot_sync(0xffffffffu, valid));
      const int leader = __ffs(peers) - 1;
      uint32_t old = 0;
      if (valid && lane == leader) old = atomicAdd(&s.warp_hist[w][d], (uint32_t)__popc(peers));
      old = __shfl_sync(0xffffffffu, old, valid ? leader : lane);
      rank[i] = (uint16_t)(old + __popc(peers & lt));
      // the leaders of successive items are different threads: order their
      // counter updates explicitly (stability depends on it)
      __syncwarp();
    }
    __syncthreads();

    // ---- per digit (threads 0..R-1): scan over warps, publish, look back
    uint32_t run = 0, wexcl = 0;
    if (t < R) {
#pragma unroll
      for (int ww = 0; ww < kRsWarps; ++ww) {
        const uint32_t c = s.warp_hist[ww][t];
        s.warp_hist[ww][t] = run;
        run += c;
      }
      atomicExch(status + (size_t)part * R + t, (part == 0 ? kFlagInc : kFlagAgg) | run);
      uint32_t x = run;  // block exclusive scan of the digit counts -> digit_start
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) s.warp_tot[w] = x;
      wexcl = x - run;
    }
    __syncthreads();
    if (t < R) {
      uint32_t pre = 0;
      for (int i = 0; i < w; ++i) pre += s.warp_tot[i];
      s.digit_start[t] = pre + wexcl;
      uint32_t excl = 0;
      if (part > 0) {
        // windowed decoupled look-back: kLookback predecessors are loaded at
        // once, summed from the nearest until the first inclusive prefix; a
        // not-yet-published predecessor restarts the window there.
        int64_t p = (int64_t)part - 1;
        for (;;) {
          uint32_t v[kLookback];
#pragma unroll
          for (int j = 0; j < kLookback; ++j)
            v[j] = (p - j >= 0) ? *reinterpret_cast<volatile uint32_t*>(status + (size_t)(p - j) * R + t)
                                : (uint32_t)kFlagInc;
          int used = 0;
          bool done = false;
#pragma unroll
          for (int j = 0; j < kLookback; ++j) {
            const uint32_t flag = v[j] & ~kCountMask;
            if (flag == 0) break;
            excl += v[j] & kCountMask;
            used = j + 1;
            if (flag == kFlagInc) {
              done = true;
              break;
            }
          }
          if (done) break;
          p -= used;
        }
        atomicExch(status + (size_t)part * R + t, kFlagInc | (excl + run));
      }
      s.global_base[t] = s.pass_base[t] + excl;
    }
    __syncthreads();

    // ---- scatter into shared memory in local sorted order
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const uint32_t idx = base + i * 32 + lane;
      if (idx < n) {
        const uint32_t d = rs_digit<K, RBITS>(keys[i], shift);
        const uint32_t pos = s.digit_start[d] + s.warp_hist[w][d] + rank[i];
        s.keys[pos] = keys[i];
        s.vals[pos] = vals[i];
      }
    }
    __syncthreads();
    const uint32_t cnt = min((uint32_t)kTile, n - part * kTile);
    for (uint32_t j = t; j < cnt; j += NT) {
      const K k = s.keys[j];
      const uint32_t d = rs_digit<K, RBITS>(k, shift);
      const uint32_t g = s.global_base[d] + j - s.digit_start[d];
      if (kout) kout[g] = k;
      vout[g] = s.vals[j];
      if (rout.ranges) {
        const uint32_t tile = (uint32_t)(k >> rout.tile_shift);
        if (j == 0 || (uint32_t)(s.keys[j - 1] >> rout.tile_shift) != tile) atomicMin(&rout.ranges[tile].x, g);
        if (j + 1 == cnt || (uint32_t)(s.keys[j + 1] >> rout.tile_shift) != tile)
          atomicMax(&rout.ranges[tile].y, g + 1);
      }
    }
    __syncthreads();
  }
}

int resident_ctas_per_sm(const void* kernel, int threads, size_t smem);
int device_sm_count();

template <typename K, int IPT, int NT = kRsThreads>
inline uint64_t rs_parts(uint64_t n) {
  return (n + NT * IPT - 1) / (NT * IPT);
}

// Sort `n_cap`-bounded pairs (count in *n_ptr on the device) over key bits
// [begin_bit, begin_bit + bits) in ceil(bits / RBITS) passes; lower bits
// travel with the key unsorted.  Ping-pongs between (k0, v0) and (k1, v1);
// *result_in_alt says whether the result is in (k1, v1).  iota_values: the
// input values are the item indices (v0 is not read).  With `rout.ranges`,
// the last pass also writes the cell ranges (and skips its key writes unless
// keep_last_keys).  hist: 16*512 u32; status: parts*512*passes u32; tickets:
// >= passes u32; all zeroed here (hist only when !hist_ready).
template <typename K, int IPT, int RBITS, int NT = kRsThreads>
int radix_sort_pairs(K* k0, uint32_t* v0, K* k1, uint32_t* v1, const uint32_t* n_ptr, uint32_t n_cap, int bits,
                     uint32_t* hist, uint32_t* status, uint32_t* tickets, bool* result_in_alt, cudaStream_t st,
                     bool iota_values = false, RsRangeOut rout = RsRangeOut{nullptr, 0}, int begin_bit = 0,
                     bool keep_last_keys = false, bool hist_ready = false, const K* k_first = nullptr,
                     const uint32_t* v_first = nullptr) {
  constexpr int R = 1 << RBITS;
  const int passes = (bits + RBITS - 1) / RBITS;
  const uint64_t parts = rs_parts<K, IPT, NT>(n_cap);
  *result_in_alt = false;
  if (n_cap == 0 || passes == 0) return SGS_OK;
  // hist_ready: the producer kernel already accumulated every pass's digit
  // counts into the (zeroed) hist; only the exclusive scan remains
  if (!hist_ready) SGS_CUDA(cudaMemsetAsync(hist, 0, (size_t)passes * R * 4, st));
  SGS_CUDA(cudaMemsetAsync(status, 0, (size_t)parts * R * 4 * passes, st));
  SGS_CUDA(cudaMemsetAsync(tickets, 0, (size_t)passes * 4, st));
  const int sms = device_sm_count();
  constexpr int V = 16 / sizeof(K);
  int hgrid = (int)std::min<uint64_t>((n_cap / V + 256 * 8 - 1) / (256 * 8), (uint64_t)sms * 4);
  if (hgrid < 1) hgrid = 1;
  const size_t hsmem = (size_t)passes * 8 * R * 4;
  static bool hattr = false;
  if (!hattr) {
    SGS_CUDA(cudaFuncSetAttribute(rs_histogram<K, RBITS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    hattr = true;
  }
  if (!hist_ready) {
    rs_histogram<K, RBITS><<<hgrid, 256, hsmem, st>>>(k_first ? k_first : k0, n_ptr, n_cap, begin_bit, passes, hist);
    SGS_LAUNCH_CHECK("rs_histogram");
  }
  const size_t smem = sizeof(RsSmem<K, IPT, RBITS, NT>);
  static bool attr_set = false;
  if (!attr_set) {
    SGS_CUDA(cudaFuncSetAttribute(rs_onesweep<K, IPT, RBITS, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    attr_set = true;
  }
  static int per_sm = 0;
  if (!per_sm) per_sm = resident_ctas_per_sm((const void*)rs_onesweep<K, IPT, RBITS, NT>, NT, smem);
  if (per_sm < 1) {
    set_error("onesweep kernel cannot be resident");
    return SGS_E_CUDA;
  }
  const int grid = (int)std::min<uint64_t>(parts, (uint64_t)sms * per_sm);
  // k_first / v_first: input keys / values of the first pass (read only);
  // the passes then ping-pong between k1 and k0 as if the first had read k0
  K* ka = k0;
  K* kb = k1;
  uint32_t* va = v0;
  uint32_t* vb = v1;
  for (int p = 0; p < passes; ++p) {
    const bool last = p + 1 == passes;
    rs_onesweep<K, IPT, RBITS, NT><<<grid, NT, smem, st>>>(
        (p == 0 && k_first) ? k_first : ka,
        (p == 0 && iota_values) ? nullptr : ((p == 0 && v_first) ? v_first : va),
        (last && rout.ranges && !keep_last_keys) ? nullptr : kb, vb,
        n_ptr, n_cap, begin_bit + RBITS * p, hist + R * p, status + (size_t)parts * R * p, tickets + p,
        last ? rout : RsRangeOut{nullptr, 0});
    SGS_LAUNCH_CHECK("rs_onesweep");
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  *result_in_alt = (passes & 1) != 0;
  return SGS_OK;
}

}  // namespace sgs
