// select.cu -- top-k keep masks for the ADMM proximal projection
// (/root/reference/pkg/src/sgsplat/prune.py:204-213, _top_k_mask):
// keep[i] = 1 for the k largest scores, ties keeping the lower index.
//
// Scores are float64.  Each becomes a 64-bit key that sorts ascending in
// order of DEcreasing score (IEEE order-preserving bit transform, inverted;
// -0.0 canonicalised to +0.0 so it ties with +0.0 as in numpy), the indices
// ride along as values, and the stable onesweep radix sort (sort.cuh) puts
// equal scores in index order -- exactly np.argsort(-scores, kind="stable").
// The first k values are then marked.
#include "common.cuh"

namespace sgs {

__global__ void topk_keys_kernel(const double* __restrict__ scores, uint32_t n, unsigned long long* __restrict__ keys,
                                 uint32_t* __restrict__ vals) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double s = scores[i];
    if (s == 0.0) s = 0.0;  // -0.0 ties with +0.0
    const unsigned long long u = (unsigned long long)__double_as_longlong(s);
    const unsigned long long asc = (u >> 63) ? ~u : (u | 0x8000000000000000ull);
    keys[i] = ~asc;
    vals[i] = i;
  }
}

__global__ void topk_mark_kernel(const uint32_t* __restrict__ vals, uint32_t n, uint32_t k,
                                 uint8_t* __restrict__ keep) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    keep[vals[i]] = i < k ? 1 : 0;
}

uint64_t sort_u64_temp_bytes(uint64_t n, int bits);
int launch_sort_u64(unsigned long long* keys, uint32_t* vals, uint32_t n, int bits, void* temp, uint64_t temp_bytes,
                    cudaStream_t st);

uint64_t topk_temp_bytes(uint64_t n) { return align256(n * 8) + align256(n * 4) + sort_u64_temp_bytes(n, 64); }

int launch_topk_mask(const double* scores, uint32_t n, uint32_t k, uint8_t* keep, void* temp, uint64_t temp_bytes,
                     cudaStream_t st) {
  if (temp_bytes < topk_temp_bytes(n)) {
    set_error("top-k temp too small: need %llu bytes", (unsigned long long)topk_temp_bytes(n));
    return SGS_E_WORKSPACE;
  }
  char* p = reinterpret_cast<char*>(temp);
  auto* keys = reinterpret_cast<unsigned long long*>(p);
  p += align256((uint64_t)n * 8);
  auto* vals = reinterpret_cast<uint32_t*>(p);
  p += align256((uint64_t)n * 4);
  const int grid = persistent_grid(n, 256, 8);
  topk_keys_kernel<<<grid, 256, 0, st>>>(scores, n, keys, vals);
  SGS_LAUNCH_CHECK("topk_keys_kernel");
  int rc = launch_sort_u64(keys, vals, n, 64, p, sort_u64_temp_bytes(n, 64), st);
  if (rc) return rc;
  topk_mark_kernel<<<grid, 256, 0, st>>>(vals, n, k, keep);
  SGS_LAUNCH_CHECK("topk_mark_kernel");
  return SGS_OK;
}

}  // namespace sgs
