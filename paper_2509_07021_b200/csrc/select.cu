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

// ------------------------------------------------------------ ADMM update
// One fused pass per stage of the penalized descent step (prune.py:162-201),
// every parameter class of a primitive in one thread, no host round trip:
//   stage 1 (delta != 0, after g1):  o -= eta r_o (g1_o + d_o (o - z_o + u_o)),  o = clip(o, 0, 1)
//   stage 2 (after g2, or after g1 when delta == 0):
//     s -= eta r_s (g_s + d_s (s - z_s + u_s))     (g_s = g2_s, or g1_s with d_s = 0)
//     o -= eta r_o g1_o                            (delta == 0 only: update_o)
//     f -= eta r_f g1_f                            (position, quat, log_scale, diffuse, axis_raw, amplitude)
//     o = clip(o, 0, 1),  s = max(s, 0)
// `ok` (device bool, may be null): 0 leaves every value unchanged (a
// non-finite gradient was seen, admm._Failure).  Arithmetic in float32 in
// the reference's operation order.
__global__ void __launch_bounds__(256) admm_update_kernel(int64_t n, int L, int stage, int update_o, sgs_admm_fields F,
                                                          sgs_admm_fields G, const float* __restrict__ gs,
                                                          const float* __restrict__ zo, const float* __restrict__ uo,
                                                          const float* __restrict__ zs, const float* __restrict__ us,
                                                          sgs_admm_rates R, const uint8_t* __restrict__ ok) {
  if (ok && !*ok) return;
  const float eta = R.eta;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (stage == 1) {
      float o = F.opacity[i];
      o = o - eta * R.opacity * (G.opacity[i] + R.delta_o * ((o - zo[i]) + uo[i]));
      F.opacity[i] = fminf(fmaxf(o, 0.0f), 1.0f);
      continue;
    }
    for (int l = 0; l < L; ++l) {
      const int64_t j = i * L + l;
      float s = F.sharpness[j];
      const float pen = R.delta_s != 0.0f ? R.delta_s * ((s - zs[j]) + us[j]) : 0.0f;
      s = s - eta * R.sharpness * (gs[j] + pen);
      F.sharpness[j] = fmaxf(s, 0.0f);
    }
    float o = F.opacity[i];
    if (update_o) o = o - eta * R.opacity * G.opacity[i];
    F.opacity[i] = fminf(fmaxf(o, 0.0f), 1.0f);
#define SGS_ADMM_SUB(FIELD, W)                                                   \
  for (int k = 0; k < (W); ++k) {                                                \
    const int64_t j = i * (W) + k;                                               \
    F.FIELD[j] = F.FIELD[j] - eta * R.FIELD * G.FIELD[j];                        \
  }
    SGS_ADMM_SUB(position, 3)
    SGS_ADMM_SUB(quat, 4)
    SGS_ADMM_SUB(log_scale, 3)
    SGS_ADMM_SUB(diffuse, 3)
    SGS_ADMM_SUB(axis_raw, 3 * L)
    SGS_ADMM_SUB(amplitude, 3 * L)
#undef SGS_ADMM_SUB
  }
}

int launch_admm_update(int64_t n, int L, int stage, int update_o, const sgs_admm_fields& F, const sgs_admm_fields& G,
                       const float* gs, const float* zo, const float* uo, const float* zs, const float* us,
                       const sgs_admm_rates& R, const uint8_t* ok, cudaStream_t st) {
  if (n <= 0) return SGS_OK;
  admm_update_kernel<<<persistent_grid((uint64_t)n, 256, 8), 256, 0, st>>>(n, L, stage, update_o, F, G, gs, zo, uo, zs,
                                                                         us, R, ok);
  SGS_LAUNCH_CHECK("admm_update_kernel");
  return SGS_OK;
}

}  // namespace sgs
