// compact.cu -- MEGS2 compact scene files straight into the device SoA
// (/root/reference/pkg/src/sgsplat/io.py:1-15 format, 173-214 read_compact).
//
// Layout (little-endian): magic "MEGS2\0", u16 version (1), u32 count, then
// per primitive 14 f32 (position 3, quaternion 4, scale 3, opacity,
// diffuse 3), a u8 lobe count and per lobe 7 f32 (axis 3, sharpness,
// amplitude 3).  Records are variable-length, so their offsets form a chain:
// the host walks it once (one byte read per record, with the reference's
// truncation / trailing-byte checks), and one GPU thread per primitive then
// decodes its record from the uploaded bytes into the renderer's SoA -- the
// same arrays SceneParams.from_scene builds (render.py:135-145): log_scale =
// log(scale) rounded from float64, missing lobe slots axis (0, 0, 1), zero
// sharpness / amplitude and lobe_mask 0.
#include <string.h>

#include "common.cuh"

namespace sgs {

constexpr uint64_t kCompactHeader = 12;  // magic 6 + version 2 + count 4
constexpr uint64_t kBaseBytes = 14 * 4 + 1;
constexpr uint64_t kLobeBytes = 7 * 4;
static const unsigned char kMagic[6] = {'M', 'E', 'G', 'S', '2', 0};

int compact_header(const uint8_t* data, uint64_t size, int64_t* count) {
  if (!data || !count) {
    set_error("null argument");
    return SGS_E_ARG;
  }
  if (size < kCompactHeader) {
    set_error("header incomplete (offset %llu)", (unsigned long long)size);
    return SGS_E_TRUNCATED;
  }
  if (memcmp(data, kMagic, 6) != 0) {
    set_error("bad magic");
    return SGS_E_FORMAT;
  }
  const uint16_t version = (uint16_t)(data[6] | (data[7] << 8));
  if (version != 1) {
    set_error("unsupported format version %u", (unsigned)version);
    return SGS_E_FORMAT;
  }
  *count = (int64_t)((uint32_t)data[8] | ((uint32_t)data[9] << 8) | ((uint32_t)data[10] << 16) |
                     ((uint32_t)data[11] << 24));
  return SGS_OK;
}

int compact_index(const uint8_t* data, uint64_t size, uint64_t* offsets, int64_t cap, int32_t* max_lobes) {
  int64_t n = 0;
  int rc = compact_header(data, size, &n);
  if (rc) return rc;
  if (!offsets || cap < n + 1 || !max_lobes) {
    set_error("offset table needs count + 1 = %lld entries", (long long)(n + 1));
    return SGS_E_ARG;
  }
  uint64_t pos = kCompactHeader;
  int ml = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (size < pos + kBaseBytes) {
      set_error("primitive record ends early (offset %llu)", (unsigned long long)size);
      return SGS_E_TRUNCATED;
    }
    offsets[i] = pos;
    const int nl = data[pos + kBaseBytes - 1];
    pos += kBaseBytes + (uint64_t)nl * kLobeBytes;
    if (size < pos) {
      set_error("lobe records end early (offset %llu)", (unsigned long long)size);
      return SGS_E_TRUNCATED;
    }
    ml = nl > ml ? nl : ml;
  }
  if (pos != size) {
    set_error("%llu trailing bytes after last primitive", (unsigned long long)(size - pos));
    return SGS_E_FORMAT;
  }
  offsets[n] = pos;
  *max_lobes = ml;
  return SGS_OK;
}

__device__ __forceinline__ float ld_f32(const uint8_t* p) {
  const uint32_t u = (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
  return __uint_as_float(u);
}

__global__ void __launch_bounds__(256) compact_decode_kernel(const uint8_t* __restrict__ data,
                                                             const uint64_t* __restrict__ offsets, int64_t n, int L,
                                                             sgs_scene_soa out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t* r = data + offsets[i];
    for (int k = 0; k < 3; ++k) out.position[3 * i + k] = ld_f32(r + 4 * k);
    for (int k = 0; k < 4; ++k) out.quat[4 * i + k] = ld_f32(r + 12 + 4 * k);
    for (int k = 0; k < 3; ++k) out.log_scale[3 * i + k] = (float)log((double)ld_f32(r + 28 + 4 * k));
    out.opacity[i] = ld_f32(r + 40);
    for (int k = 0; k < 3; ++k) out.diffuse[3 * i + k] = ld_f32(r + 44 + 4 * k);
    const int nl = r[56];
    const uint8_t* lr = r + 57;
    for (int l = 0; l < L; ++l) {
      const size_t j = (size_t)i * L + l;
      const bool has = l < nl;
      for (int k = 0; k < 3; ++k) out.axis_raw[3 * j + k] = has ? ld_f32(lr + 28 * l + 4 * k) : (k == 2 ? 1.0f : 0.0f);
      out.sharpness[j] = has ? ld_f32(lr + 28 * l + 12) : 0.0f;
      for (int k = 0; k < 3; ++k) out.amplitude[3 * j + k] = has ? ld_f32(lr + 28 * l + 16 + 4 * k) : 0.0f;
      out.lobe_mask[j] = has ? 1.0f : 0.0f;
    }
  }
}

int launch_compact_decode(const uint8_t* data, const uint64_t* offsets, int64_t n, int L, const sgs_scene_soa* out,
                          cudaStream_t st) {
  if (n == 0) return SGS_OK;
  const int grid = persistent_grid((uint64_t)n, 256, 8);
  compact_decode_kernel<<<grid, 256, 0, st>>>(data, offsets, n, L, *out);
  SGS_LAUNCH_CHECK("compact_decode_kernel");
  return SGS_OK;
}

}  // namespace sgs
