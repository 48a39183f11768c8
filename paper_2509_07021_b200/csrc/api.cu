// api.cu -- extern "C" entry points of libsgs.so (declared in include/sgs.h).
// Validation, workspace carving and kernel sequencing; no math here.
#include <stdarg.h>

#include <mutex>

#include "common.cuh"

namespace sgs {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_fail(cudaError_t e, const char* what) {
  set_error("CUDA error in %s: %s", what, cudaGetErrorString(e));
  return SGS_E_CUDA;
}

int device_sm_count() {
  static int cached = 0;
  if (!cached) {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = kNumSMs;
    cached = v;
  }
  return cached;
}

int resident_ctas_per_sm(const void* kernel, int threads, size_t smem) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem) != cudaSuccess) return 0;
  return n;
}

int launch_preprocess(const sgs_params& P, const SgsCam& cam, const sgs_workspace* ws, const Layout& lo,
                      cudaStream_t st);
int launch_project_records(const sgs_params& P, const SgsCam& cam, float* out, cudaStream_t st);
int launch_vram3s(const sgs_params& P, const SgsCam& cam, int tile_px, Counters* ctr, cudaStream_t st);
int launch_bin(const SgsCam& cam, const sgs_workspace* ws, const Layout& lo, cudaStream_t st);
bool final_in_alt(const Layout& lo);
int launch_raster_fwd(const SgsCam& cam, float3 bg, const sgs_workspace* ws, const Layout& lo, const uint32_t* vals,
                      float* img, float* T, uint32_t* nc, unsigned long long* weight_fx, unsigned long long* pairs,
                      cudaStream_t st);
int launch_raster_bwd(const SgsCam& cam, float3 bg, const sgs_workspace* ws, const Layout& lo, const uint32_t* vals,
                      const float* T, const uint32_t* nc, const float* dimg, float* grad2d, void* det_scratch,
                      cudaStream_t st);
uint64_t raster_bwd_det_scratch_bytes(int64_t n);
int launch_fixed_to_float(const unsigned long long* fx, int64_t n, int frac_bits, float* out, int acc, cudaStream_t st);
int launch_preprocess_bwd_views(const sgs_params& P, const SgsCam* cams, const float* const* grad2d, int n_views,
                                const sgs_grads& g, cudaStream_t st);
int launch_preprocess_bwd(const sgs_params& P, const SgsCam& cam, const float* grad2d, const sgs_grads& g,
                          cudaStream_t st);
int launch_export_lists(const SgsCam& cam, const sgs_workspace* ws, const Layout& lo, const uint32_t* vals,
                        unsigned long long* keys, uint32_t* out_vals, uint32_t* ranges, cudaStream_t st);
int launch_sort_u64(unsigned long long* keys, uint32_t* vals, uint32_t n, int bits, void* temp, uint64_t temp_bytes,
                    cudaStream_t st);
uint64_t sort_u64_temp_bytes(uint64_t n, int bits);

static int check_params(const sgs_params* p, const Layout* lo) {
  if (!p || p->n < 0 || p->n_lobes < 0 || p->n_lobes > SGS_MAX_LOBES) {
    set_error("invalid params");
    return SGS_E_ARG;
  }
  if (p->n > 0 && (!p->position || !p->quat || !p->log_scale || !p->opacity || !p->diffuse ||
                   (p->n_lobes > 0 && (!p->axis_raw || !p->sharpness || !p->amplitude || !p->lobe_mask)))) {
    set_error("null parameter array");
    return SGS_E_ARG;
  }
  if (lo && (p->n != lo->n || p->n_lobes != lo->L)) {
    set_error("params (n=%lld, L=%d) do not match workspace (n=%lld, L=%d)", (long long)p->n, p->n_lobes,
              (long long)lo->n, lo->L);
    return SGS_E_ARG;
  }
  return SGS_OK;
}

static const uint32_t* final_vals(const sgs_workspace* ws, const Layout& lo) {
  return at<uint32_t>(ws, final_in_alt(lo) ? lo.ent_val_alt : lo.ent_val);
}

uint64_t loss_workspace_bytes(int H, int W);
int launch_image_loss(const void* img, int img_f64, const void* tgt, int tgt_f64, int H, int W,
                      const sgs_loss_config* cfg, float* dimg, double* dimg64, double* smap, double* out,
                      void* workspace, uint64_t ws_bytes, cudaStream_t st);

uint64_t topk_temp_bytes(uint64_t n);
int launch_topk_mask(const double* scores, uint32_t n, uint32_t k, uint8_t* keep, void* temp, uint64_t temp_bytes,
                     cudaStream_t st);

int compact_header(const uint8_t* data, uint64_t size, int64_t* count);
int compact_index(const uint8_t* data, uint64_t size, uint64_t* offsets, int64_t cap, int32_t* max_lobes);
int launch_compact_decode(const uint8_t* data, const uint64_t* offsets, int64_t n, int L, const sgs_scene_soa* out,
                          cudaStream_t st);

int launch_admm_update(int64_t n, int L, int stage, int update_o, const sgs_admm_fields& F, const sgs_admm_fields& G,
                       const float* gs, const float* zo, const float* uo, const float* zs, const float* us,
                       const sgs_admm_rates& R, const uint8_t* ok, cudaStream_t st);

}  // namespace sgs

using namespace sgs;

extern "C" {

int32_t sgs_version(void) { return 200; }

int sgs_admm_update(int64_t n, int32_t n_lobes, int32_t stage, int32_t update_o, const sgs_admm_fields* params,
                    const sgs_admm_fields* g1, const float* g_sharpness, const float* z_o, const float* u_o,
                    const float* z_s, const float* u_s, const sgs_admm_rates* rates, const uint8_t* ok,
                    void* stream) {
  if (n < 0 || n_lobes < 0 || n_lobes > SGS_MAX_LOBES || !params || !g1 || !rates || (stage != 1 && stage != 2)) {
    set_error("invalid ADMM update arguments");
    return SGS_E_ARG;
  }
  if (n > 0 && (!params->opacity || !g1->opacity || (stage == 1 && (!z_o || !u_o)) ||
                (stage == 2 && (!params->position || !params->quat || !params->log_scale || !params->diffuse ||
                                !g1->position || !g1->quat || !g1->log_scale || !g1->diffuse ||
                                (n_lobes > 0 && (!params->axis_raw || !params->sharpness || !params->amplitude ||
                                                 !g1->axis_raw || !g1->amplitude || !g_sharpness ||
                                                 (rates->delta_s != 0.0f && (!z_s || !u_s)))))))) {
    set_error("null ADMM buffer");
    return SGS_E_ARG;
  }
  return sgs::launch_admm_update(n, n_lobes, stage, update_o, *params, *g1, g_sharpness, z_o, u_o, z_s, u_s, *rates,
                                 ok, as_stream(stream));
}

int sgs_abi_sizes(uint64_t out[4]) {
  if (!out) return SGS_E_ARG;
  out[0] = sizeof(sgs_camera);
  out[1] = sizeof(sgs_params);
  out[2] = sizeof(sgs_workspace);
  out[3] = sizeof(sgs_stats);
  return SGS_OK;
}

const char* sgs_last_error(void) { return g_err; }

int sgs_workspace_size(const sgs_workspace* ws, uint64_t* bytes_out) {
  Layout lo;
  int rc = make_layout(ws, &lo);
  if (rc) return rc;
  if (!bytes_out) return SGS_E_ARG;
  *bytes_out = lo.total;
  return SGS_OK;
}

int sgs_preprocess(const sgs_params* params, const sgs_camera* cam, const sgs_workspace* ws, void* stream) {
  Layout lo;
  SgsCam c;
  int rc = check_ws(ws, &lo);
  if (!rc) rc = check_params(params, &lo);
  if (!rc) rc = make_cam(cam, lo, &c);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  SGS_CUDA(cudaMemsetAsync(at<Counters>(ws, lo.counters), 0, sizeof(Counters), st));
  // the depth-digit histograms the preprocess accumulates (both sort modes)
  SGS_CUDA(cudaMemsetAsync(at<uint32_t>(ws, lo.hist) + kDepthHistOff, 0, (size_t)4 * 256 * 4, st));
  if (lo.n == 0) return SGS_OK;
  return launch_preprocess(*params, c, ws, lo, st);
}

int sgs_bin(const sgs_camera* cam, const sgs_workspace* ws, void* stream) {
  Layout lo;
  SgsCam c;
  int rc = check_ws(ws, &lo);
  if (!rc) rc = make_cam(cam, lo, &c);
  if (rc) return rc;
  return launch_bin(c, ws, lo, as_stream(stream));
}

int sgs_raster_forward(const sgs_camera* cam, const float background[3], const sgs_workspace* ws, float* out_img,
                       float* out_T, uint32_t* out_ncontrib, uint64_t* weight_sums_fx, uint64_t* pair_count,
                       void* stream) {
  Layout lo;
  SgsCam c;
  int rc = check_ws(ws, &lo);
  if (!rc) rc = make_cam(cam, lo, &c);
  if (rc) return rc;
  if (!out_img || !background) {
    set_error("null output buffer");
    return SGS_E_ARG;
  }
  float3 bg = make_float3(background[0], background[1], background[2]);
  return launch_raster_fwd(c, bg, ws, lo, final_vals(ws, lo), out_img, out_T, out_ncontrib,
                           reinterpret_cast<unsigned long long*>(weight_sums_fx),
                           reinterpret_cast<unsigned long long*>(pair_count), as_stream(stream));
}

int sgs_render_forward(const sgs_params* params, const sgs_camera* cam, const float background[3],
                       const sgs_workspace* ws, float* out_img, float* out_T, uint32_t* out_ncontrib,
                       uint64_t* weight_sums_fx, uint64_t* pair_count, void* stream) {
  int rc = sgs_preprocess(params, cam, ws, stream);
  if (!rc) rc = sgs_bin(cam, ws, stream);
  if (!rc)
    rc = sgs_raster_forward(cam, background, ws, out_img, out_T, out_ncontrib, weight_sums_fx, pair_count, stream);
  return rc;
}

int sgs_raster_backward(const sgs_camera* cam, const float background[3], const sgs_workspace* ws, const float* img,
                        const float* final_T, const uint32_t* ncontrib, const float* dimg, float* grad2d,
                        void* stream) {
  Layout lo;
  SgsCam c;
  int rc = check_ws(ws, &lo);
  if (!rc) rc = make_cam(cam, lo, &c);
  if (rc) return rc;
  if (!final_T || !ncontrib || !dimg || !grad2d || !background) {
    set_error("null buffer");
    return SGS_E_ARG;
  }
  (void)img;
  float3 bg = make_float3(background[0], background[1], background[2]);
  return launch_raster_bwd(c, bg, ws, lo, final_vals(ws, lo), final_T, ncontrib, dimg, grad2d, nullptr,
                           as_stream(stream));
}

uint64_t sgs_raster_backward_det_scratch_bytes(int64_t n) { return raster_bwd_det_scratch_bytes(n); }

int sgs_raster_backward_det(const sgs_camera* cam, const float background[3], const sgs_workspace* ws,
                            const float* img, const float* final_T, const uint32_t* ncontrib, const float* dimg,
                            float* grad2d, void* scratch, uint64_t scratch_bytes, void* stream) {
  Layout lo;
  SgsCam c;
  int rc = check_ws(ws, &lo);
  if (!rc) rc = make_cam(cam, lo, &c);
  if (rc) return rc;
  if (!final_T || !ncontrib || !dimg || !grad2d || !background || !scratch) {
    set_error("null buffer");
    return SGS_E_ARG;
  }
  if (scratch_bytes < raster_bwd_det_scratch_bytes(lo.n)) {
    set_error("deterministic backward scratch too small: need %llu bytes",
              (unsigned long long)raster_bwd_det_scratch_bytes(lo.n));
    return SGS_E_WORKSPACE;
  }
  (void)img;
  float3 bg = make_float3(background[0], background[1], background[2]);
  return launch_raster_bwd(c, bg, ws, lo, final_vals(ws, lo), final_T, ncontrib, dimg, grad2d, scratch,
                           as_stream(stream));
}

int sgs_fixed_to_float(const uint64_t* fx, int64_t n, int32_t frac_bits, float* out, int32_t accumulate,
                       void* stream) {
  if (n < 0 || (n > 0 && (!fx || !out)) || frac_bits < 0 || frac_bits > 62) {
    set_error("invalid fixed-point conversion arguments");
    return SGS_E_ARG;
  }
  return launch_fixed_to_float(reinterpret_cast<const unsigned long long*>(fx), n, frac_bits, out, accumulate,
                               as_stream(stream));
}

static int sgs_preprocess_backward_check(const sgs_params* params, const sgs_camera* cam, const float* grad2d,
                                         sgs_grads* grads) {
  int rc = check_params(params, nullptr);
  if (rc) return rc;
  if (!grads || !grad2d || (params->n > 0 && (!grads->position || !grads->quat || !grads->log_scale ||
                                              !grads->opacity || !grads->diffuse ||
                                              (params->n_lobes > 0 &&
                                               (!grads->axis_raw || !grads->sharpness || !grads->amplitude))))) {
    set_error("null gradient buffer");
    return SGS_E_ARG;
  }
  if ((grads->flags & ~(SGS_GRADS_ACCUMULATE | SGS_GRADS_MASK_LOGIT)) != 0 ||
      (reinterpret_cast<uintptr_t>(grads->quat) & 15u) != 0) {
    set_error("invalid gradient flags or unaligned quaternion gradient (16-byte rows)");
    return SGS_E_ARG;
  }
  if (!cam) {
    set_error("null camera");
    return SGS_E_ARG;
  }
  return SGS_OK;
}

int sgs_preprocess_backward(const sgs_params* params, const sgs_camera* cam, const float* grad2d, sgs_grads* grads,
                            void* stream) {
  int rc = check_params(params, nullptr);
  if (rc) return rc;
  if (!grads || !grad2d || (params->n > 0 && (!grads->position || !grads->quat || !grads->log_scale ||
                                              !grads->opacity || !grads->diffuse ||
                                              (params->n_lobes > 0 &&
                                               (!grads->axis_raw || !grads->sharpness || !grads->amplitude))))) {
    set_error("null gradient buffer");
    return SGS_E_ARG;
  }
  if ((grads->flags & ~(SGS_GRADS_ACCUMULATE | SGS_GRADS_MASK_LOGIT)) != 0 ||
      (reinterpret_cast<uintptr_t>(grads->quat) & 15u) != 0) {
    set_error("invalid gradient flags or unaligned quaternion gradient (16-byte rows)");
    return SGS_E_ARG;
  }
  Layout lo{};
  lo.W = cam ? cam->width : 0;
  lo.H = cam ? cam->height : 0;
  lo.tiles_x = (lo.W + SGS_TILE - 1) / SGS_TILE;
  lo.tiles_y = (lo.H + SGS_TILE - 1) / SGS_TILE;
  SgsCam c;
  rc = make_cam(cam, lo, &c);
  if (rc) return rc;
  if (params->n == 0) return SGS_OK;
  return launch_preprocess_bwd(*params, c, grad2d, *grads, as_stream(stream));
}


int sgs_preprocess_backward_views(const sgs_params* params, const sgs_camera* cams, int n_views,
                                  const float* const* grad2d, sgs_grads* grads, void* stream) {
  if (n_views < 1 || !cams || !grad2d) {
    set_error("need at least one view with its camera and partials");
    return SGS_E_ARG;
  }
  for (int v = 0; v < n_views; ++v)
    if (!grad2d[v]) {
      set_error("null partials for view %d", v);
      return SGS_E_ARG;
    }
  // validate like sgs_preprocess_backward (view 0), then convert every camera
  int rc = sgs_preprocess_backward_check(params, &cams[0], grad2d[0], grads);
  if (rc) return rc;
  if (params->n == 0) return SGS_OK;
  SgsCam c[64];
  for (int v0 = 0; v0 < n_views; v0 += 64) {
    const int nv = n_views - v0 < 64 ? n_views - v0 : 64;
    for (int k = 0; k < nv; ++k) {
      Layout lo{};
      lo.W = cams[v0 + k].width;
      lo.H = cams[v0 + k].height;
      lo.tiles_x = (lo.W + SGS_TILE - 1) / SGS_TILE;
      lo.tiles_y = (lo.H + SGS_TILE - 1) / SGS_TILE;
      rc = make_cam(&cams[v0 + k], lo, &c[k]);
      if (rc) return rc;
    }
    sgs_grads g = *grads;
    if (v0 > 0) g.flags |= SGS_GRADS_ACCUMULATE;
    rc = launch_preprocess_bwd_views(*params, c, grad2d + v0, nv, g, as_stream(stream));
    if (rc) return rc;
  }
  return SGS_OK;
}

int sgs_project_records(const sgs_params* params, const sgs_camera* cam, float* out, void* stream) {
  int rc = check_params(params, nullptr);
  if (rc) return rc;
  if (!out && params->n > 0) {
    set_error("null output");
    return SGS_E_ARG;
  }
  Layout lo{};
  lo.W = cam ? cam->width : 0;
  lo.H = cam ? cam->height : 0;
  lo.tiles_x = (lo.W + SGS_TILE - 1) / SGS_TILE;
  lo.tiles_y = (lo.H + SGS_TILE - 1) / SGS_TILE;
  SgsCam c;
  rc = make_cam(cam, lo, &c);
  if (rc) return rc;
  if (params->n == 0) return SGS_OK;
  return launch_project_records(*params, c, out, as_stream(stream));
}

int sgs_get_stats(const sgs_workspace* ws, sgs_stats* out, void* stream) {
  Layout lo;
  int rc = check_ws(ws, &lo);
  if (rc) return rc;
  if (!out) return SGS_E_ARG;
  Counters h;
  cudaStream_t st = as_stream(stream);
  SGS_CUDA(cudaMemcpyAsync(&h, at<Counters>(ws, lo.counters), sizeof(Counters), cudaMemcpyDeviceToHost, st));
  SGS_CUDA(cudaStreamSynchronize(st));
  out->n_visible = h.n_visible;
  out->n_emitting = h.n_emitting;
  out->n_entries = h.n_entries;
  out->capacity = (uint64_t)lo.cap;
  out->overflow = h.n_bin > (unsigned long long)lo.cap ? 1 : 0;
  out->n_bin_entries = h.n_bin;
  out->vram3s_visible = h.vram3s_visible;
  out->vram3s_entries = h.vram3s_entries;
  return SGS_OK;
}

int sgs_vram_model(const sgs_params* params, const sgs_camera* cam, int32_t tile_px, const sgs_workspace* ws,
                   void* stream) {
  Layout lo;
  SgsCam c;
  int rc = check_ws(ws, &lo);
  if (!rc) rc = check_params(params, &lo);
  if (!rc) rc = make_cam(cam, lo, &c);
  if (rc) return rc;
  if (tile_px < 1) {
    set_error("tile_px must be >= 1");
    return SGS_E_ARG;
  }
  cudaStream_t st = as_stream(stream);
  Counters* ctr = at<Counters>(ws, lo.counters);
  SGS_CUDA(cudaMemsetAsync(&ctr->vram3s_visible, 0, 16, st));
  if (lo.n == 0) return SGS_OK;
  return launch_vram3s(*params, c, tile_px, ctr, st);
}

int sgs_export_bins(const sgs_workspace* ws, const sgs_camera* cam, uint64_t* keys, uint32_t* values,
                    uint32_t* ranges, void* stream) {
  Layout lo;
  SgsCam c;
  int rc = check_ws(ws, &lo);
  if (!rc) rc = make_cam(cam, lo, &c);
  if (rc) return rc;
  if (!keys || !values || !ranges) {
    set_error("export needs keys, values and ranges buffers");
    return SGS_E_ARG;
  }
  return launch_export_lists(c, ws, lo, final_vals(ws, lo), reinterpret_cast<unsigned long long*>(keys), values,
                             ranges, as_stream(stream));
}

int sgs_export_projected(const sgs_workspace* ws, uint32_t* depth_bits, uint32_t* rect, uint32_t* tiles_touched,
                         float* records, void* stream) {
  Layout lo;
  int rc = check_ws(ws, &lo);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  const size_t n = (size_t)lo.n;
  if (depth_bits)
    SGS_CUDA(cudaMemcpyAsync(depth_bits, at<uint32_t>(ws, lo.depth_key), n * 4, cudaMemcpyDeviceToDevice, st));
  if (rect) SGS_CUDA(cudaMemcpyAsync(rect, at<uint2>(ws, lo.rect), n * 8, cudaMemcpyDeviceToDevice, st));
  if (tiles_touched)
    SGS_CUDA(cudaMemcpyAsync(tiles_touched, at<uint32_t>(ws, lo.tiles_touched), n * 4, cudaMemcpyDeviceToDevice, st));
  if (records) {
    SGS_CUDA(cudaMemcpy2DAsync(records, 64, at<float4>(ws, lo.rec_geo), 16, 16, n, cudaMemcpyDeviceToDevice, st));
    SGS_CUDA(cudaMemcpy2DAsync(records + 4, 64, at<float4>(ws, lo.rec_con), 16, 16, n, cudaMemcpyDeviceToDevice, st));
    SGS_CUDA(cudaMemcpy2DAsync(records + 8, 64, at<float4>(ws, lo.rec_eig), 16, 16, n, cudaMemcpyDeviceToDevice, st));
    SGS_CUDA(cudaMemcpy2DAsync(records + 12, 64, at<float4>(ws, lo.rec_col), 16, 16, n, cudaMemcpyDeviceToDevice, st));
  }
  return SGS_OK;
}

int sgs_debug_buffer(const sgs_workspace* ws, int32_t which, void** ptr, uint64_t* offset_bytes) {
  Layout lo;
  int rc = check_ws(ws, &lo);
  if (rc) return rc;
  const uint64_t offs[] = {lo.counters, lo.rec_geo, lo.rec_con, lo.rec_col, lo.depth_key, lo.rect,
                           lo.tiles_touched, lo.dkey_alt, lo.dkey_tmp, lo.didx, lo.didx_alt, lo.offsets,
                           lo.scan_blocks, lo.ent_key, lo.ent_key_alt, lo.ent_val, lo.ent_val_alt, lo.ranges,
                           lo.hist, lo.status};
  if (which < 0 || which >= (int)(sizeof(offs) / sizeof(offs[0])) || !ptr) {
    set_error("unknown debug buffer %d", which);
    return SGS_E_ARG;
  }
  *ptr = at<char>(ws, offs[which]);
  if (offset_bytes) *offset_bytes = offs[which];
  return SGS_OK;
}

int sgs_sort_temp_size(int64_t n, int32_t key_bits, uint64_t* bytes_out) {
  if (n < 0 || n > (int64_t)kMaxEntries || key_bits < 1 || key_bits > 64 || !bytes_out) {
    set_error("invalid sort size");
    return SGS_E_ARG;
  }
  *bytes_out = sort_u64_temp_bytes((uint64_t)n, key_bits);
  return SGS_OK;
}

int sgs_sort_pairs_u64(uint64_t* keys, uint32_t* values, int64_t n, int32_t key_bits, void* temp,
                       uint64_t temp_bytes, void* stream) {
  if (n < 0 || n > (int64_t)kMaxEntries || key_bits < 1 || key_bits > 64 || (n > 0 && (!keys || !values || !temp))) {
    set_error("invalid sort arguments");
    return SGS_E_ARG;
  }
  if (n == 0) return SGS_OK;
  return launch_sort_u64(reinterpret_cast<unsigned long long*>(keys), values, (uint32_t)n, key_bits, temp, temp_bytes,
                         as_stream(stream));
}

int sgs_loss_workspace_size(int32_t height, int32_t width, uint64_t* bytes_out) {
  if (height < 1 || width < 1 || !bytes_out) {
    set_error("invalid image size");
    return SGS_E_ARG;
  }
  *bytes_out = loss_workspace_bytes(height, width);
  return SGS_OK;
}

int sgs_image_loss(const void* img, int32_t img_is_f64, const void* target, int32_t target_is_f64, int32_t height,
                   int32_t width, const sgs_loss_config* cfg, float* dimg, double* dimg_f64, double* ssim_map,
                   double* out, void* workspace, uint64_t workspace_bytes, void* stream) {
  return launch_image_loss(img, img_is_f64, target, target_is_f64, height, width, cfg, dimg, dimg_f64, ssim_map, out,
                           workspace, workspace_bytes, as_stream(stream));
}

int sgs_topk_mask_temp_size(int64_t n, uint64_t* bytes_out) {
  if (n < 0 || n > (int64_t)kMaxEntries || !bytes_out) {
    set_error("invalid top-k size");
    return SGS_E_ARG;
  }
  *bytes_out = topk_temp_bytes((uint64_t)n);
  return SGS_OK;
}

int sgs_topk_mask(const double* scores, int64_t n, int64_t k, uint8_t* keep, void* temp, uint64_t temp_bytes,
                  void* stream) {
  if (n < 0 || n > (int64_t)kMaxEntries || k < 0 || k > n || (n > 0 && (!scores || !keep || !temp))) {
    set_error("invalid top-k arguments (need 0 <= k <= n)");
    return SGS_E_ARG;
  }
  if (n == 0) return SGS_OK;
  return launch_topk_mask(scores, (uint32_t)n, (uint32_t)k, keep, temp, temp_bytes, as_stream(stream));
}

int sgs_compact_header(const uint8_t* data, uint64_t size, int64_t* count_out) {
  return compact_header(data, size, count_out);
}

int sgs_compact_index(const uint8_t* data, uint64_t size, uint64_t* offsets, int64_t offsets_cap,
                      int32_t* max_lobes_out) {
  return compact_index(data, size, offsets, offsets_cap, max_lobes_out);
}

int sgs_compact_decode(const uint8_t* data, const uint64_t* offsets, int64_t n, int32_t n_lobes,
                       const sgs_scene_soa* out, void* stream) {
  if (n < 0 || n_lobes < 0 || n_lobes > 255 || !out ||
      (n > 0 && (!data || !offsets || !out->position || !out->quat || !out->log_scale || !out->opacity ||
                 !out->diffuse || !out->lobe_mask ||
                 (n_lobes > 0 && (!out->axis_raw || !out->sharpness || !out->amplitude))))) {
    set_error("invalid compact decode arguments");
    return SGS_E_ARG;
  }
  return launch_compact_decode(data, offsets, n, n_lobes, out, as_stream(stream));
}

}  // extern "C"
