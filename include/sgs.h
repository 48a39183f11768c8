/* sgs.h -- C ABI of the B200 SG-splat rasterizer (libsgs.so, sm_100a).
 *
 * This is the drop-in boundary for the reference's render hot path.  The
 * reference (`sgsplat`, pure Python/NumPy) has no FFI: its interface is the
 * set of Python functions in pkg/src/sgsplat/render.py.  Each entry point
 * below names the reference function (file:line) whose work it replaces; the
 * Python host layer `paper_2509_07021_b200.render` binds these through ctypes
 * and presents the reference signatures unchanged.
 *
 * Conventions
 *   - every pointer argument that names an array is a DEVICE pointer, fp32
 *     structure-of-arrays in the reference SceneParams layout
 *     (render.py:90-108): position (N,3), quat (N,4) w-first, log_scale (N,3),
 *     opacity (N) activated, diffuse (N,3), axis_raw (N,L,3), sharpness (N,L)
 *     activated, amplitude (N,L,3); plus the soft-pruning masks lobe_mask
 *     (N,L) and prim_mask (N) as floats in [0,1];
 *   - `stream` is a cudaStream_t passed as void* (0 = legacy default stream);
 *   - every call returns 0 on success or a negative SGS_E* code; no C++
 *     exception crosses the ABI.  sgs_last_error() returns a message;
 *   - all scratch lives in ONE caller-allocated device workspace whose size is
 *     given by sgs_workspace_size(), so the caller's allocator (PyTorch's
 *     caching allocator) accounts for every byte of render VRAM.
 */
#ifndef SGS_H_
#define SGS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SGS_OK 0
#define SGS_E_ARG (-1)        /* invalid argument (the reference raises ValueError) */
#define SGS_E_CUDA (-2)       /* CUDA runtime error */
#define SGS_E_WORKSPACE (-3)  /* workspace too small for N / image size */
#define SGS_E_CAPACITY (-4)   /* tile-entry capacity exceeded; grow and retry */
#define SGS_E_FORMAT (-5)     /* malformed scene file (the reference raises SceneFormatError) */
#define SGS_E_TRUNCATED (-6)  /* scene file shorter than its header promises (TruncatedFileError) */

#define SGS_SORT_DEPTH_FIRST 0  /* global depth sort of primitives + stable tile bucketing */
#define SGS_SORT_KEY64 1        /* (tile<<32 | depth_bits) keys, 64-bit onesweep radix sort */

/* Pinhole camera, render.py:30-57 (Camera).  rotation rows = (right, down,
 * forward) world-to-camera; pixel = (fx x/z + cx, fy y/z + cy).  tile_y0/1 is
 * a tile-row window [tile_y0, tile_y1) for tile-strip renders (0,0 = all);
 * lowpass is the `lowpass` argument of _prepare / project (render.py:259, 320). */
typedef struct sgs_camera {
  float rotation[9];
  float translation[3];
  float fx, fy, cx, cy;
  float near_z;
  int32_t width, height;
  int32_t tile_y0, tile_y1;
  float lowpass; /* cov2d diagonal floor in px^2, render.py:26 (0.3) */
  /* Depth in float64 (render.py:262-263, 307): the camera's third row and
   * t_z as the caller's doubles, and the near plane.  The visibility test
   * z > near and the depth ORDER use z = (w0 x + w1 y) + w2 z + t_z in
   * float64, so primitives are ordered exactly like the reference's
   * argsort of its float64 z (ties by lower index); the float32 depth key is
   * that z rounded, and equal keys are ordered by the float64 residual.
   * depth_row all zero = derive it from the float32 rotation/translation. */
  double depth_row[4];
  double near_z64;
  /* Gradient renders: bin every primitive with at least this opacity's
   * support (o_eff below it still blends with its true opacity, 0 included).
   * The reference blends every primitive into every pixel, so dL/do of a
   * primitive at o_eff = 0 is sum dL/dalpha G, not 0 (render.py:538-560);
   * with grad_floor > 0 such primitives get that gradient (and can recover
   * in the pruning loop).  0 = plain opacity-aware support. */
  float grad_floor;
} sgs_camera;

/* Packed parameter arrays, render.py:90-108 (SceneParams) + soft masks. */
typedef struct sgs_params {
  const float* position;
  const float* quat;
  const float* log_scale;
  const float* opacity;
  const float* diffuse;
  const float* axis_raw;
  const float* sharpness;
  const float* amplitude;
  const float* lobe_mask; /* (N,L); required */
  const float* prim_mask; /* (N); NULL means all ones */
  int64_t n;
  int32_t n_lobes;
} sgs_params;

/* Parameter gradients, render.py:179-194 (GradientSet) + mask gradients.
 * Outputs are OVERWRITTEN (not accumulated).  lobe_mask / prim_mask may be
 * NULL when the caller does not train masks. */
typedef struct sgs_grads {
  float* position;
  float* quat;
  float* log_scale;
  float* opacity;
  float* diffuse;
  float* axis_raw;
  float* sharpness;
  float* amplitude;
  float* lobe_mask;
  float* prim_mask;
  int32_t flags;  /* SGS_GRADS_* bits; 0 = overwrite every output row */
} sgs_grads;

/* sgs_grads.flags */
#define SGS_GRADS_ACCUMULATE 1  /* add into the outputs (a multi-view gradient sum) */
#define SGS_GRADS_MASK_LOGIT 2  /* mask gradients w.r.t. logits: x m (1 - m), m = sigmoid(logit) = the mask */

/* Device workspace descriptor.  `base` is ONE caller-allocated device buffer
 * of at least sgs_workspace_size() bytes for the same (n, n_lobes, width,
 * height, entry_capacity, sort_mode); the library carves it deterministically,
 * so the descriptor is all the state there is. */
typedef struct sgs_workspace {
  void* base;
  uint64_t bytes;
  int64_t n;
  int32_t n_lobes;
  int32_t width, height;
  int32_t sort_mode;
  int64_t entry_capacity;
} sgs_workspace;

/* Frame counters, readable after any stage (device copy inside the workspace). */
typedef struct sgs_stats {
  uint64_t n_visible;      /* z > near, render.py:263 */
  uint64_t n_emitting;     /* visible primitives with >= 1 tile entry */
  uint64_t n_entries;      /* per-tile (tile, depth) entries E of the tile lists */
  uint64_t capacity;       /* entry capacity the workspace was carved for */
  uint64_t overflow;       /* 1 if n_entries > capacity (frame must be redone) */
  uint64_t vram3s_visible; /* reference VRAM model, postprocess.py:118-135 */
  uint64_t vram3s_entries;
  uint64_t n_bin_entries;  /* entries the binning sorted: (super-tile, primitive)
                              in depth-first mode, (tile, primitive) in key64 mode;
                              the entry capacity bounds this number */
} sgs_stats;

/* Library / ABI version and last error message (thread-local). */
int32_t sgs_version(void);

/* ADMM penalized descent step (prune.py:162-201), fused: every parameter
 * class of every primitive updated in one pass per stage, no host sync.
 * Parameter / gradient arrays in the SceneParams layout (float32). */
typedef struct sgs_admm_fields {
  float* position;
  float* quat;
  float* log_scale;
  float* opacity;
  float* diffuse;
  float* axis_raw;
  float* sharpness;
  float* amplitude;
} sgs_admm_fields;

typedef struct sgs_admm_rates {
  float position, quat, log_scale, opacity, diffuse, axis_raw, sharpness, amplitude; /* group rates */
  float eta, delta_o, delta_s;                                                       /* step, penalties */
} sgs_admm_rates;

/* stage 1 (delta != 0, after the first gradient g1): the opacity step with
 * its penalty and clip.  stage 2 (after g2 -- or after g1 when delta == 0,
 * with update_o = 1 and delta_s = 0): the sharpness step with its penalty
 * (gradient g_sharpness), the other classes from g1, the clips.  proxy /
 * dual vectors z_o, u_o (N), z_s, u_s (N,L).  ok: device uint8, 0 = leave
 * everything unchanged (a non-finite gradient was seen); NULL = always. */
int sgs_admm_update(int64_t n, int32_t n_lobes, int32_t stage, int32_t update_o, const sgs_admm_fields* params,
                    const sgs_admm_fields* g1, const float* g_sharpness, const float* z_o, const float* u_o,
                    const float* z_s, const float* u_s, const sgs_admm_rates* rates, const uint8_t* ok,
                    void* stream);

/* sizeof of the ABI structs as this library was compiled: out[0..3] =
 * sgs_camera, sgs_params, sgs_workspace, sgs_stats (bindings check theirs). */
int sgs_abi_sizes(uint64_t out[4]);
const char* sgs_last_error(void);

/* Bytes of device workspace for N primitives, an image of width x height
 * and room for `entry_capacity` tile entries. */
int sgs_workspace_size(const sgs_workspace* ws, uint64_t* bytes_out);

/* K1 preprocess -- replaces _prepare (render.py:259-317) minus its depth
 * argsort: projection, EWA conic, near/opacity/frustum culling, support
 * rectangle, exact ellipse-tile counts and SG color (masked lobes skipped). */
int sgs_preprocess(const sgs_params* params, const sgs_camera* cam, const sgs_workspace* ws,
                   void* stream);

/* K2-K4 binning -- replaces the depth argsort (render.py:307).  Emits one
 * (tile, depth) entry per touched tile and sorts them stably by
 * (tile, depth, primitive index); writes per-tile [start, end) ranges.
 * ws->sort_mode picks SGS_SORT_DEPTH_FIRST or SGS_SORT_KEY64; both produce
 * bit-identical results.  Never synchronises: when E exceeds the workspace's
 * entry capacity only the first `capacity` entries are kept and
 * sgs_stats.overflow is set -- grow the workspace and redo the frame.
 * In SGS_SORT_DEPTH_FIRST mode the depth-digit histograms are accumulated by
 * sgs_preprocess, so each sgs_bin must follow its own sgs_preprocess. */
int sgs_bin(const sgs_camera* cam, const sgs_workspace* ws, void* stream);

/* K5 forward raster -- replaces _chunk_blend + _render_params
 * (render.py:355-408).  out_img (H,W,3), out_T (H,W) final transmittance,
 * out_ncontrib (H,W) number of per-tile entries consumed by each pixel.
 * out_T and out_ncontrib may be NULL for an image-only render (render.py:411);
 * sgs_raster_backward needs both from the same frame.
 * weight_sums_fx (N uint64, two's-complement fixed point in units of 2^-32)
 * is ACCUMULATED with the composited blending weights (the reference's
 * in-place np.add.at, render.py:406-407) when non-NULL: integer addition
 * makes the sums independent of the order tiles and views land in, so the
 * importance scores are bitwise reproducible; sgs_fixed_to_float(.., 32, ..)
 * converts.  pair_count (one device uint64), when non-NULL, is incremented by
 * the number of (pixel, entry) pairs evaluated before each pixel terminated
 * -- the raster's algorithmic work unit. */
int sgs_raster_forward(const sgs_camera* cam, const float background[3],
                       const sgs_workspace* ws, float* out_img, float* out_T,
                       uint32_t* out_ncontrib, uint64_t* weight_sums_fx, uint64_t* pair_count,
                       void* stream);

/* out[i] (+)= (int64)fx[i] * 2^-frac_bits for i < n (accumulate != 0: add). */
int sgs_fixed_to_float(const uint64_t* fx, int64_t n, int32_t frac_bits, float* out, int32_t accumulate,
                       void* stream);

/* Convenience: preprocess + bin + raster_forward in one call (graph-capturable). */
int sgs_render_forward(const sgs_params* params, const sgs_camera* cam, const float background[3],
                       const sgs_workspace* ws, float* out_img, float* out_T, uint32_t* out_ncontrib,
                       uint64_t* weight_sums_fx, uint64_t* pair_count, void* stream);

/* K6 backward raster -- replaces the pixel loop of _backward_from_blend
 * (render.py:535-573).  dimg (H,W,3) = dL/dimage.  grad2d (N,9) is
 * OVERWRITTEN with per-primitive [dL/dcolor(3), sum dq, sum dq dx, sum dq dy,
 * sum dq dx^2, sum dq dx dy, sum dq dy^2] where q is the conic quadratic form. */
int sgs_raster_backward(const sgs_camera* cam, const float background[3],
                        const sgs_workspace* ws, const float* img, const float* final_T,
                        const uint32_t* ncontrib, const float* dimg, float* grad2d, void* stream);

/* sgs_raster_backward with bitwise-reproducible sums: the raster runs twice
 * (per-(primitive, partial) max |partial|, then 64-bit fixed-point sums
 * scaled to it), so grad2d does not depend on the order tiles finish in.
 * scratch: device bytes >= sgs_raster_backward_det_scratch_bytes(N). */
uint64_t sgs_raster_backward_det_scratch_bytes(int64_t n);
int sgs_raster_backward_det(const sgs_camera* cam, const float background[3],
                            const sgs_workspace* ws, const float* img, const float* final_T,
                            const uint32_t* ncontrib, const float* dimg, float* grad2d,
                            void* scratch, uint64_t scratch_bytes, void* stream);

/* K7 preprocess backward -- replaces render.py:575-636 (conic -> cov2d ->
 * Sigma/J -> quat/log_scale/position, SG color path, scatter) and adds the
 * soft-mask gradients dL/dm_p = o dL/do_eff, dL/dm_l = (dL/dc_pre . a_l) e_l. */
int sgs_preprocess_backward(const sgs_params* params, const sgs_camera* cam, const float* grad2d,
                            sgs_grads* grads, void* stream);

/* K7 for several views of one primitive set (a training step): the same
 * rows as one sgs_preprocess_backward per view in view order (bit-identical),
 * with each primitive's parameters read, its view-independent terms formed and
 * its gradient rows written once per 8 views.  cams[v] / grad2d[v]: host
 * arrays of n_views cameras and device partial buffers (K6 outputs). */
int sgs_preprocess_backward_views(const sgs_params* params, const sgs_camera* cams, int n_views,
                                  const float* const* grad2d, sgs_grads* grads, void* stream);

/* Per-primitive projection (all N primitives, 16 floats each):
 * [visible, depth, mean2d x/y, cov2d 00/01/11, conic 00/01/11, color_pre rgb,
 * color rgb] -- the per-primitive outputs of _prepare (render.py:259-317) and
 * project (render.py:320-330), for the host API and inspection. */
int sgs_project_records(const sgs_params* params, const sgs_camera* cam, float* out, void* stream);

/* Read the frame counters (synchronises `stream`). */
int sgs_get_stats(const sgs_workspace* ws, sgs_stats* out, void* stream);

/* Reference VRAM model (postprocess.py:101-137): 3-sigma AABB visible count
 * and tile entries with `tile_px` tiles; results land in sgs_stats. */
int sgs_vram_model(const sgs_params* params, const sgs_camera* cam, int32_t tile_px,
                   const sgs_workspace* ws, void* stream);

/* Export the per-tile lists as 64-bit (tile<<32 | depth_bits) keys and
 * primitive-index values (device buffers of length >= n_entries), and the
 * per-tile [start, end) ranges (tiles_x*tiles_y uint32 pairs), materialised
 * from the binned lists with the raster's own membership test.  For parity
 * checks; all three buffers are required. */
int sgs_export_bins(const sgs_workspace* ws, const sgs_camera* cam, uint64_t* keys,
                    uint32_t* values, uint32_t* ranges, void* stream);

/* Export per-primitive preprocess outputs (device buffers, length N):
 * depth bits, packed tile rect (tx0|tx1<<16, ty0|ty1<<16), tile counts and
 * the 16-float raster record [geo(4) = (mean x, mean y, log2 o_eff, pmin),
 * conic(4) = (A, B, C, kx), scaled eigen form(4), color(4)] (sgs_geom.h). */
int sgs_export_projected(const sgs_workspace* ws, uint32_t* depth_bits,
                         uint32_t* rect, uint32_t* tiles_touched, float* records, void* stream);

/* Device address of an internal workspace sub-buffer (debugging / tests):
 * 0 counters, 1-3 records, 4 depth keys, 5 rects, 6 tile counts, 7-8 depth
 * sort keys, 9-10 depth order, 11 offsets, 12 scan blocks, 13-14 entry keys,
 * 15-16 entry values, 17 ranges, 18 histograms, 19 look-back status. */
int sgs_debug_buffer(const sgs_workspace* ws, int32_t which, void** ptr, uint64_t* offset_bytes);

/* Stable LSD radix sort of (key, value) pairs on the low `key_bits` bits of
 * 64-bit keys (onesweep, decoupled look-back).  In-place on keys/values;
 * `temp` of sgs_sort_temp_size() bytes. */
int sgs_sort_temp_size(int64_t n, int32_t key_bits, uint64_t* bytes_out);
int sgs_sort_pairs_u64(uint64_t* keys, uint32_t* values, int64_t n, int32_t key_bits, void* temp,
                       uint64_t temp_bytes, void* stream);

/* Image loss (render.py:197-205, 433-509): (1 - lambda) L1 + lambda (1 - SSIM)
 * with a normalised Gaussian window (odd, <= 31 taps) and zero padding. */
typedef struct sgs_loss_config {
  double lambda_ssim; /* LossConfig.lambda_ssim (0.2) */
  int32_t window;     /* LossConfig.window (11) */
  double sigma;       /* LossConfig.sigma (1.5) */
  double c1, c2;      /* LossConfig.c1 / c2 (0.01^2, 0.03^2) */
} sgs_loss_config;

/* Device scratch bytes for sgs_image_loss on an H x W x 3 image. */
int sgs_loss_workspace_size(int32_t height, int32_t width, uint64_t* bytes_out);

/* Fused loss + dL/dimg -- replaces loss / ssim / _ssim_grad / _loss_and_dimg
 * (render.py:464-509).  img and target are (H,W,3) device arrays, float32 or
 * float64 (the *_is_f64 flags).  out (device, 3 doubles) receives
 * [loss, mean |img - target|, mean SSIM].  dimg (float32) / dimg_f64 / ssim_map
 * (float64, (H,W,3)) are optional (NULL to skip).  Statistics are accumulated
 * in float64.  Never synchronises. */
int sgs_image_loss(const void* img, int32_t img_is_f64, const void* target, int32_t target_is_f64,
                   int32_t height, int32_t width, const sgs_loss_config* cfg, float* dimg,
                   double* dimg_f64, double* ssim_map, double* out, void* workspace,
                   uint64_t workspace_bytes, void* stream);

/* ADMM proximal projection support (prune.py:204-213, _top_k_mask): keep[i] =
 * 1 for the k largest of n float64 device scores, ties keeping the lower
 * index (np.argsort(-scores, kind="stable")[:k]); keep is a device uint8
 * array of n.  temp: sgs_topk_mask_temp_size() bytes of device scratch. */
int sgs_topk_mask_temp_size(int64_t n, uint64_t* bytes_out);
int sgs_topk_mask(const double* scores, int64_t n, int64_t k, uint8_t* keep, void* temp,
                  uint64_t temp_bytes, void* stream);

/* MEGS2 compact scene files (io.py:1-15 layout, 173-214 read_compact) into
 * the renderer's device SoA.  Host side: sgs_compact_header reads the
 * primitive count; sgs_compact_index walks the variable-length records of a
 * HOST buffer into count + 1 byte offsets (host array) and the largest lobe
 * count, with the reference's checks (bad magic / version / trailing bytes
 * -> SGS_E_FORMAT, short payload -> SGS_E_TRUNCATED).  Device side:
 * sgs_compact_decode reads the uploaded bytes and offsets (device arrays)
 * and writes the SceneParams arrays (render.py:135-145) for n_lobes slots:
 * log_scale = log(scale), unused slots axis (0,0,1), zero sharpness /
 * amplitude, lobe_mask 0/1. */
typedef struct sgs_scene_soa {
  float* position;  /* (N,3) */
  float* quat;      /* (N,4) */
  float* log_scale; /* (N,3) */
  float* opacity;   /* (N) */
  float* diffuse;   /* (N,3) */
  float* axis_raw;  /* (N,L,3) */
  float* sharpness; /* (N,L) */
  float* amplitude; /* (N,L,3) */
  float* lobe_mask; /* (N,L) */
} sgs_scene_soa;

int sgs_compact_header(const uint8_t* data, uint64_t size, int64_t* count_out);
int sgs_compact_index(const uint8_t* data, uint64_t size, uint64_t* offsets, int64_t offsets_cap,
                      int32_t* max_lobes_out);
int sgs_compact_decode(const uint8_t* data, const uint64_t* offsets, int64_t n, int32_t n_lobes,
                       const sgs_scene_soa* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SGS_H_ */
