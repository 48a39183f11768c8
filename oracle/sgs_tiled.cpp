// oracle/sgs_tiled.cpp -- TEST INFRASTRUCTURE ONLY.  CPU restatement of the
// tiled SG-splat pipeline that libsgs.so runs on the GPU.  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it; the
// product path never does.
//
// Role: the bit-exact authority for the integer outputs the reference does
// not define (tile keys, sorted order, per-tile ranges, tile counts,
// visibility counts), and a tolerance oracle for images and gradients at full
// frame sizes where the dense reference restatement (oracle/ref_dense.py)
// is infeasible.  It is itself pinned to the reference by tests that compare
// it with oracle/ref_dense.py and the golden fixtures generated from
// /root/reference (tests/golden/).
//
//   preprocess      -- shares the IEEE-exact geometry header
//                      paper_2509_07021_b200/csrc/sgs_geom.h (the survey's
//                      prescription for GPU<->CPU bit-exactness); compiled
//                      with -ffp-contract=off, no fast-math.
//   binning         -- independent: entries emitted in primitive-index order
//                      with the full 64-bit key (tile << 32 | depth_bits) and
//                      std::stable_sort, i.e. the definition of the order.
//   raster forward  -- independent per-pixel loop, fp32, libm exp2f.
//   raster backward -- independent, float64, explicit reverse suffix sums
//                      (restates render.py:535-573 per pixel).
//   preprocess bwd  -- independent float64 restatement of render.py:575-636
//                      plus the soft-mask gradients.
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "../paper_2509_07021_b200/csrc/sgs_geom.h"

namespace {

SgsCam make_cam(const float* R, const float* t, float fx, float fy, float cx, float cy, float near_z, int W, int H,
                int tile_y0, int tile_y1, float lowpass, const double* cam_d) {
  SgsCam c;
  c.lowpass = lowpass;
  // float64 depth row + near (sgs_camera.depth_row / near_z64): cam_d = (w0, w1, w2, tz, near)
  for (int k = 0; k < 3; ++k) c.rz[k] = cam_d ? cam_d[k] : (double)R[6 + k];
  c.tz = cam_d ? cam_d[3] : (double)t[2];
  c.near64 = cam_d ? cam_d[4] : (double)near_z;
  c.grad_floor = cam_d ? (float)cam_d[5] : 0.0f;
  for (int i = 0; i < 9; ++i) c.R[i] = R[i];
  for (int i = 0; i < 3; ++i) c.t[i] = t[i];
  for (int k = 0; k < 3; ++k) {
    double s = 0.0;
    for (int i = 0; i < 3; ++i) s += (double)R[3 * i + k] * (double)t[i];
    c.C[k] = (float)(-s);
  }
  c.fx = fx;
  c.fy = fy;
  c.cx = cx;
  c.cy = cy;
  c.near_z = near_z;
  c.width = W;
  c.height = H;
  c.tiles_x = (W + SGS_TILE - 1) / SGS_TILE;
  c.tiles_y = (H + SGS_TILE - 1) / SGS_TILE;
  if (tile_y0 == 0 && tile_y1 == 0) tile_y1 = c.tiles_y;
  c.tile_y0 = tile_y0;
  c.tile_y1 = tile_y1;
  return c;
}

}  // namespace

extern "C" {

// cam_f: R[9], t[3], fx, fy, cx, cy, near, lowpass (18 floats); cam_i: W, H, tile_y0, tile_y1
// outputs (length N): depth_bits, rect (2 u32 packed like the GPU), tiles_touched,
// records (12 floats: geo, con, col); counts[0] = visible, counts[1] = emitting.
void oracle_preprocess(int64_t n, int L, const float* pos, const float* quat, const float* ls, const float* opac,
                       const float* diffuse, const float* axis, const float* sharp, const float* amp,
                       const float* lmask, const float* pmask, const float* cam_f, const int32_t* cam_i,
                       const double* cam_d, uint32_t* depth_bits, float* depth_res, uint32_t* rect,
                       uint32_t* tiles_touched, float* records, int64_t* counts) {
  SgsCam cam = make_cam(cam_f, cam_f + 9, cam_f[12], cam_f[13], cam_f[14], cam_f[15], cam_f[16], cam_i[0], cam_i[1],
                        cam_i[2], cam_i[3], cam_f[17], cam_d);
  int64_t vis = 0, emit = 0;
  for (int64_t i = 0; i < n; ++i) {
    SgsProj pr;
    sgs_project(pos + 3 * i, quat + 4 * i, ls + 3 * i, opac[i], pmask ? pmask[i] : 1.0f, &cam, &pr);
    vis += pr.visible;
    uint32_t cnt = 0;
    float g[4] = {0, 0, 0, 0}, k[4] = {0, 0, 0, 0};
    if (pr.emits) {
      sgs_pack_geo(&pr, g, k);
      cnt = sgs_count_tiles(pr.tx0, pr.ty0, pr.tx1, pr.ty1, g, k, &cam);
    }
    tiles_touched[i] = cnt;
    depth_bits[i] = cnt ? sgs_float_to_bits(pr.depth) : 0x7fffffffu;
    depth_res[i] = cnt ? pr.depth_res : 0.0f;
    rect[2 * i] = (uint32_t)(pr.tx0 & 0xffff) | ((uint32_t)(pr.tx1 & 0xffff) << 16);
    rect[2 * i + 1] = (uint32_t)(pr.ty0 & 0xffff) | ((uint32_t)(pr.ty1 & 0xffff) << 16);
    float* rec = records + 16 * i;
    memset(rec, 0, 16 * sizeof(float));
    if (cnt) {
      ++emit;
      const SgsSpan sp = sgs_span(g, k);
      float span2[3];
      sgs_span_cache(&sp, &k[3], span2);
      float c_pre[3], c[3];
      sgs_color(pos + 3 * i, diffuse + 3 * i, axis + (size_t)i * L * 3, sharp + (size_t)i * L, amp + (size_t)i * L * 3,
                lmask + (size_t)i * L, L, &cam, c_pre, c);
      float e4[4];
      sgs_pack_eig(&pr, e4);
      memcpy(rec, g, 16);
      memcpy(rec + 4, k, 16);
      memcpy(rec + 8, e4, 16);
      rec[12] = c[0];
      rec[13] = c[1];
      rec[14] = c[2];
    }
  }
  counts[0] = vis;
  counts[1] = emit;
}

// Count entries (returns E).
int64_t oracle_count_entries(int64_t n, const uint32_t* tiles_touched) {
  int64_t e = 0;
  for (int64_t i = 0; i < n; ++i) e += tiles_touched[i];
  return e;
}

// Emit (tile<<32 | depth_bits, index) in index order, stable sort on the key
// and, for equal keys, the float64 depth residual: the per-tile order is the
// reference's stable argsort of float64 z (render.py:307).  keys/vals have
// room for E entries; ranges has tiles_x*tiles_y*2 u32 (zeroed here).
void oracle_bin(int64_t n, const uint32_t* depth_bits, const float* depth_res, const uint32_t* rect,
                const uint32_t* tiles_touched, const float* records, const float* cam_f, const int32_t* cam_i,
                uint64_t* keys, uint32_t* vals, uint32_t* ranges) {
  SgsCam cam = make_cam(cam_f, cam_f + 9, cam_f[12], cam_f[13], cam_f[14], cam_f[15], cam_f[16], cam_i[0], cam_i[1],
                        cam_i[2], cam_i[3], cam_f[17], nullptr);
  std::vector<std::pair<uint64_t, uint32_t>> ent;
  for (int64_t i = 0; i < n; ++i) {
    if (!tiles_touched[i]) continue;
    int tx0 = (int)(rect[2 * i] & 0xffff), tx1 = (int)(int16_t)(rect[2 * i] >> 16);
    int ty0 = (int)(rect[2 * i + 1] & 0xffff), ty1 = (int)(int16_t)(rect[2 * i + 1] >> 16);
    const float* g = records + 16 * i;
    const float* k = g + 4;
    const SgsSpan sp = sgs_span(g, k);
    for (int ty = ty0; ty <= ty1; ++ty) {
      int first;
      const int cnt = sgs_row_span(&sp, &cam, ty, tx0, tx1, &first);
      for (int tx = first; tx < first + cnt; ++tx)
        ent.emplace_back(((uint64_t)(ty * cam.tiles_x + tx) << 32) | depth_bits[i], (uint32_t)i);
    }
  }
  std::stable_sort(ent.begin(), ent.end(),
                   [depth_res](const std::pair<uint64_t, uint32_t>& a, const std::pair<uint64_t, uint32_t>& b) {
                     if (a.first != b.first) return a.first < b.first;
                     return depth_res[a.second] < depth_res[b.second];
                   });
  const size_t T = (size_t)cam.tiles_x * cam.tiles_y;
  memset(ranges, 0, T * 2 * sizeof(uint32_t));
  for (size_t j = 0; j < ent.size(); ++j) {
    keys[j] = ent[j].first;
    vals[j] = ent[j].second;
    uint32_t t = (uint32_t)(ent[j].first >> 32);
    if (j == 0 || (uint32_t)(ent[j - 1].first >> 32) != t) ranges[2 * t] = (uint32_t)j;
    if (j + 1 == ent.size() || (uint32_t)(ent[j + 1].first >> 32) != t) ranges[2 * t + 1] = (uint32_t)(j + 1);
  }
}

// Forward: img (H,W,3), T (H,W), nc (H,W); weight_sums (N) accumulated if non-null.
void oracle_raster_forward(const uint32_t* ranges, const uint32_t* vals, const float* records, const float* cam_f,
                           const int32_t* cam_i, const float* bg, float* img, float* Tout, uint32_t* nc_out,
                           double* weight_sums) {
  SgsCam cam = make_cam(cam_f, cam_f + 9, cam_f[12], cam_f[13], cam_f[14], cam_f[15], cam_f[16], cam_i[0], cam_i[1],
                        cam_i[2], cam_i[3], cam_f[17], nullptr);
  for (int py = cam.tile_y0 * SGS_TILE; py < std::min(cam.height, cam.tile_y1 * SGS_TILE); ++py)
    for (int px = 0; px < cam.width; ++px) {
      const int tile = (py / SGS_TILE) * cam.tiles_x + px / SGS_TILE;
      const uint32_t s = ranges[2 * tile], e = std::max(ranges[2 * tile + 1], s);
      const float fx = (float)px + 0.5f, fy = (float)py + 0.5f;
      float T = 1.0f, C[3] = {0, 0, 0};
      uint32_t nc = 0;
      for (uint32_t j = s; j < e; ++j) {
        const float* r = records + 16 * (size_t)vals[j];
        const float dx = fx - r[0], dy = fy - r[1];
        // scaled eigen form with log2(o_eff) folded in (sgs_pack_eig), same
        // operation order as the GPU raster: p = log2(o_eff G)
        const float t1 = fmaf(r[9], dy, r[8] * dx), t2 = fmaf(r[10], dy, -(r[11] * dx));
        const float p = fmaf(-t1, t1, fmaf(-t2, t2, r[2]));
        // every listed primitive is blended (alpha < 1e-7 outside its support)
        const float a = exp2f(p);
        const float alpha = std::min(a, SGS_ALPHA_MAX);
        const float w = alpha * T;
        const float Tn = T - w;  // the GPU's blend step (sgs_geom.h SGS_T_KEEP)
        if (Tn < SGS_T_KEEP) break;
        for (int c = 0; c < 3; ++c) C[c] += w * r[12 + c];
        if (weight_sums) weight_sums[vals[j]] += w;
        T = Tn;
        nc = j - s + 1;
      }
      const size_t pix = (size_t)py * cam.width + px;
      for (int c = 0; c < 3; ++c) img[3 * pix + c] = C[c] + T * bg[c];
      Tout[pix] = T;
      nc_out[pix] = nc;
    }
}

// Backward (float64): per pixel, recompute the kept prefix front to back,
// then suffix sums back to front.  grad2d (N,9) accumulated (caller zeroes):
// [dL/dc (3), sum dq, sum dq dx, sum dq dy, sum dq dx^2, sum dq dx dy, sum dq dy^2].
void oracle_raster_backward(const uint32_t* ranges, const uint32_t* vals, const float* records, const float* cam_f,
                            const int32_t* cam_i, const float* bg, const float* dimg, double* grad2d) {
  SgsCam cam = make_cam(cam_f, cam_f + 9, cam_f[12], cam_f[13], cam_f[14], cam_f[15], cam_f[16], cam_i[0], cam_i[1],
                        cam_i[2], cam_i[3], cam_f[17], nullptr);
  struct Item {
    uint32_t g;
    double G, a, alpha, T, dx, dy;
  };
  std::vector<Item> kept;
  for (int py = cam.tile_y0 * SGS_TILE; py < std::min(cam.height, cam.tile_y1 * SGS_TILE); ++py)
    for (int px = 0; px < cam.width; ++px) {
      const int tile = (py / SGS_TILE) * cam.tiles_x + px / SGS_TILE;
      const uint32_t s = ranges[2 * tile], e = std::max(ranges[2 * tile + 1], s);
      const double fx = px + 0.5, fy = py + 0.5;
      kept.clear();
      double T = 1.0;
      for (uint32_t j = s; j < e; ++j) {
        const float* r = records + 16 * (size_t)vals[j];
        const double dx = fx - r[0], dy = fy - r[1];
        const double t1 = (double)r[8] * dx + (double)r[9] * dy, t2 = (double)r[10] * dy - (double)r[11] * dx;
        const double p = (double)r[2] - t1 * t1 - t2 * t2;  // log2(o_eff G)
        const double a = exp2(p);
        // o_eff G: dq below is -1/2 o G dalpha; a record at o_eff = 0 (binned
        // by the gradient floor) carries G itself, the opacity partial per
        // unit opacity (its geometry partials are zero: alpha = 0 G)
        const double G = std::isinf(r[2]) ? exp2(-t1 * t1 - t2 * t2) : a;
        const double alpha = std::min(a, 0.99);
        const double Tn = T * (1.0 - alpha);
        if (Tn < (double)SGS_T_KEEP) break;
        kept.push_back({vals[j], G, a, alpha, T, dx, dy});
        T = Tn;
      }
      const size_t pix = (size_t)py * cam.width + px;
      const double g0 = dimg[3 * pix], g1 = dimg[3 * pix + 1], g2 = dimg[3 * pix + 2];
      double S = T * (g0 * bg[0] + g1 * bg[1] + g2 * bg[2]);
      for (size_t q = kept.size(); q-- > 0;) {
        const Item& it = kept[q];
        const float* r = records + 16 * (size_t)it.g;
        const double cg = r[12] * g0 + r[13] * g1 + r[14] * g2;
        const double w = it.alpha * it.T;
        const double om = 1.0 - it.alpha;
        const double dalpha = it.a < 0.99 ? (it.T * cg - S / om) : 0.0;
        S += w * cg;
        const double dq = -0.5 * it.G * dalpha;
        double* d = grad2d + 9 * (size_t)it.g;
        d[0] += w * g0;
        d[1] += w * g1;
        d[2] += w * g2;
        d[3] += dq;
        d[4] += dq * it.dx;
        d[5] += dq * it.dy;
        d[6] += dq * it.dx * it.dx;
        d[7] += dq * it.dx * it.dy;
        d[8] += dq * it.dy * it.dy;
      }
    }
}

// Preprocess backward in float64 (render.py:575-636 + mask gradients).
// Outputs are overwritten; lobe-mask / prim-mask gradients optional (nullable).
void oracle_preprocess_backward(int64_t n, int L, const float* pos, const float* quat, const float* ls,
                                const float* opac, const float* diffuse, const float* axis, const float* sharp,
                                const float* amp, const float* lmask, const float* pmask, const float* cam_f,
                                const double* grad2d, double* d_pos, double* d_quat, double* d_ls, double* d_op,
                                double* d_diff, double* d_axis, double* d_sharp, double* d_amp, double* d_lmask,
                                double* d_pmask) {
  const float* W = cam_f;
  const float* tv = cam_f + 9;
  const double fx = cam_f[12], fy = cam_f[13];
  double Cc[3];
  for (int k = 0; k < 3; ++k) {
    double s = 0.0;
    for (int i = 0; i < 3; ++i) s += (double)W[3 * i + k] * (double)tv[i];
    Cc[k] = -s;
  }
  for (int64_t i = 0; i < n; ++i) {
    const double* gv = grad2d + 9 * i;
    double dp[3] = {0, 0, 0}, dq4[4] = {0, 0, 0, 0}, dl[3] = {0, 0, 0};
    double dop = 0, dpm = 0;
    bool any = false;
    for (int c = 0; c < 9; ++c) any |= gv[c] != 0.0;
    const double P[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
    if (any) {
      double pc[3];
      for (int r = 0; r < 3; ++r) pc[r] = W[3 * r] * P[0] + W[3 * r + 1] * P[1] + W[3 * r + 2] * P[2] + tv[r];
      const double x = pc[0], y = pc[1], z = pc[2];
      double q[4] = {quat[4 * i], quat[4 * i + 1], quat[4 * i + 2], quat[4 * i + 3]};
      const double qn = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
      const double w_ = q[0] / qn, x_ = q[1] / qn, y_ = q[2] / qn, z_ = q[3] / qn;
      double R[9] = {1 - 2 * (y_ * y_ + z_ * z_), 2 * (x_ * y_ - w_ * z_),     2 * (x_ * z_ + w_ * y_),
                     2 * (x_ * y_ + w_ * z_),     1 - 2 * (x_ * x_ + z_ * z_), 2 * (y_ * z_ - w_ * x_),
                     2 * (x_ * z_ - w_ * y_),     2 * (y_ * z_ + w_ * x_),     1 - 2 * (x_ * x_ + y_ * y_)};
      double D[3];
      for (int k = 0; k < 3; ++k) D[k] = exp(2.0 * ls[3 * i + k]);
      double S[9];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
          double s = 0;
          for (int k = 0; k < 3; ++k) s += R[3 * a + k] * D[k] * R[3 * b + k];
          S[3 * a + b] = s;
        }
      const double J[6] = {fx / z, 0, -fx * x / (z * z), 0, fy / z, -fy * y / (z * z)};
      double M[6];
      for (int r = 0; r < 2; ++r)
        for (int k = 0; k < 3; ++k) {
          double s = 0;
          for (int j = 0; j < 3; ++j) s += J[3 * r + j] * W[3 * j + k];
          M[3 * r + k] = s;
        }
      double MS[6];
      for (int r = 0; r < 2; ++r)
        for (int k = 0; k < 3; ++k) {
          double s = 0;
          for (int j = 0; j < 3; ++j) s += M[3 * r + j] * S[3 * j + k];
          MS[3 * r + k] = s;
        }
      double cov[4];
      for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 2; ++c) {
          double s = 0;
          for (int j = 0; j < 3; ++j) s += MS[3 * r + j] * M[3 * c + j];
          cov[2 * r + c] = s;
        }
      cov[0] += (double)cam_f[17];
      cov[3] += (double)cam_f[17];
      const double det = cov[0] * cov[3] - cov[1] * cov[2];
      const double K[4] = {cov[3] / det, -cov[1] / det, -cov[2] / det, cov[0] / det};
      const double zg0 = ((double)opac[i] * (pmask ? pmask[i] : 1.0f)) > 0 ? 1.0 : 0.0;
      const double dK[4] = {zg0 * gv[6], zg0 * gv[7], zg0 * gv[7], zg0 * gv[8]};
      const double dmx = -2.0 * zg0 * (K[0] * gv[4] + K[1] * gv[5]);
      const double dmy = -2.0 * zg0 * (K[2] * gv[4] + K[3] * gv[5]);
      const double oe = (double)opac[i] * (pmask ? pmask[i] : 1.0f);
      // o_eff = 0: the raster stored -1/2 sum G dalpha (per unit opacity) and
      // the mean / conic partials of alpha = 0 G are zero
      const double doe = oe > 0 ? -2.0 * gv[3] / oe : -2.0 * gv[3];
      dop = (pmask ? pmask[i] : 1.0f) * doe;
      dpm = opac[i] * doe;
      double KdK[4], dcov[4];
      for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 2; ++c) KdK[2 * r + c] = K[2 * r] * dK[c] + K[2 * r + 1] * dK[2 + c];
      for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 2; ++c) dcov[2 * r + c] = -(KdK[2 * r] * K[c] + KdK[2 * r + 1] * K[2 + c]);
      double dS[9];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
          double s = 0;
          for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 2; ++c) s += M[3 * r + a] * dcov[2 * r + c] * M[3 * c + b];
          dS[3 * a + b] = s;
        }
      double dM[6];
      for (int r = 0; r < 2; ++r)
        for (int k = 0; k < 3; ++k) dM[3 * r + k] = 2.0 * (dcov[2 * r] * MS[k] + dcov[2 * r + 1] * MS[3 + k]);
      double dJ[6];
      for (int r = 0; r < 2; ++r)
        for (int j = 0; j < 3; ++j) {
          double s = 0;
          for (int k = 0; k < 3; ++k) s += dM[3 * r + k] * W[3 * j + k];
          dJ[3 * r + j] = s;
        }
      double dpc[3];
      dpc[0] = dJ[2] * (-fx / (z * z)) + dmx * fx / z;
      dpc[1] = dJ[5] * (-fy / (z * z)) + dmy * fy / z;
      dpc[2] = dJ[0] * (-fx / (z * z)) + dJ[4] * (-fy / (z * z)) + dJ[2] * (2 * fx * x / (z * z * z)) +
               dJ[5] * (2 * fy * y / (z * z * z)) - dmx * fx * x / (z * z) - dmy * fy * y / (z * z);
      for (int k = 0; k < 3; ++k) dp[k] = W[k] * dpc[0] + W[3 + k] * dpc[1] + W[6 + k] * dpc[2];
      double dR[9];
      for (int a = 0; a < 3; ++a)
        for (int k = 0; k < 3; ++k) {
          double s = 0;
          for (int j = 0; j < 3; ++j) s += dS[3 * a + j] * R[3 * j + k];
          dR[3 * a + k] = 2.0 * s * D[k];
        }
      for (int k = 0; k < 3; ++k) {
        double s = 0;
        for (int a = 0; a < 3; ++a)
          for (int j = 0; j < 3; ++j) s += R[3 * a + k] * dS[3 * a + j] * R[3 * j + k];
        dl[k] = 2.0 * D[k] * s;
      }
      // dR/dq (w,x,y,z), each scaled by 2
      const double Dw[9] = {0, -z_, y_, z_, 0, -x_, -y_, x_, 0};
      const double Dx[9] = {0, y_, z_, y_, -2 * x_, -w_, z_, w_, -2 * x_};
      const double Dy[9] = {-2 * y_, x_, w_, x_, 0, z_, -w_, z_, -2 * y_};
      const double Dz[9] = {-2 * z_, -w_, x_, w_, -2 * z_, y_, x_, y_, 0};
      double gq[4] = {0, 0, 0, 0};
      for (int k = 0; k < 9; ++k) {
        gq[0] += 2 * Dw[k] * dR[k];
        gq[1] += 2 * Dx[k] * dR[k];
        gq[2] += 2 * Dy[k] * dR[k];
        gq[3] += 2 * Dz[k] * dR[k];
      }
      const double qh[4] = {w_, x_, y_, z_};
      const double qd = qh[0] * gq[0] + qh[1] * gq[1] + qh[2] * gq[2] + qh[3] * gq[3];
      for (int k = 0; k < 4; ++k) dq4[k] = (gq[k] - qh[k] * qd) / qn;
    }
    // color path
    double v[3] = {P[0] - Cc[0], P[1] - Cc[1], P[2] - Cc[2]};
    const double rd = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    for (int k = 0; k < 3; ++k) v[k] /= rd;
    double cpre[3] = {diffuse[3 * i], diffuse[3 * i + 1], diffuse[3 * i + 2]};
    std::vector<double> e(L), dt(L), mu(3 * L), un(L);
    for (int l = 0; l < L; ++l) {
      const float* u = axis + ((size_t)i * L + l) * 3;
      un[l] = sqrt((double)u[0] * u[0] + (double)u[1] * u[1] + (double)u[2] * u[2]);
      for (int k = 0; k < 3; ++k) mu[3 * l + k] = u[k] / un[l];
      dt[l] = mu[3 * l] * v[0] + mu[3 * l + 1] * v[1] + mu[3 * l + 2] * v[2];
      e[l] = exp((double)sharp[(size_t)i * L + l] * (dt[l] - 1.0));
      for (int c = 0; c < 3; ++c) cpre[c] += e[l] * lmask[(size_t)i * L + l] * amp[((size_t)i * L + l) * 3 + c];
    }
    double dcp[3];
    for (int c = 0; c < 3; ++c) dcp[c] = cpre[c] > 0 ? gv[c] : 0.0;
    double dv[3] = {0, 0, 0};
    for (int l = 0; l < L; ++l) {
      const size_t li = (size_t)i * L + l;
      const double m = lmask[li], s = sharp[li];
      const double da = dcp[0] * amp[3 * li] + dcp[1] * amp[3 * li + 1] + dcp[2] * amp[3 * li + 2];
      for (int c = 0; c < 3; ++c) d_amp[3 * li + c] = dcp[c] * e[l] * m;
      const double ga = da * e[l] * m;
      d_sharp[li] = ga * (dt[l] - 1.0);
      if (d_lmask) d_lmask[li] = da * e[l];
      const double dm[3] = {ga * s * v[0], ga * s * v[1], ga * s * v[2]};
      const double pr = mu[3 * l] * dm[0] + mu[3 * l + 1] * dm[1] + mu[3 * l + 2] * dm[2];
      for (int k = 0; k < 3; ++k) {
        d_axis[3 * li + k] = (dm[k] - mu[3 * l + k] * pr) / un[l];
        dv[k] += ga * s * mu[3 * l + k];
      }
    }
    const double pv = v[0] * dv[0] + v[1] * dv[1] + v[2] * dv[2];
    for (int k = 0; k < 3; ++k) dp[k] += (dv[k] - v[k] * pv) / rd;
    for (int k = 0; k < 3; ++k) {
      d_pos[3 * i + k] = dp[k];
      d_ls[3 * i + k] = dl[k];
      d_diff[3 * i + k] = dcp[k];
    }
    for (int k = 0; k < 4; ++k) d_quat[4 * i + k] = dq4[k];
    d_op[i] = dop;
    if (d_pmask) d_pmask[i] = dpm;
  }
}

// Exposed for tests of the shared polynomial exp/log.
float oracle_sgs_expf(float x) { return sgs_expf(x); }
float oracle_sgs_logf(float x) { return sgs_logf(x); }

}  // extern "C"
