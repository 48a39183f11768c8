// preprocess_bwd.cu -- K7: per-primitive chain rule from the raster partials
// (dL/dcolor, conic moments) to every parameter class and the soft masks.
// Replaces /root/reference/pkg/src/sgsplat/render.py:575-636 (conic ->
// cov2d -> Sigma / J -> quaternion / log-scale / position, SG color path,
// np.add.at scatter) and adds
//   dL/dm_p = o   dL/do_eff          (o_eff = m_p o)
//   dL/dm_l = (dL/dc_pre . a_l) e_l  (c_pre = diffuse + sum_l m_l a_l e_l)
// One thread per primitive; every output row is written (zeros for
// primitives no pixel kept), so outputs need no memset.  With
// SGS_GRADS_ACCUMULATE the rows are added to the outputs instead (a training
// step sums its views straight into one gradient bucket), and with
// SGS_GRADS_MASK_LOGIT the mask gradients are taken through the sigmoid that
// produced the masks: dL/dlogit = dL/dm m (1 - m).
#include "common.cuh"

namespace sgs {

constexpr int kG2 = 9;

template <bool kAcc>
__device__ __forceinline__ void put(float* p, int64_t i, float v) {
  if (kAcc)
    p[i] += v;
  else
    p[i] = v;
}

// One view (the drop-in loss_and_grads, importance passes, the ADMM step):
// rows written directly, fewer live registers than the multi-view kernel.
template <bool kAcc, int kL>
__global__ void __launch_bounds__(128) preprocess_bwd_kernel1(sgs_params P, SgsCam cam,
                                                             const float* __restrict__ grad2d, sgs_grads out) {
  const bool logit = (out.flags & SGS_GRADS_MASK_LOGIT) != 0;
  const int64_t n = P.n;
  const int L = kL > 0 ? kL : P.n_lobes;  // kL = 3: lobe loops unrolled, per-lobe arrays in registers
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float gv[kG2];
    bool any = false;
#pragma unroll
    for (int c = 0; c < kG2; ++c) {
      gv[c] = grad2d[i * kG2 + c];
      any |= gv[c] != 0.0f;
    }
    float d_pos[3] = {0, 0, 0}, d_q[4] = {0, 0, 0, 0}, d_ls[3] = {0, 0, 0}, d_diff[3] = {0, 0, 0};
    float d_op = 0.0f, d_pm = 0.0f;
    const float* Wr = cam.R;
    const float pos[3] = {P.position[3 * i], P.position[3 * i + 1], P.position[3 * i + 2]};
    const float op = P.opacity[i];
    const float pm = P.prim_mask ? P.prim_mask[i] : 1.0f;

    if (any) {
      // ---------------- forward recompute, float64 like K1's projection
      // (sgs_geom.h sgs_project): for elongated splats cov2d is nearly
      // singular before the low-pass floor, and the conic and the chain
      // d cov = -K dK K amplify float32 cancellation far beyond rtol 1e-3.
      const double p0 = pos[0], p1 = pos[1], p2 = pos[2];
      const double x = (double)Wr[0] * p0 + (double)Wr[1] * p1 + (double)Wr[2] * p2 + (double)cam.t[0];
      const double y = (double)Wr[3] * p0 + (double)Wr[4] * p1 + (double)Wr[5] * p2 + (double)cam.t[1];
      const double z = (double)Wr[6] * p0 + (double)Wr[7] * p1 + (double)Wr[8] * p2 + (double)cam.t[2];
      const float4 q4 = reinterpret_cast<const float4*>(P.quat)[i];
      const double qn = sqrt((double)q4.x * q4.x + (double)q4.y * q4.y + (double)q4.z * q4.z + (double)q4.w * q4.w);
      const double qw = q4.x / qn, qx = q4.y / qn, qy = q4.z / qn, qz = q4.w / qn;
      double R[9];
      R[0] = 1.0 - 2.0 * (qy * qy + qz * qz);
      R[1] = 2.0 * (qx * qy - qw * qz);
      R[2] = 2.0 * (qx * qz + qw * qy);
      R[3] = 2.0 * (qx * qy + qw * qz);
      R[4] = 1.0 - 2.0 * (qx * qx + qz * qz);
      R[5] = 2.0 * (qy * qz - qw * qx);
      R[6] = 2.0 * (qx * qz - qw * qy);
      R[7] = 2.0 * (qy * qz + qw * qx);
      R[8] = 1.0 - 2.0 * (qx * qx + qy * qy);
      double D[3];
      for (int k = 0; k < 3; ++k) D[k] = exp(2.0 * (double)P.log_scale[3 * i + k]);
      double S[9];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
          S[3 * a + b] = R[3 * a] * D[0] * R[3 * b] + R[3 * a + 1] * D[1] * R[3 * b + 1] + R[3 * a + 2] * D[2] * R[3 * b + 2];
      const double iz = 1.0 / z, iz2 = iz * iz;
      const double fxd = cam.fx, fyd = cam.fy;
      const double J00 = fxd * iz, J02 = -fxd * x * iz2, J11 = fyd * iz, J12 = -fyd * y * iz2;
      double M[6];
      for (int k = 0; k < 3; ++k) {
        M[k] = J00 * Wr[k] + J02 * Wr[6 + k];
        M[3 + k] = J11 * Wr[3 + k] + J12 * Wr[6 + k];
      }
      double MS[6];  // M Sigma
      for (int r = 0; r < 2; ++r)
        for (int k = 0; k < 3; ++k)
          MS[3 * r + k] = M[3 * r] * S[k] + M[3 * r + 1] * S[3 + k] + M[3 * r + 2] * S[6 + k];
      const double lp = cam.lowpass;
      const double ca = MS[0] * M[0] + MS[1] * M[1] + MS[2] * M[2] + lp;
      const double cb = MS[0] * M[3] + MS[1] * M[4] + MS[2] * M[5];
      const double cc = MS[3] * M[3] + MS[4] * M[4] + MS[5] * M[5] + lp;
      const double idet = 1.0 / (ca * cc - cb * cb);
      const double k00 = cc * idet, k01 = -cb * idet, k11 = ca * idet;

      // ---------------- 2D partials
      // o_eff = 0 (binned by the gradient floor): K6 stored the dq partials
      // per unit opacity, and alpha = 0 G has no mean / conic gradient
      const float oeff = op * pm;
      const double zg = oeff > 0.0f ? 1.0 : 0.0;
      const double m0 = gv[3], m1x = zg * gv[4], m1y = zg * gv[5], m2xx = zg * gv[6], m2xy = zg * gv[7],
                   m2yy = zg * gv[8];
      const double dmx = -2.0 * (k00 * m1x + k01 * m1y);
      const double dmy = -2.0 * (k01 * m1x + k11 * m1y);
      const float d_oeff = (float)(oeff > 0.0f ? -2.0 * m0 / (double)oeff : -2.0 * m0);
      d_op = pm * d_oeff;
      d_pm = op * d_oeff;
      // d_cov = -K dK K (K = conic, dK symmetric with off-diagonals m2xy)
      const double t00 = k00 * m2xx + k01 * m2xy, t01 = k00 * m2xy + k01 * m2yy;
      const double t10 = k01 * m2xx + k11 * m2xy, t11 = k01 * m2xy + k11 * m2yy;
      const double dc00 = -(t00 * k00 + t01 * k01), dc01 = -(t00 * k01 + t01 * k11);
      const double dc10 = -(t10 * k00 + t11 * k01), dc11 = -(t10 * k01 + t11 * k11);
      // dSigma = M^T dcov M ; dM = 2 dcov M Sigma (dcov symmetric)
      double dS[9];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
          dS[3 * a + b] = M[a] * (dc00 * M[b] + dc01 * M[3 + b]) + M[3 + a] * (dc10 * M[b] + dc11 * M[3 + b]);
      double dM[6];
      for (int k = 0; k < 3; ++k) {
        dM[k] = 2.0 * (dc00 * MS[k] + dc01 * MS[3 + k]);
        dM[3 + k] = 2.0 * (dc10 * MS[k] + dc11 * MS[3 + k]);
      }
      // dJ = dM W^T (only J00, J02, J11, J12 are live)
      const double dJ00 = dM[0] * Wr[0] + dM[1] * Wr[1] + dM[2] * Wr[2];
      const double dJ02 = dM[0] * Wr[6] + dM[1] * Wr[7] + dM[2] * Wr[8];
      const double dJ11 = dM[3] * Wr[3] + dM[4] * Wr[4] + dM[5] * Wr[5];
      const double dJ12 = dM[3] * Wr[6] + dM[4] * Wr[7] + dM[5] * Wr[8];
      const double iz3 = iz2 * iz;
      const double dpc0 = dJ02 * (-fxd * iz2) + dmx * fxd * iz;
      const double dpc1 = dJ12 * (-fyd * iz2) + dmy * fyd * iz;
      const double dpc2 = dJ00 * (-fxd * iz2) + dJ11 * (-fyd * iz2) + dJ02 * (2.0 * fxd * x * iz3) +
                          dJ12 * (2.0 * fyd * y * iz3) - dmx * fxd * x * iz2 - dmy * fyd * y * iz2;
      for (int k = 0; k < 3; ++k) d_pos[k] = (float)(Wr[k] * dpc0 + Wr[3 + k] * dpc1 + Wr[6 + k] * dpc2);

      // Sigma = R D R^T
      double dR[9];
      for (int a = 0; a < 3; ++a)
        for (int k = 0; k < 3; ++k)
          dR[3 * a + k] = 2.0 * (dS[3 * a] * R[k] + dS[3 * a + 1] * R[3 + k] + dS[3 * a + 2] * R[6 + k]) * D[k];
      for (int k = 0; k < 3; ++k) {
        double s = 0.0;
        for (int a = 0; a < 3; ++a)
          s += R[3 * a + k] * (dS[3 * a] * R[k] + dS[3 * a + 1] * R[3 + k] + dS[3 * a + 2] * R[6 + k]);
        d_ls[k] = (float)(2.0 * D[k] * s);
      }
      // d qhat = sum_ij dR_ij dR_ij/dqhat (render.py:217-229)
      const double gw = 2.0 * (-qz * dR[1] + qy * dR[2] + qz * dR[3] - qx * dR[5] - qy * dR[6] + qx * dR[7]);
      const double gx = 2.0 * (qy * dR[1] + qz * dR[2] + qy * dR[3] - 2.0 * qx * dR[4] - qw * dR[5] + qz * dR[6] +
                               qw * dR[7] - 2.0 * qx * dR[8]);
      const double gy = 2.0 * (-2.0 * qy * dR[0] + qx * dR[1] + qw * dR[2] + qx * dR[3] + qz * dR[5] - qw * dR[6] +
                               qz * dR[7] - 2.0 * qy * dR[8]);
      const double gz = 2.0 * (-2.0 * qz * dR[0] - qw * dR[1] + qx * dR[2] + qw * dR[3] - 2.0 * qz * dR[4] +
                               qy * dR[5] + qx * dR[6] + qy * dR[7]);
      const double qd = qw * gw + qx * gx + qy * gy + qz * gz;
      d_q[0] = (float)((gw - qw * qd) / qn);
      d_q[1] = (float)((gx - qx * qd) / qn);
      d_q[2] = (float)((gy - qy * qd) / qn);
      d_q[3] = (float)((gz - qz * qd) / qn);
    }

    // ---------------- color path (all lobes, masked ones too: dL/dm_l)
    const float v0r = pos[0] - cam.C[0], v1r = pos[1] - cam.C[1], v2r = pos[2] - cam.C[2];
    const float rd = sqrtf(v0r * v0r + v1r * v1r + v2r * v2r);
    const float v0 = v0r / rd, v1 = v1r / rd, v2 = v2r / rd;
    float cpre[3] = {P.diffuse[3 * i], P.diffuse[3 * i + 1], P.diffuse[3 * i + 2]};
    float e[SGS_MAX_LOBES], dotv[SGS_MAX_LOBES];
#pragma unroll
    for (int l = 0; l < (kL > 0 ? kL : L); ++l) {
      const float* u = P.axis_raw + (i * L + l) * 3;
      const float un = sqrtf(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
      dotv[l] = (u[0] * v0 + u[1] * v1 + u[2] * v2) / un;
      e[l] = expf(P.sharpness[i * L + l] * (dotv[l] - 1.0f));
      const float m = P.lobe_mask[i * L + l];
      if (m != 0.0f)
        for (int c = 0; c < 3; ++c) cpre[c] += e[l] * m * P.amplitude[(i * L + l) * 3 + c];
    }
    float dcp[3];
    for (int c = 0; c < 3; ++c) {
      dcp[c] = cpre[c] > 0.0f ? gv[c] : 0.0f;
      d_diff[c] = dcp[c];
    }
    float dv[3] = {0, 0, 0};
#pragma unroll
    for (int l = 0; l < (kL > 0 ? kL : L); ++l) {
      const float* u = P.axis_raw + (i * L + l) * 3;
      const float* a = P.amplitude + (i * L + l) * 3;
      const float m = P.lobe_mask[i * L + l];
      const float s = P.sharpness[i * L + l];
      const float da = dcp[0] * a[0] + dcp[1] * a[1] + dcp[2] * a[2];
      const float em = e[l] * m;
      for (int c = 0; c < 3; ++c) put<kAcc>(out.amplitude, (i * L + l) * 3 + c, dcp[c] * em);
      const float ga = da * em;
      put<kAcc>(out.sharpness, i * L + l, ga * (dotv[l] - 1.0f));
      if (out.lobe_mask) put<kAcc>(out.lobe_mask, i * L + l, logit ? da * e[l] * (m * (1.0f - m)) : da * e[l]);
      const float un = sqrtf(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
      const float mu0 = u[0] / un, mu1 = u[1] / un, mu2 = u[2] / un;
      // d mu = ga s v ; d u = (I - mu mu^T) d mu / |u|
      const float gs = ga * s;
      const float dm0 = gs * v0, dm1 = gs * v1, dm2 = gs * v2;
      const float pr = mu0 * dm0 + mu1 * dm1 + mu2 * dm2;
      put<kAcc>(out.axis_raw, (i * L + l) * 3 + 0, (dm0 - mu0 * pr) / un);
      put<kAcc>(out.axis_raw, (i * L + l) * 3 + 1, (dm1 - mu1 * pr) / un);
      put<kAcc>(out.axis_raw, (i * L + l) * 3 + 2, (dm2 - mu2 * pr) / un);
      dv[0] += gs * mu0;
      dv[1] += gs * mu1;
      dv[2] += gs * mu2;
    }
    const float pv = v0 * dv[0] + v1 * dv[1] + v2 * dv[2];
    d_pos[0] += (dv[0] - v0 * pv) / rd;
    d_pos[1] += (dv[1] - v1 * pv) / rd;
    d_pos[2] += (dv[2] - v2 * pv) / rd;

    for (int k = 0; k < 3; ++k) {
      put<kAcc>(out.position, 3 * i + k, d_pos[k]);
      put<kAcc>(out.log_scale, 3 * i + k, d_ls[k]);
      put<kAcc>(out.diffuse, 3 * i + k, d_diff[k]);
    }
    float4 q = make_float4(d_q[0], d_q[1], d_q[2], d_q[3]);
    if (kAcc) {
      const float4 o = reinterpret_cast<const float4*>(out.quat)[i];
      q = make_float4(o.x + q.x, o.y + q.y, o.z + q.z, o.w + q.w);
    }
    reinterpret_cast<float4*>(out.quat)[i] = q;
    put<kAcc>(out.opacity, i, d_op);
    if (out.prim_mask) put<kAcc>(out.prim_mask, i, logit ? d_pm * (pm * (1.0f - pm)) : d_pm);
  }
}

// Up to kMaxBwdViews views of one primitive set per launch (a training step
// or an importance pass): each primitive's parameters are read, its
// view-independent quantities (normalised quaternion, exp(2 log_scale)) formed
// and its gradient rows written once, the per-view chains summed in view
// order in registers.  The sum is seeded with the output row when
// accumulating, so the result is bit-identical to one launch per view.
constexpr int kMaxBwdViews = 8;
struct BwdViews {
  SgsCam cam[kMaxBwdViews];
  const float* g2d[kMaxBwdViews];
  int n;
};

#ifndef SGS_K7_MIN_BLOCKS
#define SGS_K7_MIN_BLOCKS 3  // 168 registers (a few spills): ~1.5 % more training views/s than 254
#endif
template <bool kAcc, int kL>
__global__ void __launch_bounds__(128, SGS_K7_MIN_BLOCKS) preprocess_bwd_kernel(sgs_params P, BwdViews V, sgs_grads out) {
  const bool logit = (out.flags & SGS_GRADS_MASK_LOGIT) != 0;
  const int64_t n = P.n;
  const int L = kL > 0 ? kL : P.n_lobes;  // kL = 3: lobe loops unrolled, per-lobe arrays in registers
  constexpr int LA = kL > 0 ? kL : SGS_MAX_LOBES;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float pos[3] = {P.position[3 * i], P.position[3 * i + 1], P.position[3 * i + 2]};
    const float op = P.opacity[i];
    const float pm = P.prim_mask ? P.prim_mask[i] : 1.0f;
    // view-independent parts of the float64 projection (as K1 / sgs_project),
    // formed for the first view that has partials for this primitive
    bool pre = false;
    double qn = 1.0, qw = 1.0, qx = 0.0, qy = 0.0, qz = 0.0, D[3] = {1.0, 1.0, 1.0};

    // gradient rows, seeded with the outputs when accumulating
    float a_pos[3], a_q[4], a_ls[3], a_diff[3], a_op, a_pm = 0.0f;
    float a_amp[LA][3], a_sh[LA], a_lm[LA], a_ax[LA][3];
    for (int k = 0; k < 3; ++k) {
      a_pos[k] = kAcc ? out.position[3 * i + k] : 0.0f;
      a_ls[k] = kAcc ? out.log_scale[3 * i + k] : 0.0f;
      a_diff[k] = kAcc ? out.diffuse[3 * i + k] : 0.0f;
    }
    {
      const float4 o = kAcc ? reinterpret_cast<const float4*>(out.quat)[i] : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      a_q[0] = o.x;
      a_q[1] = o.y;
      a_q[2] = o.z;
      a_q[3] = o.w;
    }
    a_op = kAcc ? out.opacity[i] : 0.0f;
    if (out.prim_mask) a_pm = kAcc ? out.prim_mask[i] : 0.0f;
#pragma unroll
    for (int l = 0; l < LA; ++l) {
      if (kL == 0 && l >= L) break;
      for (int c = 0; c < 3; ++c) {
        a_amp[l][c] = kAcc ? out.amplitude[(i * L + l) * 3 + c] : 0.0f;
        a_ax[l][c] = kAcc ? out.axis_raw[(i * L + l) * 3 + c] : 0.0f;
      }
      a_sh[l] = kAcc ? out.sharpness[i * L + l] : 0.0f;
      a_lm[l] = (out.lobe_mask && kAcc) ? out.lobe_mask[i * L + l] : 0.0f;
    }

    for (int v = 0; v < V.n; ++v) {
      const SgsCam& cam = V.cam[v];
      const float* grad2d = V.g2d[v];
      float gv[kG2];
      bool any = false;
#pragma unroll
      for (int c = 0; c < kG2; ++c) {
        gv[c] = grad2d[i * kG2 + c];
        any |= gv[c] != 0.0f;
      }
      float d_pos[3] = {0, 0, 0}, d_q[4] = {0, 0, 0, 0}, d_ls[3] = {0, 0, 0};
      float d_op = 0.0f, d_pm = 0.0f;
      const float* Wr = cam.R;

      if (any) {
        if (!pre) {
          const float4 q4 = reinterpret_cast<const float4*>(P.quat)[i];
          qn = sqrt((double)q4.x * q4.x + (double)q4.y * q4.y + (double)q4.z * q4.z + (double)q4.w * q4.w);
          qw = q4.x / qn;
          qx = q4.y / qn;
          qy = q4.z / qn;
          qz = q4.w / qn;
          for (int k = 0; k < 3; ++k) D[k] = exp(2.0 * (double)P.log_scale[3 * i + k]);
          pre = true;
        }
        // ---------------- forward recompute, float64 like K1's projection
        // (sgs_geom.h sgs_project): for elongated splats cov2d is nearly
        // singular before the low-pass floor, and the conic and the chain
        // d cov = -K dK K amplify float32 cancellation far beyond rtol 1e-3.
        const double p0 = pos[0], p1 = pos[1], p2 = pos[2];
        const double x = (double)Wr[0] * p0 + (double)Wr[1] * p1 + (double)Wr[2] * p2 + (double)cam.t[0];
        const double y = (double)Wr[3] * p0 + (double)Wr[4] * p1 + (double)Wr[5] * p2 + (double)cam.t[1];
        const double z = (double)Wr[6] * p0 + (double)Wr[7] * p1 + (double)Wr[8] * p2 + (double)cam.t[2];
        double R[9];
        R[0] = 1.0 - 2.0 * (qy * qy + qz * qz);
        R[1] = 2.0 * (qx * qy - qw * qz);
        R[2] = 2.0 * (qx * qz + qw * qy);
        R[3] = 2.0 * (qx * qy + qw * qz);
        R[4] = 1.0 - 2.0 * (qx * qx + qz * qz);
        R[5] = 2.0 * (qy * qz - qw * qx);
        R[6] = 2.0 * (qx * qz - qw * qy);
        R[7] = 2.0 * (qy * qz + qw * qx);
        R[8] = 1.0 - 2.0 * (qx * qx + qy * qy);
        double S[9];
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b)
            S[3 * a + b] =
                R[3 * a] * D[0] * R[3 * b] + R[3 * a + 1] * D[1] * R[3 * b + 1] + R[3 * a + 2] * D[2] * R[3 * b + 2];
        const double iz = 1.0 / z, iz2 = iz * iz;
        const double fxd = cam.fx, fyd = cam.fy;
        const double J00 = fxd * iz, J02 = -fxd * x * iz2, J11 = fyd * iz, J12 = -fyd * y * iz2;
        double M[6];
        for (int k = 0; k < 3; ++k) {
          M[k] = J00 * Wr[k] + J02 * Wr[6 + k];
          M[3 + k] = J11 * Wr[3 + k] + J12 * Wr[6 + k];
        }
        double MS[6];  // M Sigma
        for (int r = 0; r < 2; ++r)
          for (int k = 0; k < 3; ++k)
            MS[3 * r + k] = M[3 * r] * S[k] + M[3 * r + 1] * S[3 + k] + M[3 * r + 2] * S[6 + k];
        const double lp = cam.lowpass;
        const double ca = MS[0] * M[0] + MS[1] * M[1] + MS[2] * M[2] + lp;
        const double cb = MS[0] * M[3] + MS[1] * M[4] + MS[2] * M[5];
        const double cc = MS[3] * M[3] + MS[4] * M[4] + MS[5] * M[5] + lp;
        const double idet = 1.0 / (ca * cc - cb * cb);
        const double k00 = cc * idet, k01 = -cb * idet, k11 = ca * idet;

        // ---------------- 2D partials
        // o_eff = 0 (binned by the gradient floor): K6 stored the dq partials
        // per unit opacity, and alpha = 0 G has no mean / conic gradient
        const float oeff = op * pm;
        const double zg = oeff > 0.0f ? 1.0 : 0.0;
        const double m0 = gv[3], m1x = zg * gv[4], m1y = zg * gv[5], m2xx = zg * gv[6], m2xy = zg * gv[7],
                     m2yy = zg * gv[8];
        const double dmx = -2.0 * (k00 * m1x + k01 * m1y);
        const double dmy = -2.0 * (k01 * m1x + k11 * m1y);
        const float d_oeff = (float)(oeff > 0.0f ? -2.0 * m0 / (double)oeff : -2.0 * m0);
        d_op = pm * d_oeff;
        d_pm = op * d_oeff;
        // d_cov = -K dK K (K = conic, dK symmetric with off-diagonals m2xy)
        const double t00 = k00 * m2xx + k01 * m2xy, t01 = k00 * m2xy + k01 * m2yy;
        const double t10 = k01 * m2xx + k11 * m2xy, t11 = k01 * m2xy + k11 * m2yy;
        const double dc00 = -(t00 * k00 + t01 * k01), dc01 = -(t00 * k01 + t01 * k11);
        const double dc10 = -(t10 * k00 + t11 * k01), dc11 = -(t10 * k01 + t11 * k11);
        // dSigma = M^T dcov M ; dM = 2 dcov M Sigma (dcov symmetric)
        double dS[9];
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b)
            dS[3 * a + b] = M[a] * (dc00 * M[b] + dc01 * M[3 + b]) + M[3 + a] * (dc10 * M[b] + dc11 * M[3 + b]);
        double dM[6];
        for (int k = 0; k < 3; ++k) {
          dM[k] = 2.0 * (dc00 * MS[k] + dc01 * MS[3 + k]);
          dM[3 + k] = 2.0 * (dc10 * MS[k] + dc11 * MS[3 + k]);
        }
        // dJ = dM W^T (only J00, J02, J11, J12 are live)
        const double dJ00 = dM[0] * Wr[0] + dM[1] * Wr[1] + dM[2] * Wr[2];
        const double dJ02 = dM[0] * Wr[6] + dM[1] * Wr[7] + dM[2] * Wr[8];
        const double dJ11 = dM[3] * Wr[3] + dM[4] * Wr[4] + dM[5] * Wr[5];
        const double dJ12 = dM[3] * Wr[6] + dM[4] * Wr[7] + dM[5] * Wr[8];
        const double iz3 = iz2 * iz;
        const double dpc0 = dJ02 * (-fxd * iz2) + dmx * fxd * iz;
        const double dpc1 = dJ12 * (-fyd * iz2) + dmy * fyd * iz;
        const double dpc2 = dJ00 * (-fxd * iz2) + dJ11 * (-fyd * iz2) + dJ02 * (2.0 * fxd * x * iz3) +
                            dJ12 * (2.0 * fyd * y * iz3) - dmx * fxd * x * iz2 - dmy * fyd * y * iz2;
        for (int k = 0; k < 3; ++k) d_pos[k] = (float)(Wr[k] * dpc0 + Wr[3 + k] * dpc1 + Wr[6 + k] * dpc2);

        // Sigma = R D R^T
        double dR[9];
        for (int a = 0; a < 3; ++a)
          for (int k = 0; k < 3; ++k)
            dR[3 * a + k] = 2.0 * (dS[3 * a] * R[k] + dS[3 * a + 1] * R[3 + k] + dS[3 * a + 2] * R[6 + k]) * D[k];
        for (int k = 0; k < 3; ++k) {
          double sum = 0.0;
          for (int a = 0; a < 3; ++a)
            sum += R[3 * a + k] * (dS[3 * a] * R[k] + dS[3 * a + 1] * R[3 + k] + dS[3 * a + 2] * R[6 + k]);
          d_ls[k] = (float)(2.0 * D[k] * sum);
        }
        // d qhat = sum_ij dR_ij dR_ij/dqhat (render.py:217-229)
        const double gw = 2.0 * (-qz * dR[1] + qy * dR[2] + qz * dR[3] - qx * dR[5] - qy * dR[6] + qx * dR[7]);
        const double gx = 2.0 * (qy * dR[1] + qz * dR[2] + qy * dR[3] - 2.0 * qx * dR[4] - qw * dR[5] +
                                 qz * dR[6] + qw * dR[7] - 2.0 * qx * dR[8]);
        const double gy = 2.0 * (-2.0 * qy * dR[0] + qx * dR[1] + qw * dR[2] + qx * dR[3] + qz * dR[5] -
                                 qw * dR[6] + qz * dR[7] - 2.0 * qy * dR[8]);
        const double gz = 2.0 * (-2.0 * qz * dR[0] - qw * dR[1] + qx * dR[2] + qw * dR[3] - 2.0 * qz * dR[4] +
                                 qy * dR[5] + qx * dR[6] + qy * dR[7]);
        const double qd = qw * gw + qx * gx + qy * gy + qz * gz;
        d_q[0] = (float)((gw - qw * qd) / qn);
        d_q[1] = (float)((gx - qx * qd) / qn);
        d_q[2] = (float)((gy - qy * qd) / qn);
        d_q[3] = (float)((gz - qz * qd) / qn);
      }

      // ---------------- color path (all lobes, masked ones too: dL/dm_l)
      const float v0r = pos[0] - cam.C[0], v1r = pos[1] - cam.C[1], v2r = pos[2] - cam.C[2];
      const float rd = sqrtf(v0r * v0r + v1r * v1r + v2r * v2r);
      const float v0 = v0r / rd, v1 = v1r / rd, v2 = v2r / rd;
      float cpre[3] = {P.diffuse[3 * i], P.diffuse[3 * i + 1], P.diffuse[3 * i + 2]};
      float e[LA], dotv[LA];
#pragma unroll
      for (int l = 0; l < LA; ++l) {
        if (kL == 0 && l >= L) break;
        const float* u = P.axis_raw + (i * L + l) * 3;
        const float un = sqrtf(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
        dotv[l] = (u[0] * v0 + u[1] * v1 + u[2] * v2) / un;
        e[l] = expf(P.sharpness[i * L + l] * (dotv[l] - 1.0f));
        const float m = P.lobe_mask[i * L + l];
        if (m != 0.0f)
          for (int c = 0; c < 3; ++c) cpre[c] += e[l] * m * P.amplitude[(i * L + l) * 3 + c];
      }
      float dcp[3];
      for (int c = 0; c < 3; ++c) {
        dcp[c] = cpre[c] > 0.0f ? gv[c] : 0.0f;
        a_diff[c] += dcp[c];
      }
      float dv[3] = {0, 0, 0};
#pragma unroll
      for (int l = 0; l < LA; ++l) {
        if (kL == 0 && l >= L) break;
        const float* u = P.axis_raw + (i * L + l) * 3;
        const float* a = P.amplitude + (i * L + l) * 3;
        const float m = P.lobe_mask[i * L + l];
        const float s = P.sharpness[i * L + l];
        const float da = dcp[0] * a[0] + dcp[1] * a[1] + dcp[2] * a[2];
        const float em = e[l] * m;
        for (int c = 0; c < 3; ++c) a_amp[l][c] += dcp[c] * em;
        const float ga = da * em;
        a_sh[l] += ga * (dotv[l] - 1.0f);
        if (out.lobe_mask) a_lm[l] += logit ? da * e[l] * (m * (1.0f - m)) : da * e[l];
        const float un = sqrtf(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
        const float mu0 = u[0] / un, mu1 = u[1] / un, mu2 = u[2] / un;
        // d mu = ga s v ; d u = (I - mu mu^T) d mu / |u|
        const float gs = ga * s;
        const float dm0 = gs * v0, dm1 = gs * v1, dm2 = gs * v2;
        const float pr = mu0 * dm0 + mu1 * dm1 + mu2 * dm2;
        a_ax[l][0] += (dm0 - mu0 * pr) / un;
        a_ax[l][1] += (dm1 - mu1 * pr) / un;
        a_ax[l][2] += (dm2 - mu2 * pr) / un;
        dv[0] += gs * mu0;
        dv[1] += gs * mu1;
        dv[2] += gs * mu2;
      }
      const float pv = v0 * dv[0] + v1 * dv[1] + v2 * dv[2];
      d_pos[0] += (dv[0] - v0 * pv) / rd;
      d_pos[1] += (dv[1] - v1 * pv) / rd;
      d_pos[2] += (dv[2] - v2 * pv) / rd;
      for (int k = 0; k < 3; ++k) {
        a_pos[k] += d_pos[k];
        a_ls[k] += d_ls[k];
      }
      for (int k = 0; k < 4; ++k) a_q[k] += d_q[k];
      a_op += d_op;
      if (out.prim_mask) a_pm += logit ? d_pm * (pm * (1.0f - pm)) : d_pm;
    }

    for (int k = 0; k < 3; ++k) {
      out.position[3 * i + k] = a_pos[k];
      out.log_scale[3 * i + k] = a_ls[k];
      out.diffuse[3 * i + k] = a_diff[k];
    }
    reinterpret_cast<float4*>(out.quat)[i] = make_float4(a_q[0], a_q[1], a_q[2], a_q[3]);
    out.opacity[i] = a_op;
    if (out.prim_mask) out.prim_mask[i] = a_pm;
#pragma unroll
    for (int l = 0; l < LA; ++l) {
      if (kL == 0 && l >= L) break;
      for (int c = 0; c < 3; ++c) {
        out.amplitude[(i * L + l) * 3 + c] = a_amp[l][c];
        out.axis_raw[(i * L + l) * 3 + c] = a_ax[l][c];
      }
      out.sharpness[i * L + l] = a_sh[l];
      if (out.lobe_mask) out.lobe_mask[i * L + l] = a_lm[l];
    }
  }
}

int launch_preprocess_bwd_views(const sgs_params& P, const SgsCam* cams, const float* const* grad2d, int n_views,
                                const sgs_grads& g, cudaStream_t st) {
  int grid = persistent_grid((uint64_t)P.n, 128, 16);
  const bool acc = (g.flags & SGS_GRADS_ACCUMULATE) != 0;
  for (int v0 = 0; v0 < n_views; v0 += kMaxBwdViews) {
    BwdViews V;
    V.n = n_views - v0 < kMaxBwdViews ? n_views - v0 : kMaxBwdViews;
    for (int k = 0; k < V.n; ++k) {
      V.cam[k] = cams[v0 + k];
      V.g2d[k] = grad2d[v0 + k];
    }
    sgs_grads gg = g;
    if (v0 > 0) gg.flags |= SGS_GRADS_ACCUMULATE;  // later groups add to the first group's rows
    const bool a = acc || v0 > 0;
    if (P.n_lobes == 3) {
      if (a)
        preprocess_bwd_kernel<true, 3><<<grid, 128, 0, st>>>(P, V, gg);
      else
        preprocess_bwd_kernel<false, 3><<<grid, 128, 0, st>>>(P, V, gg);
    } else {
      if (a)
        preprocess_bwd_kernel<true, 0><<<grid, 128, 0, st>>>(P, V, gg);
      else
        preprocess_bwd_kernel<false, 0><<<grid, 128, 0, st>>>(P, V, gg);
    }
    SGS_LAUNCH_CHECK("preprocess_bwd_kernel");
  }
  return SGS_OK;
}

int launch_preprocess_bwd(const sgs_params& P, const SgsCam& cam, const float* grad2d, const sgs_grads& g,
                          cudaStream_t st) {
  int grid = persistent_grid((uint64_t)P.n, 128, 16);
  const bool acc = (g.flags & SGS_GRADS_ACCUMULATE) != 0;
  if (P.n_lobes == 3) {
    if (acc)
      preprocess_bwd_kernel1<true, 3><<<grid, 128, 0, st>>>(P, cam, grad2d, g);
    else
      preprocess_bwd_kernel1<false, 3><<<grid, 128, 0, st>>>(P, cam, grad2d, g);
  } else {
    if (acc)
      preprocess_bwd_kernel1<true, 0><<<grid, 128, 0, st>>>(P, cam, grad2d, g);
    else
      preprocess_bwd_kernel1<false, 0><<<grid, 128, 0, st>>>(P, cam, grad2d, g);
  }
  SGS_LAUNCH_CHECK("preprocess_bwd_kernel1");
  return SGS_OK;
}

}  // namespace sgs
