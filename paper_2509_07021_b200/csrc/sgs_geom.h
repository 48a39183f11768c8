// sgs_geom.h -- per-primitive preprocess math shared by the sm_100a kernels and
// the CPU tiled restatement under oracle/.
//
// Everything that decides a tile key, a sorted order, a per-tile range or a
// visibility count flows through this header: camera transform, EWA
// covariance projection, conic, the opacity-aware support radius, the tile
// rectangle and the exact ellipse-vs-tile test.  Bit-exactness between the
// GPU and the CPU restatement is guaranteed by construction:
//   * every operation is an explicitly IEEE-rounded primitive (F_MUL/F_ADD/
//     F_FMA ...): on the device these are the __f*_rn intrinsics, which ptxas
//     never contracts; on the host the oracle is compiled with
//     -ffp-contract=off and no fast-math, and fmaf is the correctly rounded
//     fused multiply-add;
//   * exp and log are evaluated by the polynomial restatements below (Cody-
//     Waite reduction + minimax polynomial), not by libdevice / glibc, whose
//     last-bit behaviour differs.
//
// Semantics follow the reference renderer:
//   _prepare            /root/reference/pkg/src/sgsplat/render.py:259-317
//   quat_to_rot         /root/reference/pkg/src/sgsplat/render.py:208-214
//   Camera/pixel model  /root/reference/pkg/src/sgsplat/render.py:30-76, 333-337
//   SG lobe color       /root/reference/pkg/src/sgsplat/render.py:298-305
//                       (independent form: sg.py:55-79 eval_sg_lobe/eval_color)
// The reference blends every visible primitive against every pixel (no
// spatial cutoff).  This build bins with the opacity-aware support
//   o_eff * exp(-q/2) >= SGS_EPS   <=>   q <= qmax = 2 (ln o_eff - ln SGS_EPS)
// with SGS_EPS = 1e-7, which SURVEY.md §0.4 measured at 2.1e-7 max-abs image
// error against the no-cutoff reference (the 3-sigma rule is 2.2e-3).
#pragma once

#include <stdint.h>
#include <math.h>
#include <string.h>

#if defined(__CUDACC__)
#define SGS_HD __host__ __device__ __forceinline__
#else
#define SGS_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define F_MUL(a, b) __fmul_rn((a), (b))
#define F_ADD(a, b) __fadd_rn((a), (b))
#define F_SUB(a, b) __fsub_rn((a), (b))
#define F_DIV(a, b) __fdiv_rn((a), (b))
#define F_SQRT(a) __fsqrt_rn((a))
#define F_FMA(a, b, c) __fmaf_rn((a), (b), (c))
#define F_RINT(a) rintf((a))
#define F_FLOOR(a) floorf((a))
#define D_MUL(a, b) __dmul_rn((a), (b))
#define D_ADD(a, b) __dadd_rn((a), (b))
#define D_SUB(a, b) __dsub_rn((a), (b))
#define D_DIV(a, b) __ddiv_rn((a), (b))
#define D_SQRT(a) __dsqrt_rn((a))
#else
#define F_MUL(a, b) ((float)(a) * (float)(b))
#define F_ADD(a, b) ((float)(a) + (float)(b))
#define F_SUB(a, b) ((float)(a) - (float)(b))
#define F_DIV(a, b) ((float)(a) / (float)(b))
#define F_SQRT(a) sqrtf((a))
#define F_FMA(a, b, c) fmaf((a), (b), (c))
#define F_RINT(a) rintf((a))
#define F_FLOOR(a) floorf((a))
#define D_MUL(a, b) ((double)(a) * (double)(b))
#define D_ADD(a, b) ((double)(a) + (double)(b))
#define D_SUB(a, b) ((double)(a) - (double)(b))
#define D_DIV(a, b) ((double)(a) / (double)(b))
#define D_SQRT(a) sqrt((double)(a))
#endif

#define SGS_TILE 16
#define SGS_ALPHA_MAX 0.99f      // render.py:24
#define SGS_T_CUTOFF 1e-4f       // render.py:25
// The fp32 blend step is  w = min(a, 0.99) T,  T_next = T - w  (the real
// value T (1 - alpha) of the reference's cumprod, render.py:374-384, in one
// FMUL + one FADD), and a primitive is kept iff T_next >= SGS_T_KEEP.  The
// reference keeps iff its float64 T_next >= 1e-4.  The common boundary is
// structural, not random: two alpha-clamped primitives give T = 0.01^2,
// which float64 rounds to 1.0000000000000018e-4 (kept) but this fp32 step to
// 9.999983e-5.  Lowering the fp32 threshold by a relative 2e-6 reproduces the
// float64 decision there; the price is a 2e-6-wide band where fp32 keeps what
// float64 drops, each such pair contributing <= 1e-4 |c|.
#define SGS_T_KEEP 9.99998e-5f
#define SGS_LOWPASS 0.3f         // render.py:26
#define SGS_EPS 1e-7f            // opacity-aware support threshold
#define SGS_LN_EPS (-16.11809565095832f)  // ln(1e-7)
#define SGS_LOG2E 1.4426950408889634f
#define SGS_MAX_LOBES 8

SGS_HD int min_i32_(int a, int b) { return a < b ? a : b; }

SGS_HD float sgs_bits_to_float(uint32_t u) {
#if defined(__CUDA_ARCH__)
  return __uint_as_float(u);
#else
  float f;
  memcpy(&f, &u, 4);
  return f;
#endif
}

SGS_HD uint32_t sgs_float_to_bits(float f) {
#if defined(__CUDA_ARCH__)
  return __float_as_uint(f);
#else
  uint32_t u;
  memcpy(&u, &f, 4);
  return u;
#endif
}

// exp(x): Cody-Waite reduction by ln2 (hi part has 9 significant bits so
// k*ln2_hi is exact), degree-6 polynomial on |r| <= ln2/2 (Cephes expf
// coefficients), then an exact power-of-two scale.
SGS_HD float sgs_expf(float x) {
  if (!(x == x)) return x;
  if (x > 88.72283f) return INFINITY;
  if (x < -103.97208f) return 0.0f;
  float kf = F_RINT(F_MUL(x, 1.44269504088896341f));
  float r = F_FMA(kf, -0.693359375f, x);
  r = F_FMA(kf, 2.12194440e-4f, r);
  float p = 1.9875691500e-4f;
  p = F_FMA(p, r, 1.3981999507e-3f);
  p = F_FMA(p, r, 8.3334519073e-3f);
  p = F_FMA(p, r, 4.1665795894e-2f);
  p = F_FMA(p, r, 1.6666665459e-1f);
  p = F_FMA(p, r, 5.0000001201e-1f);
  p = F_FMA(F_MUL(p, r), r, r);
  p = F_ADD(p, 1.0f);
  int k = (int)kf;
  if (k > 127) {
    p = F_MUL(p, 2.0f);
    k -= 1;
  }
  if (k < -125) {
    p = F_MUL(p, 5.421010862427522e-20f);  // 2^-64
    k += 64;
  }
  return F_MUL(p, sgs_bits_to_float((uint32_t)(k + 127) << 23));
}

// ln(x) for finite x > 0: split x = m * 2^e with m in [sqrt(1/2), sqrt(2)),
// f = m - 1 (exact), Cephes logf polynomial, ln2 in two parts.
SGS_HD float sgs_logf(float x) {
  if (!(x > 0.0f)) return (x == 0.0f) ? -INFINITY : NAN;
  if (x == INFINITY) return x;
  int e = 0;
  if (x < 1.17549435e-38f) {  // subnormal: scale into the normal range
    x = F_MUL(x, 8388608.0f);
    e = -23;
  }
  uint32_t bits = sgs_float_to_bits(x);
  e += (int)((bits >> 23) & 0xffu) - 127;
  float m = sgs_bits_to_float((bits & 0x007fffffu) | 0x3f800000u);
  if (m > 1.41421356f) {
    m = F_MUL(m, 0.5f);
    e += 1;
  }
  float f = F_SUB(m, 1.0f);
  float z = F_MUL(f, f);
  float y = 7.0376836292e-2f;
  y = F_FMA(y, f, -1.1514610310e-1f);
  y = F_FMA(y, f, 1.1676998740e-1f);
  y = F_FMA(y, f, -1.2420140846e-1f);
  y = F_FMA(y, f, 1.4249322787e-1f);
  y = F_FMA(y, f, -1.6668057665e-1f);
  y = F_FMA(y, f, 2.0000714765e-1f);
  y = F_FMA(y, f, -2.4999993993e-1f);
  y = F_FMA(y, f, 3.3333331174e-1f);
  y = F_MUL(F_MUL(y, f), z);
  float ef = (float)e;
  y = F_FMA(ef, -2.12194440e-4f, y);
  y = F_FMA(-0.5f, z, y);
  float r = F_ADD(f, y);
  return F_FMA(ef, 0.693359375f, r);
}

// Camera in the reference convention: rows of R are (right, down, forward),
// p_cam = R x + t, pixel = (fx x/z + cx, fy y/z + cy), pixel (row, col) has
// center (col + 0.5, row + 0.5).  C = -R^T t is the camera center.
typedef struct SgsCam {
  float R[9];
  float t[3];
  float C[3];
  float fx, fy, cx, cy;
  float near_z;
  int32_t width, height;
  int32_t tiles_x, tiles_y;
  int32_t tile_y0, tile_y1;  // tile-row window [y0, y1) for strip renders
  float lowpass;             // px^2 added to the cov2d diagonal (render.py:26, 285-286)
  double rz[3], tz;          // float64 depth row: z64 = (rz0 x + rz1 y) + rz2 z + tz (render.py:262)
  double near64;             // visible iff z64 > near64 (render.py:263)
  float grad_floor;          // binning opacity floor of gradient renders (sgs_camera.grad_floor)
} SgsCam;

// Projected primitive: everything the binning stage and the forward raster
// read.  conic/cov are the symmetric 2x2 (00, 01, 11) entries.
typedef struct SgsProj {
  float depth;       // float32 rounding of z64: the depth key (monotone in z64)
  float depth_res;   // z64 - depth, rounded: orders equal keys like z64 does
  float mx, my;
  float cov00, cov01, cov11;
  float con00, con01, con11;
  // eigen form of the same quadratic: q = t1^2 / lmax + t2^2 / lmin with
  // t1 = u . d, t2 = u x d (u = unit major axis of cov2d)
  float ux, uy, ilmax, ilmin;
  float o_eff;
  float ln_o;        // ln(max(o_eff, grad_floor)) (sgs_logf): the support, valid when emits
  float ln_oe;       // ln(o_eff): the blend (-inf at o_eff = 0)
  float qmax;
  int32_t tx0, ty0, tx1, ty1;
  int32_t visible;   // z > near (render.py:263)
  int32_t emits;     // visible, o_eff > eps, support rectangle on the image
} SgsProj;

// render.py:208-214, w-first unit quaternion -> rotation matrix rows.
SGS_HD void sgs_quat_to_rot(float w, float x, float y, float z, float R[9]) {
  float xx = F_MUL(x, x), yy = F_MUL(y, y), zz = F_MUL(z, z);
  float xy = F_MUL(x, y), xz = F_MUL(x, z), yz = F_MUL(y, z);
  float wx = F_MUL(w, x), wy = F_MUL(w, y), wz = F_MUL(w, z);
  R[0] = F_SUB(1.0f, F_MUL(2.0f, F_ADD(yy, zz)));
  R[1] = F_MUL(2.0f, F_SUB(xy, wz));
  R[2] = F_MUL(2.0f, F_ADD(xz, wy));
  R[3] = F_MUL(2.0f, F_ADD(xy, wz));
  R[4] = F_SUB(1.0f, F_MUL(2.0f, F_ADD(xx, zz)));
  R[5] = F_MUL(2.0f, F_SUB(yz, wx));
  R[6] = F_MUL(2.0f, F_SUB(xz, wy));
  R[7] = F_MUL(2.0f, F_ADD(yz, wx));
  R[8] = F_SUB(1.0f, F_MUL(2.0f, F_ADD(xx, yy)));
}

SGS_HD float sgs_dot3(float a0, float a1, float a2, float b0, float b1, float b2) {
  return F_ADD(F_ADD(F_MUL(a0, b0), F_MUL(a1, b1)), F_MUL(a2, b2));
}

// Camera-space depth: float32 z (float32 camera, for the projection) and
// float64 z64 from the caller's float64 camera row -- the reference orders by
// its float64 z (render.py:307), which the float32 z does not reproduce for
// near-ties.  Returns visibility, z64 > near (render.py:263).
SGS_HD int sgs_depth(const float pos[3], const SgsCam* cam, float* z, double* z64) {
  const float* W = cam->R;
  *z = F_ADD(sgs_dot3(W[6], W[7], W[8], pos[0], pos[1], pos[2]), cam->t[2]);
  *z64 = D_ADD(D_ADD(D_ADD(D_MUL(cam->rz[0], (double)pos[0]), D_MUL(cam->rz[1], (double)pos[1])),
                     D_MUL(cam->rz[2], (double)pos[2])),
               cam->tz);
  return *z64 > cam->near64 && *z > 0.0f;
}

// Geometry of one primitive (render.py:262-292 plus the support rectangle).
SGS_HD void sgs_project(const float pos[3], const float quat[4], const float ls[3],
                        float opacity, float pmask, const SgsCam* cam, SgsProj* o) {
  const float* W = cam->R;
  float x = F_ADD(sgs_dot3(W[0], W[1], W[2], pos[0], pos[1], pos[2]), cam->t[0]);
  float y = F_ADD(sgs_dot3(W[3], W[4], W[5], pos[0], pos[1], pos[2]), cam->t[1]);
  float z;
  double z64;
  o->visible = sgs_depth(pos, cam, &z, &z64);
  o->depth = (float)z64;
  o->depth_res = (float)D_SUB(z64, (double)o->depth);
  o->emits = 0;
  o->tx0 = o->ty0 = 0;
  o->tx1 = o->ty1 = -1;
  if (!o->visible) return;

  // one IEEE reciprocal per divisor, then products (the CPU restatement
  // performs the identical sequence, so results stay bit-identical)
  float iz = F_DIV(1.0f, z);
  o->mx = F_ADD(F_MUL(F_MUL(cam->fx, x), iz), cam->cx);
  o->my = F_ADD(F_MUL(F_MUL(cam->fy, y), iz), cam->cy);

  // Sigma = R diag(exp(2 ls)) R^T
  float qn = F_SQRT(F_ADD(F_ADD(F_ADD(F_MUL(quat[0], quat[0]), F_MUL(quat[1], quat[1])),
                                F_MUL(quat[2], quat[2])), F_MUL(quat[3], quat[3])));
  float R[9];
  float iq = F_DIV(1.0f, qn);
  sgs_quat_to_rot(F_MUL(quat[0], iq), F_MUL(quat[1], iq), F_MUL(quat[2], iq), F_MUL(quat[3], iq), R);
  float D0 = sgs_expf(F_MUL(2.0f, ls[0]));
  float D1 = sgs_expf(F_MUL(2.0f, ls[1]));
  float D2 = sgs_expf(F_MUL(2.0f, ls[2]));
  double S[9];
  for (int i = 0; i < 3; ++i)
    for (int k = i; k < 3; ++k) {
      double s = D_ADD(D_ADD(D_MUL(D_MUL((double)R[3 * i + 0], (double)D0), (double)R[3 * k + 0]),
                             D_MUL(D_MUL((double)R[3 * i + 1], (double)D1), (double)R[3 * k + 1])),
                       D_MUL(D_MUL((double)R[3 * i + 2], (double)D2), (double)R[3 * k + 2]));
      S[3 * i + k] = s;
      S[3 * k + i] = s;
    }

  // J (render.py:278-282), M = J W, cov2d = M Sigma M^T + lowpass I and its
  // inverse are formed in float64: for elongated splats cov2d is nearly
  // singular before the low-pass floor, and float32 cancellation there would
  // cost ~1e-5 relative in the small eigenvalue.
  const double dz = (double)z, dx_ = (double)x, dy_ = (double)y;
  const double diz = D_DIV(1.0, dz), diz2 = D_MUL(diz, diz);
  const double J00 = D_MUL((double)cam->fx, diz);
  const double J02 = -D_MUL(D_MUL((double)cam->fx, dx_), diz2);
  const double J11 = D_MUL((double)cam->fy, diz);
  const double J12 = -D_MUL(D_MUL((double)cam->fy, dy_), diz2);
  double M0[3], M1[3];
  for (int k = 0; k < 3; ++k) {
    M0[k] = D_ADD(D_MUL(J00, (double)W[k]), D_MUL(J02, (double)W[6 + k]));
    M1[k] = D_ADD(D_MUL(J11, (double)W[3 + k]), D_MUL(J12, (double)W[6 + k]));
  }
  double T0[3], T1[3];
  for (int k = 0; k < 3; ++k) {
    T0[k] = D_ADD(D_ADD(D_MUL(M0[0], S[k]), D_MUL(M0[1], S[3 + k])), D_MUL(M0[2], S[6 + k]));
    T1[k] = D_ADD(D_ADD(D_MUL(M1[0], S[k]), D_MUL(M1[1], S[3 + k])), D_MUL(M1[2], S[6 + k]));
  }
  const double lp = (double)cam->lowpass;
  const double a = D_ADD(D_ADD(D_ADD(D_MUL(T0[0], M0[0]), D_MUL(T0[1], M0[1])), D_MUL(T0[2], M0[2])), lp);
  const double b = D_ADD(D_ADD(D_MUL(T0[0], M1[0]), D_MUL(T0[1], M1[1])), D_MUL(T0[2], M1[2]));
  const double c = D_ADD(D_ADD(D_ADD(D_MUL(T1[0], M1[0]), D_MUL(T1[1], M1[1])), D_MUL(T1[2], M1[2])), lp);
  o->cov00 = (float)a;
  o->cov01 = (float)b;
  o->cov11 = (float)c;
  const double det = D_SUB(D_MUL(a, c), D_MUL(b, b));
  const double idet = D_DIV(1.0, det);
  o->con00 = (float)D_MUL(c, idet);
  o->con01 = (float)(-D_MUL(b, idet));
  o->con11 = (float)D_MUL(a, idet);
  {
    // eigen decomposition of cov2d (PD): lmax = m + r, lmin = det / lmax,
    // major axis from whichever of (b, lmax - a), (lmax - c, b) is longer
    const double m = D_MUL(0.5, D_ADD(a, c));
    const double h = D_MUL(0.5, D_SUB(a, c));
    const double r = D_SQRT(D_ADD(D_MUL(h, h), D_MUL(b, b)));
    const double lmax = D_ADD(m, r);
    const double lmin = D_DIV(det, lmax);
    double ex = b, ey = D_SUB(lmax, a);
    const double fx2 = D_SUB(lmax, c), fy2 = b;
    if (D_ADD(D_MUL(fx2, fx2), D_MUL(fy2, fy2)) > D_ADD(D_MUL(ex, ex), D_MUL(ey, ey))) {
      ex = fx2;
      ey = fy2;
    }
    const double en = D_SQRT(D_ADD(D_MUL(ex, ex), D_MUL(ey, ey)));
    if (en > 0.0) {
      o->ux = (float)D_DIV(ex, en);
      o->uy = (float)D_DIV(ey, en);
    } else {  // isotropic: any axis
      o->ux = 1.0f;
      o->uy = 0.0f;
    }
    o->ilmax = (float)D_DIV(1.0, lmax);
    o->ilmin = (float)D_DIV(1.0, lmin);
  }
  float oe = F_MUL(opacity, pmask);
  o->o_eff = oe;
  const float ob = oe > cam->grad_floor ? oe : cam->grad_floor;  // support opacity
  if (!(ob > SGS_EPS) || !(det > 0.0)) {
    o->qmax = 0.0f;
    return;
  }
  o->ln_o = sgs_logf(ob);
  o->ln_oe = ob == oe ? o->ln_o : sgs_logf(oe);
  float qmax = F_MUL(2.0f, F_SUB(o->ln_o, SGS_LN_EPS));
  o->qmax = qmax;
  // exact bounding box of {d : d^T cov^-1 d <= qmax} is sqrt(qmax * cov_ii)
  float rx = F_SQRT(F_MUL(qmax, o->cov00));
  float ry = F_SQRT(F_MUL(qmax, o->cov11));
  float x0 = F_SUB(o->mx, rx), x1 = F_ADD(o->mx, rx);
  float y0 = F_SUB(o->my, ry), y1 = F_ADD(o->my, ry);
  if (!(x1 > 0.0f && x0 < (float)cam->width && y1 > 0.0f && y0 < (float)cam->height)) return;
  const float inv_tile = 1.0f / SGS_TILE;
  float ftx0 = F_FLOOR(F_MUL(x0, inv_tile)), ftx1 = F_FLOOR(F_MUL(x1, inv_tile));
  float fty0 = F_FLOOR(F_MUL(y0, inv_tile)), fty1 = F_FLOOR(F_MUL(y1, inv_tile));
  float mxx = (float)(cam->tiles_x - 1);
  ftx0 = fminf(fmaxf(ftx0, 0.0f), mxx);
  ftx1 = fminf(fmaxf(ftx1, 0.0f), mxx);
  fty0 = fminf(fmaxf(fty0, (float)cam->tile_y0), (float)(cam->tile_y1 - 1));
  fty1 = fminf(fmaxf(fty1, (float)cam->tile_y0), (float)(cam->tile_y1 - 1));
  if (!(y1 > (float)(cam->tile_y0 * SGS_TILE) && y0 < (float)(cam->tile_y1 * SGS_TILE))) return;
  o->tx0 = (int32_t)ftx0;
  o->tx1 = (int32_t)ftx1;
  o->ty0 = (int32_t)fty0;
  o->ty1 = (int32_t)fty1;
  o->emits = 1;
}

// Support shape of one packed record (see sgs_pack_geo): the ellipse
//   E = {(dx, dy) : A dx^2 + B dx dy + C dy^2 >= pmin},  A, C < 0, 4AC > B^2,
// with (dx, dy) = pixel center - mean.  Its x-extreme points lie on the line
// dy = kx dx, its y-extremes on dx = ky dy; xm / ym are the half extents.
typedef struct SgsSpan {
  float mx, my;
  float kx, xm, ym, i2a;  // i2a = 1 / (2 A)
  // crossing of the boundary with the line dy:  A x^2 + B dy x + (C dy^2 - pmin) = 0
  //   x = kb dy -/+ sqrt(Q - D dy^2) i2a,  kb = -B i2a,  D = 4AC - B^2,  Q = 4A pmin
  float kb, D, Q;
  int valid;
} SgsSpan;

SGS_HD SgsSpan sgs_span_from(float mx, float my, float A, float B, float C, float pmin) {
  SgsSpan s;
  s.mx = mx;
  s.my = my;
  // D = 4AC - B^2 > 0 for a negative-definite form
  const float D = F_SUB(F_MUL(F_MUL(4.0f, A), C), F_MUL(B, B));
  s.valid = D > 0.0f && A < 0.0f && C < 0.0f && pmin < 0.0f;
  s.kx = -F_DIV(B, F_MUL(2.0f, C));
  const float iD = F_DIV(1.0f, D);
  s.xm = s.valid ? F_SQRT(F_MUL(F_MUL(F_MUL(4.0f, C), pmin), iD)) : 0.0f;
  s.ym = s.valid ? F_SQRT(F_MUL(F_MUL(F_MUL(4.0f, A), pmin), iD)) : 0.0f;
  s.i2a = F_DIV(1.0f, F_MUL(2.0f, A));
  s.kb = F_MUL(-B, s.i2a);
  s.D = D;
  s.Q = F_MUL(F_MUL(4.0f, A), pmin);
  return s;
}

SGS_HD SgsSpan sgs_span(const float geo[4], const float con[4]) {
  return sgs_span_from(geo[0], geo[1], con[0], con[1], con[2], geo[3]);
}

// The span parameters are cached per primitive by the preprocess: kx in the
// conic record's 4th slot, (xm, ym, i2a) in rec_span (xm < 0 marks an invalid
// form); kb, D, Q are recomputed from the conic with the same operations.
// Rebuilding SgsSpan from the cache is bit-identical to sgs_span.
SGS_HD void sgs_span_cache(const SgsSpan* s, float* kx, float span2[3]) {
  *kx = s->kx;
  span2[0] = s->valid ? s->xm : -1.0f;
  span2[1] = s->ym;
  span2[2] = s->i2a;
}

SGS_HD SgsSpan sgs_span_cached(const float geo[4], const float con[4], const float span2[3]) {
  SgsSpan s;
  s.mx = geo[0];
  s.my = geo[1];
  s.kx = con[3];
  s.valid = span2[0] >= 0.0f;
  s.xm = s.valid ? span2[0] : 0.0f;
  s.ym = span2[1];
  s.i2a = span2[2];
  s.kb = F_MUL(-con[1], s.i2a);
  s.D = F_SUB(F_MUL(F_MUL(4.0f, con[0]), con[2]), F_MUL(con[1], con[1]));
  s.Q = F_MUL(F_MUL(4.0f, con[0]), geo[3]);
  return s;
}

// x where the ellipse boundary crosses the horizontal line dy (the larger root
// when `right`, else the smaller); the caller guarantees |dy| <= ym up to
// rounding, and a slightly negative discriminant is clamped to 0.
SGS_HD float sgs_span_root(const SgsSpan* s, float dy, int right) {
  const float disc = F_FMA(-s->D, F_MUL(dy, dy), s->Q);
  const float ri = F_MUL(F_SQRT(fmaxf(disc, 0.0f)), s->i2a);
  // i2a < 0: kb dy - r i2a is the larger root
  return F_FMA(s->kb, dy, right ? -ri : ri);
}

// Tiles of tile-row `ty` (clipped to [tx0, tx1]) whose pixel-center box meets
// the support: the ellipse's x-interval over the row's pixel-center band
// [yc0, yc1] is exact -- its right end is the ellipse's rightmost point when
// that lies inside the band, else the crossing at the band edge nearest to
// it (likewise on the left) -- and tile tx is hit iff its pixel-center
// columns [16 tx + 0.5, 16 tx + 15.5] meet that interval.  One definition
// serves the tile counts (preprocess), the emission (binning) and the CPU
// oracle, so counts, keys and ranges agree bit for bit.  Returns the count
// and the first hit column.
SGS_HD int sgs_row_span(const SgsSpan* s, const SgsCam* cam, int ty, int tx0, int tx1, int* first) {
  // Branch-free: both crossings are always evaluated and the early outs are
  // folded into `hit`, so the lanes of a warp never diverge here.  The values
  // selected are exactly those of the branching definition above.
  const float yc0 = (float)(ty * SGS_TILE) + 0.5f;
  const float yc1 = (float)min_i32_(ty * SGS_TILE + SGS_TILE - 1, cam->height - 1) + 0.5f;
  const float dy0 = F_SUB(yc0, s->my), dy1 = F_SUB(yc1, s->my);
  int hit = s->valid && !(dy1 < -s->ym || dy0 > s->ym);
  const float dyr = F_MUL(s->kx, s->xm);  // dy of the rightmost point; leftmost is at -dyr
  const float dyl = -dyr;
  const int rin = dyr >= dy0 && dyr <= dy1;
  const int lin = dyl >= dy0 && dyl <= dy1;
  const float rr = sgs_span_root(s, dyr < dy0 ? dy0 : dy1, 1);
  const float rl = sgs_span_root(s, dyl < dy0 ? dy0 : dy1, 0);
  const float xr = rin ? s->xm : rr;
  const float xl = lin ? -s->xm : rl;
  const float XL = F_ADD(s->mx, xl), XR = F_ADD(s->mx, xr);
  hit = hit && (XR >= 0.5f && XL <= (float)cam->width - 0.5f && XL <= XR);
  const float inv_tile = 1.0f / SGS_TILE;
  const float flo = ceilf(F_MUL(F_SUB(XL, 15.5f), inv_tile));
  const float fhi = F_FLOOR(F_MUL(F_SUB(XR, 0.5f), inv_tile));
  // clamp to [tx0, tx1 + 1] / [tx0 - 1, tx1] before converting (integral
  // floats, so identical to clamping after; NaN-safe via fmin/fmax)
  const int lo = (int)fminf(fmaxf(flo, (float)tx0), (float)tx1 + 1.0f);
  const int hi = (int)fmaxf(fminf(fhi, (float)tx1), (float)tx0 - 1.0f);
  hit = hit && hi >= lo;
  *first = hit ? lo : 0;
  return hit ? hi - lo + 1 : 0;
}

// Number of tiles whose box meets the support, over the rectangle rows.
SGS_HD uint32_t sgs_count_tiles(int tx0, int ty0, int tx1, int ty1, const float geo[4], const float con[4],
                                const SgsCam* cam) {
  SgsSpan s = sgs_span(geo, con);
  uint32_t n = 0;
  int first;
  for (int ty = ty0; ty <= ty1; ++ty) n += (uint32_t)sgs_row_span(&s, cam, ty, tx0, tx1, &first);
  return n;
}

// Super-tiles: SGS_SUPER x SGS_SUPER tiles (64 x 64 px).  The depth-first
// binning sorts (super-tile, primitive) entries -- about a tenth of the
// (tile, primitive) entries -- and the raster filters each super-tile list
// down to its own tile with the exact per-tile test above, so the per-tile
// lists (and everything downstream) are identical to sorting tile entries.
// A primitive's super-tile set: for each super row, the super columns
// spanned by [min, max] of its tile rows' spans -- a superset of the super
// tiles that contain a hit tile, built from the same per-row spans, so no
// tile hit can be lost to rounding.
#define SGS_SUPER 4

// Super row `sr` with its tile rows' spans (first[r], cnt[r]), r = ty - 4 sr
// (cnt = 0 outside the rectangle), for the per-entry tile masks.
SGS_HD int sgs_super_row_spans(const SgsSpan* s, const SgsCam* cam, int tx0, int ty0, int tx1, int ty1, int sr,
                               int first[SGS_SUPER], int cnt[SGS_SUPER], int* first_sc) {
  int lo = 0x7fffffff, hi = -1;
  for (int r = 0; r < SGS_SUPER; ++r) {
    // rows outside the rectangle are evaluated on a clamped row and masked
    // (no divergence); their count is 0
    const int ty = sr * SGS_SUPER + r;
    const int in = ty >= ty0 && ty <= ty1;
    int f;
    const int c = sgs_row_span(s, cam, in ? ty : ty0, tx0, tx1, &f);
    first[r] = in ? f : 0;
    cnt[r] = in ? c : 0;
    if (cnt[r] > 0) {
      const int a = first[r] / SGS_SUPER, b = (first[r] + cnt[r] - 1) / SGS_SUPER;
      lo = a < lo ? a : lo;
      hi = b > hi ? b : hi;
    }
  }
  *first_sc = hi >= lo ? lo : 0;
  return hi >= lo ? hi - lo + 1 : 0;
}

// 16-bit membership mask of super-tile column sc: bit (r * 4 + c) set iff
// tile (4 sc + c, 4 sr + r) is in the primitive's tile set.
SGS_HD uint32_t sgs_super_mask(const int first[SGS_SUPER], const int cnt[SGS_SUPER], int sc) {
  uint32_t m = 0;
  for (int r = 0; r < SGS_SUPER; ++r)
    for (int c = 0; c < SGS_SUPER; ++c) {
      const int tx = sc * SGS_SUPER + c;
      if (tx >= first[r] && tx < first[r] + cnt[r]) m |= 1u << (r * SGS_SUPER + c);
    }
  return m;
}

// sgs_super_mask with per-row bit arithmetic (same value): row r's members
// are tile columns [max(first, 4 sc), min(first + cnt, 4 sc + 4)) of the
// super column, a run of bits ((1 << hi) - (1 << lo)) in nibble r.
SGS_HD uint32_t sgs_super_mask_fast(const int first[SGS_SUPER], const int cnt[SGS_SUPER], int sc) {
  uint32_t m = 0;
  const int x0 = sc * SGS_SUPER;
  for (int r = 0; r < SGS_SUPER; ++r) {
    int lo = first[r] - x0, hi = first[r] + cnt[r] - x0;
    lo = lo < 0 ? 0 : lo;
    hi = hi > SGS_SUPER ? SGS_SUPER : hi;
    const uint32_t run = hi > lo ? (1u << hi) - (1u << lo) : 0u;
    m |= run << (r * SGS_SUPER);
  }
  return m;
}

// SG color for the camera-to-center view direction (render.py:294-305):
//   c_pre = diffuse + sum_l m_l a_l exp(s_l (mu_l . v - 1)),  c = max(c_pre, 0)
// Lobes with mask exactly 0 are skipped (bit-identical to multiplying by 0).
SGS_HD void sgs_color(const float pos[3], const float diffuse[3], const float* axis,
                      const float* sharp, const float* amp, const float* lmask, int L,
                      const SgsCam* cam, float c_pre[3], float c[3]) {
  float d0 = F_SUB(pos[0], cam->C[0]), d1 = F_SUB(pos[1], cam->C[1]), d2 = F_SUB(pos[2], cam->C[2]);
  float r = F_SQRT(sgs_dot3(d0, d1, d2, d0, d1, d2));
  float ir = F_DIV(1.0f, r);
  float v0 = F_MUL(d0, ir), v1 = F_MUL(d1, ir), v2 = F_MUL(d2, ir);
  float acc0 = 0.0f, acc1 = 0.0f, acc2 = 0.0f;
  for (int l = 0; l < L; ++l) {
    float m = lmask[l];
    if (m == 0.0f) continue;
    const float* u = axis + 3 * l;
    float un = F_SQRT(sgs_dot3(u[0], u[1], u[2], u[0], u[1], u[2]));
    float iun = F_DIV(1.0f, un);
    float dot = sgs_dot3(F_MUL(u[0], iun), F_MUL(u[1], iun), F_MUL(u[2], iun), v0, v1, v2);
    float e = F_MUL(sgs_expf(F_MUL(sharp[l], F_SUB(dot, 1.0f))), m);
    acc0 = F_ADD(acc0, F_MUL(e, amp[3 * l + 0]));
    acc1 = F_ADD(acc1, F_MUL(e, amp[3 * l + 1]));
    acc2 = F_ADD(acc2, F_MUL(e, amp[3 * l + 2]));
  }
  c_pre[0] = F_ADD(diffuse[0], acc0);
  c_pre[1] = F_ADD(diffuse[1], acc1);
  c_pre[2] = F_ADD(diffuse[2], acc2);
  c[0] = fmaxf(c_pre[0], 0.0f);
  c[1] = fmaxf(c_pre[1], 0.0f);
  c[2] = fmaxf(c_pre[2], 0.0f);
}

// Raster record packing.  The binning stage reads
//   geo = (mx, my, lo, pmin), con = (A, B, C, kx)
// where p2 = A dx^2 + B dx dy + C dy^2 (= -q/2 * log2 e) and pmin = -qmax/2 *
// log2 e bound the support (sgs_span).  The rasterizers evaluate the same
// quadratic in a scaled eigen form, with the opacity folded in:
//   eig = (s1 ux, s1 uy, s2 ux, s2 uy),  s_i = sqrt(log2(e) / (2 l_i)),
//   t1 = s1 (ux dx + uy dy),  t2 = s2 (ux dy - uy dx),
//   p  = lo - t1^2 - t2^2 = log2(o_eff G),   alpha = min(2^p, 0.99),
// with lo = log2(o_eff).  Every term is <= 0, so there is no cancellation for
// elongated splats, and the support test o_eff G >= SGS_EPS is the constant
// comparison p >= SGS_LOG2_EPS.
#define SGS_LOG2_EPS (-23.253496664211536f)  // log2(1e-7)

SGS_HD void sgs_pack_eig(const SgsProj* p, float eig[4]) {
  const float k = 0.5f * SGS_LOG2E;
  const float s1 = F_SQRT(F_MUL(k, p->ilmax));
  const float s2 = F_SQRT(F_MUL(k, p->ilmin));
  eig[0] = F_MUL(s1, p->ux);
  eig[1] = F_MUL(s1, p->uy);
  eig[2] = F_MUL(s2, p->ux);
  eig[3] = F_MUL(s2, p->uy);
}

SGS_HD void sgs_pack_geo(const SgsProj* p, float geo[4], float con[4]) {
  const float k = -0.5f * SGS_LOG2E;
  geo[0] = p->mx;
  geo[1] = p->my;
  geo[2] = F_MUL(p->ln_oe, SGS_LOG2E);  // blend: log2 o_eff (-inf at 0); geo[3] holds the support
  geo[3] = F_MUL(k, p->qmax);
  con[0] = F_MUL(k, p->con00);
  con[1] = F_MUL(2.0f * k, p->con01);
  con[2] = F_MUL(k, p->con11);
  con[3] = 0.0f;  // replaced by the span cache's kx (sgs_span_cache)
}
