// loss.cu -- fused image loss: (1 - lambda) L1 + lambda (1 - SSIM) and its
// exact gradient with respect to the image, replacing the reference's
// _ssim_terms / _ssim_grad / _loss_and_dimg
// (/root/reference/pkg/src/sgsplat/render.py:446-509).
//
// Semantics (render.py:433-466): per channel, the five local statistics
// mu_x, mu_y, E[xx], E[yy], E[xy] are the separable correlation of the
// planes with a normalised Gaussian window (zero padding outside the image);
//   A1 = 2 mu_x mu_y + c1,  A2 = 2 (E[xy] - mu_x mu_y) + c2,
//   B1 = mu_x^2 + mu_y^2 + c1,  B2 = (E[xx] - mu_x^2) + (E[yy] - mu_y^2) + c2,
//   S = A1 A2 / (B1 B2),  loss = (1-l) mean|x - y| + l (1 - mean S),
// means over all H*W*3 values.  The gradient (render.py:469-486) is
//   dS/dx = [G*(dmu) + 2 x G*(dB2) + y G*(2 dA2)] / size
// with dA1 = A2/(B1 B2), dA2 = A1/(B1 B2), dB1 = -S/B1, dB2 = -S/B2,
// dmu = 2 mu_y dA1 + 2 mu_x dB1 - 2 mu_x dB2 - 2 mu_y dA2, and the L1 term
// (1-l) sign(x - y) / size (np.sign: 0 at 0).
//
// Two tiled kernels, 32x32 output pixels per CTA (512 threads, two
// vertically adjacent outputs each; the horizontal passes compute two
// adjacent columns per item, so loaded values feed two windows), one channel
// at a time: the
// forward stages the (8+2r) x (32+2r) halo of x and y in shared memory as
// float64, filters rows then columns (all five statistics at once), writes
// the three per-pixel float64 derivative planes (dmu, dB2, 2 dA2) and reduces the L1
// and SSIM sums; the backward filters those planes the same way and forms
// dL/dimg.  Statistics are accumulated in float64 (E[xx] - mu^2 cancels in
// flat regions; B200 runs FP64 at half the FP32 rate), so results agree with
// the float64 reference to rounding.  Inputs may be float32 or float64.
#include "common.cuh"

namespace sgs {

#ifndef SGS_LOSS_TH
#define SGS_LOSS_TH 16
#endif
#ifndef SGS_LOSS_MIN_BLOCKS
#define SGS_LOSS_MIN_BLOCKS 2
#endif
// each thread owns kLossRows vertically adjacent outputs of a column
constexpr int kLossRows = 2;
constexpr int kLossTW = 32, kLossTH = SGS_LOSS_TH * kLossRows, kLossThreads = kLossTW * SGS_LOSS_TH;
constexpr int kMaxWindow = 31;

struct LossParams {
  double w[kMaxWindow];
  int r;
  int H, W;
  double lam, c1, c2, inv_size;
};

template <typename T>
__device__ __forceinline__ double ld(const T* p, size_t i) {
  return (double)p[i];
}

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kLossThreads / 32; ++i) s += red[i];
  return s;
}

// Each block writes its sums of the loss terms to its own slot (part[2 b],
// part[2 b + 1]); loss_finish_kernel adds the slots in a fixed order, so the
// loss value is bitwise reproducible (a float atomicAdd per block would
// depend on which block lands first).

// Shared layout (doubles): sx, sy [(TH+2r) x (TW+2r)], then hs[5][(TH+2r) x TW].
__host__ __device__ inline size_t loss_smem_doubles(int r, int nplanes_in, int nplanes_h) {
  return (size_t)nplanes_in * (kLossTH + 2 * r) * (kLossTW + 2 * r) + (size_t)nplanes_h * (kLossTH + 2 * r) * kLossTW;
}

// R > 0: the window radius as a compile-time constant (the default 11-tap
// window, R = 5: unrolled taps, weights as constant-bank immediates, halo
// index arithmetic by constants); R = 0 reads it from P.
template <typename TI, typename TT, int R>
__global__ void __launch_bounds__(kLossThreads, SGS_LOSS_MIN_BLOCKS) ssim_fwd_kernel(const TI* __restrict__ img, const TT* __restrict__ tgt,
                                                                LossParams P, double* __restrict__ dmu,
                                                                double* __restrict__ dxx, double* __restrict__ dxy,
                                                                double* __restrict__ smap, double* __restrict__ sums) {
  extern __shared__ double sh[];
  __shared__ double red[kLossThreads / 32];
  const int r = R > 0 ? R : P.r, HW = kLossTW + 2 * r, HH = kLossTH + 2 * r;
  double* sx = sh;
  double* sy = sx + HH * HW;
  double* hs = sy + HH * HW;  // 5 planes of HH x TW
  const int x0 = blockIdx.x * kLossTW, y0 = blockIdx.y * kLossTH;
  const int t = threadIdx.x;
  const int ox = t % kLossTW, oy0 = (t / kLossTW) * kLossRows;
  const int px = x0 + ox;
  double l1 = 0.0, ss = 0.0;
  for (int c = 0; c < 3; ++c) {
    for (int i = t; i < HH * HW; i += kLossThreads) {
      const int yy = y0 - r + i / HW, xx = x0 - r + i % HW;
      const bool in = yy >= 0 && yy < P.H && xx >= 0 && xx < P.W;
      const size_t g = ((size_t)yy * P.W + xx) * 3 + c;
      sx[i] = in ? ld(img, g) : 0.0;
      sy[i] = in ? ld(tgt, g) : 0.0;
    }
    __syncthreads();
    // two adjacent output columns per item: each loaded input (and its
    // products) feeds both windows
    for (int i = t; i < HH * (kLossTW / 2); i += kLossThreads) {
      const int row = i / (kLossTW / 2), col = 2 * (i % (kLossTW / 2));
      double a0 = 0, b0 = 0, aa0 = 0, bb0 = 0, ab0 = 0, a1 = 0, b1 = 0, aa1 = 0, bb1 = 0, ab1 = 0;
      #pragma unroll
      for (int k = 0; k <= 2 * r + 1; ++k) {
        const double u = sx[row * HW + col + k], v = sy[row * HW + col + k];
        const double uu = u * u, vv = v * v, uv = u * v;
        if (k <= 2 * r) {
          const double wx = P.w[k];
          a0 = fma(wx, u, a0);
          b0 = fma(wx, v, b0);
          aa0 = fma(wx, uu, aa0);
          bb0 = fma(wx, vv, bb0);
          ab0 = fma(wx, uv, ab0);
        }
        if (k >= 1) {
          const double wx = P.w[k - 1];
          a1 = fma(wx, u, a1);
          b1 = fma(wx, v, b1);
          aa1 = fma(wx, uu, aa1);
          bb1 = fma(wx, vv, bb1);
          ab1 = fma(wx, uv, ab1);
        }
      }
      const int o = row * kLossTW + col;
      hs[o] = a0;
      hs[o + 1] = a1;
      hs[HH * kLossTW + o] = b0;
      hs[HH * kLossTW + o + 1] = b1;
      hs[2 * HH * kLossTW + o] = aa0;
      hs[2 * HH * kLossTW + o + 1] = aa1;
      hs[3 * HH * kLossTW + o] = bb0;
      hs[3 * HH * kLossTW + o + 1] = bb1;
      hs[4 * HH * kLossTW + o] = ab0;
      hs[4 * HH * kLossTW + o + 1] = ab1;
    }
    __syncthreads();
    {
      // the thread's kLossRows outputs share their column's loads
      double m[kLossRows][5] = {};
      #pragma unroll
      for (int k = 0; k < 2 * r + kLossRows; ++k) {
        const int o = (oy0 + k) * kLossTW + ox;
        const double h0 = hs[o], h1 = hs[HH * kLossTW + o], h2 = hs[2 * HH * kLossTW + o],
                     h3 = hs[3 * HH * kLossTW + o], h4 = hs[4 * HH * kLossTW + o];
        #pragma unroll
        for (int q = 0; q < kLossRows; ++q) {
          if (k - q < 0 || k - q > 2 * r) continue;
          const double wy = P.w[k - q];
          m[q][0] = fma(wy, h0, m[q][0]);
          m[q][1] = fma(wy, h1, m[q][1]);
          m[q][2] = fma(wy, h2, m[q][2]);
          m[q][3] = fma(wy, h3, m[q][3]);
          m[q][4] = fma(wy, h4, m[q][4]);
        }
      }
      #pragma unroll
      for (int q = 0; q < kLossRows; ++q) {
        const int oy = oy0 + q, py = y0 + oy;
        if (px >= P.W || py >= P.H) continue;
        const double mx = m[q][0], my = m[q][1], mxx = m[q][2], myy = m[q][3], mxy = m[q][4];
        const double sxv = mxx - mx * mx, syv = myy - my * my, sxy = mxy - mx * my;
        const double A1 = 2.0 * mx * my + P.c1, A2 = 2.0 * sxy + P.c2;
        const double B1 = mx * mx + my * my + P.c1, B2 = sxv + syv + P.c2;
        const double inv = 1.0 / (B1 * B2);
        const double S = A1 * A2 * inv;
        // 1 / B1 = B2 inv, 1 / B2 = B1 inv: one division
        const double dA1 = A2 * inv, dA2 = A1 * inv, dB1 = -S * (B2 * inv), dB2 = -S * (B1 * inv);
        const size_t g = ((size_t)py * P.W + px) * 3 + c;
        dmu[g] = 2.0 * my * dA1 + 2.0 * mx * dB1 - 2.0 * mx * dB2 - 2.0 * my * dA2;
        dxx[g] = dB2;
        dxy[g] = 2.0 * dA2;
        if (smap) smap[g] = S;
        const double xv = sx[(oy + r) * HW + ox + r], yv = sy[(oy + r) * HW + ox + r];
        l1 += fabs(xv - yv);
        ss += S;
      }
    }
    __syncthreads();
  }
  const double tl1 = block_sum(l1, red);
  const double tss = block_sum(ss, red);
  if (t == 0) {
    const size_t b = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
    sums[2 * b] = tl1;
    sums[2 * b + 1] = tss;
  }
}

template <typename TI, typename TT, int R>
__global__ void __launch_bounds__(kLossThreads, SGS_LOSS_MIN_BLOCKS) ssim_bwd_kernel(const TI* __restrict__ img, const TT* __restrict__ tgt,
                                                                LossParams P, const double* __restrict__ dmu,
                                                                const double* __restrict__ dxx,
                                                                const double* __restrict__ dxy, float* __restrict__ dimg,
                                                                double* __restrict__ dimg64) {
  extern __shared__ double sh[];
  const int r = R > 0 ? R : P.r, HW = kLossTW + 2 * r, HH = kLossTH + 2 * r;
  double* s0 = sh;
  double* s1 = s0 + HH * HW;
  double* s2 = s1 + HH * HW;
  double* hs = s2 + HH * HW;  // 3 planes of HH x TW
  const int x0 = blockIdx.x * kLossTW, y0 = blockIdx.y * kLossTH;
  const int t = threadIdx.x;
  const int ox = t % kLossTW, oy0 = (t / kLossTW) * kLossRows;
  const int px = x0 + ox;
  for (int c = 0; c < 3; ++c) {
    if (P.lam != 0.0) {
      for (int i = t; i < HH * HW; i += kLossThreads) {
        const int yy = y0 - r + i / HW, xx = x0 - r + i % HW;
        const bool in = yy >= 0 && yy < P.H && xx >= 0 && xx < P.W;
        const size_t g = ((size_t)yy * P.W + xx) * 3 + c;
        s0[i] = in ? dmu[g] : 0.0;
        s1[i] = in ? dxx[g] : 0.0;
        s2[i] = in ? dxy[g] : 0.0;
      }
      __syncthreads();
      for (int i = t; i < HH * (kLossTW / 2); i += kLossThreads) {  // two output columns per item
        const int row = i / (kLossTW / 2), col = 2 * (i % (kLossTW / 2));
        double a0 = 0, b0 = 0, d0 = 0, a1 = 0, b1 = 0, d1 = 0;
        #pragma unroll
        for (int k = 0; k <= 2 * r + 1; ++k) {
          const int o = row * HW + col + k;
          const double x0 = s0[o], x1 = s1[o], x2 = s2[o];
          if (k <= 2 * r) {
            const double wx = P.w[k];
            a0 = fma(wx, x0, a0);
            b0 = fma(wx, x1, b0);
            d0 = fma(wx, x2, d0);
          }
          if (k >= 1) {
            const double wx = P.w[k - 1];
            a1 = fma(wx, x0, a1);
            b1 = fma(wx, x1, b1);
            d1 = fma(wx, x2, d1);
          }
        }
        const int o = row * kLossTW + col;
        hs[o] = a0;
        hs[o + 1] = a1;
        hs[HH * kLossTW + o] = b0;
        hs[HH * kLossTW + o + 1] = b1;
        hs[2 * HH * kLossTW + o] = d0;
        hs[2 * HH * kLossTW + o + 1] = d1;
      }
      __syncthreads();
    }
    {
      // the thread's kLossRows outputs share their column's loads
      double f[kLossRows][3] = {};
      if (P.lam != 0.0) {
        #pragma unroll
        for (int k = 0; k < 2 * r + kLossRows; ++k) {
          const int o = (oy0 + k) * kLossTW + ox;
          const double h0 = hs[o], h1 = hs[HH * kLossTW + o], h2 = hs[2 * HH * kLossTW + o];
          #pragma unroll
          for (int q = 0; q < kLossRows; ++q) {
            if (k - q < 0 || k - q > 2 * r) continue;
            const double wy = P.w[k - q];
            f[q][0] = fma(wy, h0, f[q][0]);
            f[q][1] = fma(wy, h1, f[q][1]);
            f[q][2] = fma(wy, h2, f[q][2]);
          }
        }
      }
      #pragma unroll
      for (int q = 0; q < kLossRows; ++q) {
        const int py = y0 + oy0 + q;
        if (px >= P.W || py >= P.H) continue;
        const size_t g = ((size_t)py * P.W + px) * 3 + c;
        const double xv = ld(img, g), yv = ld(tgt, g);
        const double diff = xv - yv;
        double out = (1.0 - P.lam) * (double)((diff > 0.0) - (diff < 0.0)) * P.inv_size;
        if (P.lam != 0.0) out -= P.lam * (f[q][0] + 2.0 * xv * f[q][1] + yv * f[q][2]) * P.inv_size;
        if (dimg) dimg[g] = (float)out;
        if (dimg64) dimg64[g] = out;
      }
    }
    if (P.lam != 0.0) __syncthreads();
  }
}

// L1-only forward sums (lambda == 0).
template <typename TI, typename TT>
__global__ void __launch_bounds__(kLossThreads) l1_sum_kernel(const TI* __restrict__ img, const TT* __restrict__ tgt,
                                                              size_t n, double* __restrict__ sums) {
  __shared__ double red[kLossThreads / 32];
  double s = 0.0;
  for (size_t i = (size_t)blockIdx.x * kLossThreads + threadIdx.x; i < n; i += (size_t)gridDim.x * kLossThreads)
    s += fabs(ld(img, i) - ld(tgt, i));
  const double tot = block_sum(s, red);
  if (threadIdx.x == 0) {
    sums[2 * blockIdx.x] = tot;
    sums[2 * blockIdx.x + 1] = 0.0;
  }
}

// One CTA: thread t sums slots t, t + 256, ... in order, then a fixed tree.
__global__ void __launch_bounds__(256) loss_finish_kernel(double* out, const double* __restrict__ part, int nparts,
                                                          double lam, double inv_size) {
  __shared__ double r0[256], r1[256];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nparts; i += 256) {
    a += part[2 * i];
    b += part[2 * i + 1];
  }
  r0[threadIdx.x] = a;
  r1[threadIdx.x] = b;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      r0[threadIdx.x] += r0[threadIdx.x + w];
      r1[threadIdx.x] += r1[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  out[3] = r0[0];
  out[4] = r1[0];
  const double l1 = out[3] * inv_size, sm = out[4] * inv_size;
  out[0] = lam == 0.0 ? (1.0 - lam) * l1 : (1.0 - lam) * l1 + lam * (1.0 - sm);
  out[1] = l1;
  out[2] = lam == 0.0 ? 0.0 : sm;
}

template <typename TI, typename TT>
static int run_loss(const TI* img, const TT* tgt, const LossParams& P, float* dimg, double* dimg64, double* smap,
                    double* out, double* planes, cudaStream_t st) {
  const size_t n = (size_t)P.H * P.W * 3;
  SGS_CUDA(cudaMemsetAsync(out, 0, 5 * sizeof(double), st));
  double* dmu = planes;
  double* dxx = planes + n;
  double* dxy = planes + 2 * n;
  double* part = planes + 3 * n;  // per-block partial sums (loss_workspace_bytes)
  const dim3 grid((P.W + kLossTW - 1) / kLossTW, (P.H + kLossTH - 1) / kLossTH);
  int nparts = (int)(grid.x * grid.y);
  if (P.lam != 0.0) {
    const size_t smem = loss_smem_doubles(P.r, 2, 5) * sizeof(double);
    if (P.r == 5) {
      SGS_CUDA(cudaFuncSetAttribute(ssim_fwd_kernel<TI, TT, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      ssim_fwd_kernel<TI, TT, 5><<<grid, kLossThreads, smem, st>>>(img, tgt, P, dmu, dxx, dxy, smap, part);
    } else {
      SGS_CUDA(cudaFuncSetAttribute(ssim_fwd_kernel<TI, TT, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      ssim_fwd_kernel<TI, TT, 0><<<grid, kLossThreads, smem, st>>>(img, tgt, P, dmu, dxx, dxy, smap, part);
    }
    SGS_LAUNCH_CHECK("ssim_fwd_kernel");
  } else {
    const int g = persistent_grid(n, kLossThreads * 8, 4);
    nparts = g;
    l1_sum_kernel<TI, TT><<<g, kLossThreads, 0, st>>>(img, tgt, n, part);
    SGS_LAUNCH_CHECK("l1_sum_kernel");
  }
  loss_finish_kernel<<<1, 256, 0, st>>>(out, part, nparts, P.lam, P.inv_size);
  SGS_LAUNCH_CHECK("loss_finish_kernel");
  if (dimg || dimg64) {
    const size_t smem = P.lam != 0.0 ? loss_smem_doubles(P.r, 3, 3) * sizeof(double) : 0;
    if (P.r == 5) {
      SGS_CUDA(cudaFuncSetAttribute(ssim_bwd_kernel<TI, TT, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      ssim_bwd_kernel<TI, TT, 5><<<grid, kLossThreads, smem, st>>>(img, tgt, P, dmu, dxx, dxy, dimg, dimg64);
    } else {
      SGS_CUDA(cudaFuncSetAttribute(ssim_bwd_kernel<TI, TT, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      ssim_bwd_kernel<TI, TT, 0><<<grid, kLossThreads, smem, st>>>(img, tgt, P, dmu, dxx, dxy, dimg, dimg64);
    }
    SGS_LAUNCH_CHECK("ssim_bwd_kernel");
  }
  return SGS_OK;
}

uint64_t loss_workspace_bytes(int H, int W) {
  const uint64_t blocks = (uint64_t)((W + kLossTW - 1) / kLossTW) * ((H + kLossTH - 1) / kLossTH);
  const uint64_t parts = blocks > (uint64_t)kNumSMs * 4 ? blocks : (uint64_t)kNumSMs * 4;
  return (uint64_t)3 * H * W * 3 * sizeof(double) + 2 * parts * sizeof(double);
}

int launch_image_loss(const void* img, int img_f64, const void* tgt, int tgt_f64, int H, int W,
                      const sgs_loss_config* cfg, float* dimg, double* dimg64, double* smap, double* out,
                      void* workspace, uint64_t ws_bytes, cudaStream_t st) {
  if (!img || !tgt || !cfg || !out || H < 1 || W < 1 || cfg->window < 1 || cfg->window > kMaxWindow ||
      (cfg->window & 1) == 0 || !(cfg->sigma > 0.0)) {
    set_error("invalid loss arguments (window must be odd and <= %d)", kMaxWindow);
    return SGS_E_ARG;
  }
  if (ws_bytes < loss_workspace_bytes(H, W) || !workspace) {
    set_error("loss workspace too small: need %llu bytes", (unsigned long long)loss_workspace_bytes(H, W));
    return SGS_E_WORKSPACE;
  }
  LossParams P;
  // normalised Gaussian window, render.py:435-438
  const int win = cfg->window;
  double tot = 0.0;
  for (int k = 0; k < win; ++k) {
    const double tt = (double)k - (win - 1) / 2.0;
    P.w[k] = exp(-0.5 * (tt / cfg->sigma) * (tt / cfg->sigma));
    tot += P.w[k];
  }
  for (int k = 0; k < win; ++k) P.w[k] /= tot;
  P.r = win / 2;
  P.H = H;
  P.W = W;
  P.lam = cfg->lambda_ssim;
  P.c1 = cfg->c1;
  P.c2 = cfg->c2;
  P.inv_size = 1.0 / ((double)H * W * 3);
  double* planes = reinterpret_cast<double*>(workspace);
  if (img_f64) {
    const double* i = reinterpret_cast<const double*>(img);
    if (tgt_f64) return run_loss(i, reinterpret_cast<const double*>(tgt), P, dimg, dimg64, smap, out, planes, st);
    return run_loss(i, reinterpret_cast<const float*>(tgt), P, dimg, dimg64, smap, out, planes, st);
  }
  const float* i = reinterpret_cast<const float*>(img);
  if (tgt_f64) return run_loss(i, reinterpret_cast<const double*>(tgt), P, dimg, dimg64, smap, out, planes, st);
  return run_loss(i, reinterpret_cast<const float*>(tgt), P, dimg, dimg64, smap, out, planes, st);
}

}  // namespace sgs
