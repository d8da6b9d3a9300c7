// Deterministic (raw-probability) mode and its reverse-mode gradient (BASELINE C4).
//
// Forward = step_deterministic_into (engine.hpp:147-175) in fp32 over [env][cell] planes:
//   lambda(v) = sum_k [p_burn(u_k) != 0] p_burn(u_k) * pot(u_k, k)      (fixed k order)
//   p_ig = 1 - exp(-gamma(v) lambda);  newly = un p_ig;
//   burn' = newly + burn pc;  un' = un - newly;  bd' = bd + burn (1 - pc).
// pot / gamma come from a per-launch fp32 table built on the device from the terrain
// statics (kernel.hpp:21-45 association).  With `record`, (un_t, burn_t) of every step are
// kept in HBM for the backward pass.
//
// Backward (the adjoint of the above, replacing the reference's forward-mode Dual<6>,
// calibrate.cpp:130-162): per step t = T-1..0, two kernels
//   back1 (per cell v): a_newly = A_burn - A_un, a_x = a_newly un e^{-x}, a_lambda = a_x gamma,
//          A_un <- A_un + a_newly p_ig;  d/d alpha_gamma += a_x lambda F(v),
//          d/d p_continue += burn (A_burn - A_bd)
//   back2 (per source cell u): A_burn <- A_burn pc + A_bd (1-pc) + [burn(u)!=0] sum_k a_lambda(u+d_k) pot(u,k),
//          d/d{p_base, alpha_w1, alpha_w2, alpha_s} += a_lambda(u+d_k) burn(u) dpot(u,k)/dtheta
// Parameter gradients accumulate in fp64 per (env, CTA) in a fixed order (deterministic)
// and are reduced per env at the end.
#include <cuda_runtime.h>

#include <cstdint>

#include "ember_device.cuh"
#include "ember_kernels.h"
#include "ember_params.h"

namespace ebl {

namespace {

__device__ __forceinline__ double block_sum_d(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) t += red[i];  // fixed order
  return t;
}

}  // namespace

// pot32[env][cell][8], gam32[env][cell], F[env][cell] = (1+veg)(1+den) from terrain statics.
__global__ void k_det_tables(DetArgs d) {
  const StepArgs& a = d.s;
  const int ncell = a.h * a.w;
  const int env = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ncell) return;
  const TerrainView t = terrain_view(a, env);
  const int r = i / a.w, c = i - r * a.w;
  const uint8_t cls = t.fuel[i];
  const float src = t.pal_src32[cls];
  const size_t o = static_cast<size_t>(env) * ncell + i;
  d.gam32[o] = t.pal_gam32[cls];
  d.F32[o] = a.pal32[512 + cls];
  const float zu = t.elev[i];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int vr = r + kDy[k], vc = c + kDx[k];  // target of direction k from source u
    float pot = 0.f;
    if (vr >= 0 && vr < a.h && vc >= 0 && vc < a.w) {
      const float s = atanf((t.elev[vr * a.w + vc] - zu) * t.inv_dist32[k & 1]);
      pot = src * t.kw32[k] * expf(t.alpha_s32 * s);
    }
    d.pot32[o * 8 + k] = pot;
  }
}

__global__ void k_det_forward(DetArgs d, int t) {
  const StepArgs& a = d.s;
  const int ncell = a.h * a.w;
  const int env = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ncell) return;
  const size_t base = static_cast<size_t>(env) * ncell;
  const int r = i / a.w, c = i - r * a.w;
  const float* burn = d.burn;
  float lam = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int ur = r - kDy[k], uc = c - kDx[k];
    if (ur < 0 || ur >= a.h || uc < 0 || uc >= a.w) continue;
    const size_t u = base + ur * a.w + uc;
    const float wgt = burn[u];
    if (wgt == 0.f) continue;  // kernel.hpp:63 zero-weight skip
    lam += wgt * d.pot32[u * 8 + k];
  }
  const float e = expf(-d.gam32[base + i] * lam);
  const float p_ig = 1.f - e;
  const float un = d.un[base + i], bu = burn[base + i], bd = d.bd[base + i];
  const float newly = un * p_ig;
  d.burn_o[base + i] = newly + bu * d.pc32;
  d.un_o[base + i] = un - newly;
  d.bd_o[base + i] = bd + bu * (1.f - d.pc32);
  if (d.traj_un) {
    const size_t tr = static_cast<size_t>(t) * a.n_envs * ncell + base + i;
    d.traj_un[tr] = un;
    d.traj_burn[tr] = bu;
  }
}

// Loss (calibrate.hpp:120-146) per env and dL/dpred -> initial adjoints.  One CTA per env.
__global__ void k_det_loss(DetArgs d) {
  __shared__ double red[32];
  const StepArgs& a = d.s;
  const int ncell = a.h * a.w;
  const int env = blockIdx.x;
  const size_t base = static_cast<size_t>(env) * ncell;
  const int pool = d.pool;
  const int oh = (a.h + pool - 1) / pool, ow = (a.w + pool - 1) / pool;
  const double eps = 1e-6;
  double bce = 0.0, mse = 0.0;
  for (int i = threadIdx.x; i < ncell; i += blockDim.x) {
    const double pred = static_cast<double>(d.burn[base + i]) + static_cast<double>(d.bd[base + i]);
    const double m = d.mask[base + i];
    const double p = fmin(fmax(pred, eps), 1.0 - eps);
    bce += -(m * log(p) + (1.0 - m) * log(1.0 - p));
    double g = 0.0;
    if (pred >= eps && pred <= 1.0 - eps) g = (-(m / p) + (1.0 - m) / (1.0 - p)) / ncell;
    d.grad_pred[base + i] = d.bce_w * g;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < oh * ow; q += blockDim.x) {
    const int pr = q / ow, pc = q - pr * ow;
    double sp = 0.0, sm = 0.0;
    int cnt = 0;
    for (int r = pr * pool; r < (pr + 1) * pool && r < a.h; ++r)
      for (int c = pc * pool; c < (pc + 1) * pool && c < a.w; ++c) {
        const size_t i = base + r * a.w + c;
        sp += static_cast<double>(d.burn[i]) + static_cast<double>(d.bd[i]);
        sm += d.mask[i];
        ++cnt;
      }
    const double diff = sp / cnt - sm / cnt;
    mse += diff * diff;
    const double g = d.mse_w * 2.0 * diff / (static_cast<double>(oh) * ow) / cnt;
    for (int r = pr * pool; r < (pr + 1) * pool && r < a.h; ++r)
      for (int c = pc * pool; c < (pc + 1) * pool && c < a.w; ++c) d.grad_pred[base + r * a.w + c] += g;
  }
  bce = block_sum_d(bce, red);
  mse = block_sum_d(mse, red);
  if (threadIdx.x == 0)
    d.loss[env] = d.bce_w * (bce / ncell) + d.mse_w * (mse / (static_cast<double>(oh) * ow));
  __syncthreads();
  for (int i = threadIdx.x; i < ncell; i += blockDim.x) {
    const float g = static_cast<float>(d.grad_pred[base + i]);
    d.A_burn[base + i] = g;  // pred = p_burn + p_bd
    d.A_bd[base + i] = g;
    d.A_un[base + i] = 0.f;
  }
}

// back1: lambda, a_lambda, A_un update, gamma / p_continue gradients.
__global__ void k_det_back1(DetArgs d, int t) {
  __shared__ double red[32];
  const StepArgs& a = d.s;
  const int ncell = a.h * a.w;
  const int env = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const size_t base = static_cast<size_t>(env) * ncell;
  const size_t tr = static_cast<size_t>(t) * a.n_envs * ncell + base;
  double g_gamma = 0.0, g_pc = 0.0;
  if (i < ncell) {
    const int r = i / a.w, c = i - r * a.w;
    float lam = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int ur = r - kDy[k], uc = c - kDx[k];
      if (ur < 0 || ur >= a.h || uc < 0 || uc >= a.w) continue;
      const int u = ur * a.w + uc;
      const float wgt = d.traj_burn[tr + u];
      if (wgt == 0.f) continue;
      lam += wgt * d.pot32[(base + u) * 8 + k];
    }
    const float gam = d.gam32[base + i];
    const float e = expf(-gam * lam);
    const float p_ig = 1.f - e;
    const float un = d.traj_un[tr + i], bu = d.traj_burn[tr + i];
    const float Au = d.A_un[base + i], Ab = d.A_burn[base + i], Ad = d.A_bd[base + i];
    const float a_newly = Ab - Au;
    const float a_x = a_newly * un * e;
    d.a_lam[base + i] = a_x * gam;
    d.A_un[base + i] = Au + a_newly * p_ig;
    g_gamma = static_cast<double>(a_x) * lam * d.F32[base + i];
    g_pc = static_cast<double>(bu) * (static_cast<double>(Ab) - Ad);
  }
  g_gamma = block_sum_d(g_gamma, red);
  g_pc = block_sum_d(g_pc, red);
  if (threadIdx.x == 0) {
    double* acc = d.acc + (static_cast<size_t>(env) * gridDim.x + blockIdx.x) * 8;
    acc[4] += g_gamma;
    acc[5] += g_pc;
  }
}

// back2: A_burn, A_bd updates and the pot-parameter gradients (source-cell gather).
__global__ void k_det_back2(DetArgs d, int t) {
  __shared__ double red[32];
  const StepArgs& a = d.s;
  const int ncell = a.h * a.w;
  const int env = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const size_t base = static_cast<size_t>(env) * ncell;
  const size_t tr = static_cast<size_t>(t) * a.n_envs * ncell + base;
  double gp = 0.0, gw1 = 0.0, gw2 = 0.0, gs = 0.0;
  if (i < ncell) {
    const int r = i / a.w, c = i - r * a.w;
    const float bu = d.traj_burn[tr + i];
    const float Ab = d.A_burn[base + i], Ad = d.A_bd[base + i];
    float acc_burn = Ab * d.pc32 + Ad * (1.f - d.pc32);
    if (bu != 0.f) {
      const TerrainView tv = terrain_view(a, env);
      const float V = d.wind_speed32[env * d.wind_stride];
      const float zu = tv.elev[i];
      const float Fu = d.F32[base + i];
      double s_gp = 0.0, s_gw1 = 0.0, s_gw2 = 0.0, s_gs = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int vr = r + kDy[k], vc = c + kDx[k];
        if (vr < 0 || vr >= a.h || vc < 0 || vc >= a.w) continue;
        const float al = d.a_lam[base + vr * a.w + vc];
        if (al == 0.f) continue;
        const float pot = d.pot32[(base + i) * 8 + k];
        acc_burn += al * pot;
        const float slope = atanf((tv.elev[vr * a.w + vc] - zu) * tv.inv_dist32[k & 1]);
        // pot = p_base F kw ks:  dpot/dp_base = F kw ks,  dpot/dalpha_w1 = pot V,
        // dpot/dalpha_w2 = pot V (cos - 1),  dpot/dalpha_s = pot S   (kernel.hpp:21-45)
        const double ab = static_cast<double>(al) * bu;
        const double q = ab * pot;
        s_gp += ab * (static_cast<double>(Fu) * tv.kw32[k] * expf(tv.alpha_s32 * slope));
        s_gw1 += q * V;
        s_gw2 += q * V * d.align32[env * d.wind_stride * 8 + k];
        s_gs += q * slope;
      }
      gp = s_gp;
      gw1 = s_gw1;
      gw2 = s_gw2;
      gs = s_gs;
    }
    d.A_burn[base + i] = acc_burn;
    // A_bd is unchanged (bd' = bd + ...)
  }
  gp = block_sum_d(gp, red);
  gw1 = block_sum_d(gw1, red);
  gw2 = block_sum_d(gw2, red);
  gs = block_sum_d(gs, red);
  if (threadIdx.x == 0) {
    double* acc = d.acc + (static_cast<size_t>(env) * gridDim.x + blockIdx.x) * 8;
    acc[0] += gp;
    acc[1] += gw1;
    acc[2] += gw2;
    acc[3] += gs;
  }
}

__global__ void k_det_reduce(DetArgs d, int blocks_per_env) {
  const int env = blockIdx.x;
  const int k = threadIdx.x;
  if (k >= 6) return;
  double s = 0.0;
  for (int b = 0; b < blocks_per_env; ++b) s += d.acc[(static_cast<size_t>(env) * blocks_per_env + b) * 8 + k];
  d.grad[env * 6 + k] = s;
}

cudaError_t launch_det_tables(const DetArgs& d, cudaStream_t s) {
  const int ncell = d.s.h * d.s.w;
  k_det_tables<<<dim3((ncell + 255) / 256, d.s.n_envs), 256, 0, s>>>(d);
  return cudaGetLastError();
}

cudaError_t launch_det_forward(const DetArgs& d, int t, cudaStream_t s) {
  const int ncell = d.s.h * d.s.w;
  k_det_forward<<<dim3((ncell + 255) / 256, d.s.n_envs), 256, 0, s>>>(d, t);
  return cudaGetLastError();
}

cudaError_t launch_det_loss(const DetArgs& d, cudaStream_t s) {
  k_det_loss<<<d.s.n_envs, 256, 0, s>>>(d);
  return cudaGetLastError();
}

cudaError_t launch_det_backward(const DetArgs& d, int t, cudaStream_t s) {
  const int ncell = d.s.h * d.s.w;
  const dim3 grid((ncell + 255) / 256, d.s.n_envs);
  k_det_back1<<<grid, 256, 0, s>>>(d, t);
  k_det_back2<<<grid, 256, 0, s>>>(d, t);
  return cudaGetLastError();
}

cudaError_t launch_det_reduce(const DetArgs& d, cudaStream_t s) {
  const int ncell = d.s.h * d.s.w;
  k_det_reduce<<<d.s.n_envs, 32, 0, s>>>(d, (ncell + 255) / 256);
  return cudaGetLastError();
}

}  // namespace ebl
