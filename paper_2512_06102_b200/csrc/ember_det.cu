// Deterministic (raw-probability) mode and its reverse-mode gradient (BASELINE C4).
//
// Forward = step_deterministic_into (engine.hpp:147-175), evaluated in the reference's fp64
// arithmetic and association (explicit __dadd_rn/__dmul_rn, no FMA contraction):
//   lambda(v) = sum_k [p_burn(u_k) != 0] p_burn(u_k) * pot(u_k, k)      (k order, zero skip)
//   p_ig = 1 - exp(-(gamma(v) lambda));  newly = un p_ig;
//   burn' = newly + burn pc;  un' = un - newly;  bd' = bd + burn (1 - pc).
// pot / gamma are the reference's SpreadTables<double> values, built on the host with the
// same libm (ember_host.cpp) and kept resident.  Why fp64 and not fp32: the
// reference's 1 - exp(-x) is quantised to multiples of 2^-53 for tiny x, and the leading edge
// of the probability front grows those quanta geometrically, so its step-100 state moves by
// ~4e-2 under 1-ulp changes of exp alone; matching it to 1e-4 needs its exact arithmetic,
// including a correctly rounded exp for tiny arguments (glibc's is, there).
//
// Backward (the adjoint of the above; the reference differentiates forward-mode with
// Dual<6>, calibrate.cpp:130-162), per step t = T-1..0, two kernels:
//   back1 (per cell v): a_newly = A_burn - A_un, a_x = a_newly un e^{-x}, a_lambda = a_x gamma,
//          A_un <- A_un + a_newly p_ig;  d/dalpha_gamma += a_x lambda F(v),
//          d/dp_continue += burn (A_burn - A_bd)
//   back2 (per source cell u): A_burn <- A_burn pc + A_bd (1-pc) + [burn(u)!=0] sum_k a_lambda(u+d_k) pot(u,k),
//          d/d{p_base, alpha_w1, alpha_w2, alpha_s} += a_lambda(u+d_k) burn(u) dpot(u,k)/dtheta
// (the zero-weight skip drops the same tangent paths Dual's skip does).  Parameter gradients
// are reduced per (env, CTA) and then per env in a fixed order: deterministic.
#include <cuda_runtime.h>

#include <cstdint>

#include "ember_device.cuh"
#include "ember_exp.cuh"
#include "ember_kernels.h"
#include "ember_pdl.cuh"
#include "ember_params.h"

namespace ebl {


namespace {

// Fixed-order block sums of N values at once (one shared round trip instead of N); the result
// is valid in thread 0 only (the callers' only reader).
template <int N>
__device__ __forceinline__ void block_sum_n(double (&v)[N], double* red) {
#pragma unroll
  for (int q = 0; q < N; ++q)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
  __syncthreads();  // red[] may still be read by a previous call
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int q = 0; q < N; ++q) red[q * 32 + (threadIdx.x >> 5)] = v[q];
  __syncthreads();
  if (threadIdx.x == 0)
#pragma unroll
    for (int q = 0; q < N; ++q) {
      double t = 0.0;
      for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) t += red[q * 32 + i];  // fixed order
      v[q] = t;
    }
}

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

// exp(-x) for x >= 0, correctly rounded where it matters for 1 - exp(-x): for x < 2^-20 the
// value is 1 - x + x^2/2 - ... summed as a double-double (two_sum of 1 and -x, then the tail),
// rounded once; beyond that CUDA's exp (1 - exp(-x) is then insensitive to its last ulp).
__device__ __forceinline__ double exp_neg(double x) {
  if (x < 0x1.0p-20) {
    const double s = -x;
    const double hi = __dadd_rn(1.0, s);
    const double lo = __dsub_rn(s, __dsub_rn(hi, 1.0));  // exact: two_sum with |s| < 1
    const double s2 = s * s;
    const double tail = s2 * (0.5 + s * (1.0 / 6.0 + s * (1.0 / 24.0 + s * (1.0 / 120.0))));
    return __dadd_rn(hi, __dadd_rn(lo, tail));
  }
  return exp(-x);
}

// gamma(v) of the SpreadTables: for terrain layers the palette entry of the cell's class (the same
// fp64 expression the host table holds, (alpha_gamma (1+veg)) (1+den), kernel.hpp:75-76): one byte
// per cell instead of eight; general layers read the table.
__device__ __forceinline__ double gamma_at(const DetArgs& d, size_t tb, int env, int i) {
  const StepArgs& a = d.s;
  if (a.fuel && !d.fac_pb) return a.pal64[256 + a.fuel[static_cast<size_t>(env) * a.ter_stride + i]];
  return d.gam[tb + i];
}

__device__ __forceinline__ double lambda_at(const double* __restrict__ burn, const double* __restrict__ pot,
                                            int h, int w, int r, int c) {
  double lam = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int ur = r - kDy[k], uc = c - kDx[k];
    if (ur < 0 || ur >= h || uc < 0 || uc >= w) continue;
    const int u = ur * w + uc;
    const double wgt = burn[u];
    if (wgt == 0.0) continue;  // kernel.hpp:63 zero-weight skip
    lam = __dadd_rn(lam, __dmul_rn(wgt, pot[static_cast<size_t>(u) * 8 + k]));
  }
  return lam;
}

}  // namespace

// lambda from the target-ordered table: the 8 source terms of cell v are one contiguous 64-byte row
// (four 16-byte loads issued together, coalesced across the warp) instead of 8 loads strided by a
// source row each; same k-ordered fold with the zero-weight skip, same fp64 operations.
__device__ __forceinline__ double lambda_at_t(const double* __restrict__ burn, const double* __restrict__ potT, int h,
                                              int w, int r, int c) {
  double wk[8];
  bool any = false;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int ur = r - kDy[k], uc = c - kDx[k];
    wk[k] = (ur < 0 || ur >= h || uc < 0 || uc >= w) ? 0.0 : burn[ur * w + uc];
    any |= wk[k] != 0.0;
  }
  if (!any) return 0.0;  // no burning source: the row is not needed (lambda = 0, as the skip gives)
  const size_t i = static_cast<size_t>(r) * w + c;
  const double2 p01 = __ldg(reinterpret_cast<const double2*>(potT + i * 8));
  const double2 p23 = __ldg(reinterpret_cast<const double2*>(potT + i * 8 + 2));
  const double2 p45 = __ldg(reinterpret_cast<const double2*>(potT + i * 8 + 4));
  const double2 p67 = __ldg(reinterpret_cast<const double2*>(potT + i * 8 + 6));
  const double pk[8] = {p01.x, p01.y, p23.x, p23.y, p45.x, p45.y, p67.x, p67.y};
  double lam = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if (wk[k] != 0.0) lam = __dadd_rn(lam, __dmul_rn(wk[k], pk[k]));  // k order, zero-weight skip
  return lam;
}

__global__ void k_pot_target(const double* __restrict__ pot, double* __restrict__ potT, int n_tables, int h, int w) {
  const size_t ncell = static_cast<size_t>(h) * w, total = static_cast<size_t>(n_tables) * ncell * 8;
  for (size_t j = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < total;
       j += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(j & 7);
    const size_t tc = j >> 3, t = tc / ncell, v = tc - t * ncell;
    const int r = static_cast<int>(v / w), c = static_cast<int>(v % w);
    const int ur = r - kDy[k], uc = c - kDx[k];
    potT[j] = (ur < 0 || ur >= h || uc < 0 || uc >= w) ? 0.0 : pot[(t * ncell + static_cast<size_t>(ur) * w + uc) * 8 + k];
  }
}

cudaError_t launch_pot_target(const double* pot, double* potT, int n_tables, int h, int w, cudaStream_t s) {
  const size_t total = static_cast<size_t>(n_tables) * h * w * 8;
  const unsigned blocks = static_cast<unsigned>(std::min<size_t>((total + 255) / 256, 148 * 8));
  k_pot_target<<<blocks, 256, 0, s>>>(pot, potT, n_tables, h, w);
  return cudaGetLastError();
}

__global__ void k_det_forward(DetArgs d, int t) {
  const StepArgs& a = d.s;
  const int ncell = a.h * a.w;
  const int env = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ncell) return;
  const size_t base = static_cast<size_t>(env) * ncell;
  const size_t tb = static_cast<size_t>(env) * d.tab_stride;
  const double lam = d.potT ? lambda_at_t(d.burn + base, d.potT + tb * 8, a.h, a.w, i / a.w, i % a.w)
                            : lambda_at(d.burn + base, d.pot + tb * 8, a.h, a.w, i / a.w, i % a.w);
  const double p_ig = __dsub_rn(1.0, exp_neg(__dmul_rn(gamma_at(d, tb, env, i), lam)));
  const double un = d.un[base + i], bu = d.burn[base + i];
  const double newly = __dmul_rn(un, p_ig);
  d.burn_o[base + i] = __dadd_rn(newly, __dmul_rn(bu, d.pc));
  d.un_o[base + i] = __dsub_rn(un, newly);
  if (d.bd)  // (record mode: p_bd is accumulated after the run from the recorded p_burn, k_det_bd_run)
    d.bd_o[base + i] = __dadd_rn(d.bd[base + i], __dmul_rn(bu, __dsub_rn(1.0, d.pc)));
  // record mode: the states of steps >= 1 are written straight into their trajectory slots (the
  // host points un_o / burn_o there), so only step 0 copies its input; lambda every step
  const size_t tr = static_cast<size_t>(t) * a.n_envs * ncell + base + i;
  if (d.traj_un) {
    d.traj_un[tr] = un;
    d.traj_burn[tr] = bu;
  }
  if (d.traj_lam) d.traj_lam[tr] = lam;
}

// The forward with two horizontally adjacent cells per thread (target-ordered pot, even widths):
// the state and trajectory planes move as 16-byte vectors and every thread keeps twice the loads in
// flight; each cell's arithmetic is k_det_forward's.
#ifndef EBL_DET_FWD2
#define EBL_DET_FWD2 1
#endif
#ifndef EBL_DET_FWD_MINB
#define EBL_DET_FWD_MINB 12  // 40 registers at 128 threads (256: 6 CTAs/SM, C4 14.95 -> 14.58 ms; 5: 14.73, 7: 16.30)
#endif
#ifndef EBL_DET_FWD_THREADS
#define EBL_DET_FWD_THREADS 128  // C4: 128 x 12 CTAs/SM 14.37 ms, 256 x 6 14.58, 64 x 24 14.38, 512 x 3 14.93
#endif
__global__ void __launch_bounds__(EBL_DET_FWD_THREADS, EBL_DET_FWD_MINB) k_det_forward2(DetArgs d, int t) {
  pdl_enter();
  const StepArgs& a = d.s;
  const int ncell = a.h * a.w;
  const int env = blockIdx.y;
  const int i0 = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (i0 >= ncell) return;
  const size_t base = static_cast<size_t>(env) * ncell;
  const size_t tb = static_cast<size_t>(env) * d.tab_stride;
  const int r = i0 / a.w, c = i0 % a.w;
  const double2 un2 = *reinterpret_cast<const double2*>(d.un + base + i0);
  const double2 bu2 = *reinterpret_cast<const double2*>(d.burn + base + i0);
  double lam[2], pig[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    lam[k] = lambda_at_t(d.burn + base, d.potT + tb * 8, a.h, a.w, r, c + k);
    pig[k] = __dsub_rn(1.0, exp_neg(__dmul_rn(gamma_at(d, tb, env, i0 + k), lam[k])));
  }
  const double un[2] = {un2.x, un2.y}, bu[2] = {bu2.x, bu2.y};
  double o_b[2], o_u[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double newly = __dmul_rn(un[k], pig[k]);
    o_b[k] = __dadd_rn(newly, __dmul_rn(bu[k], d.pc));
    o_u[k] = __dsub_rn(un[k], newly);
  }
  *reinterpret_cast<double2*>(d.burn_o + base + i0) = make_double2(o_b[0], o_b[1]);
  *reinterpret_cast<double2*>(d.un_o + base + i0) = make_double2(o_u[0], o_u[1]);
  if (d.bd) {  // (record mode: p_bd is accumulated after the run from the recorded p_burn, k_det_bd_run)
    const double2 bd2 = *reinterpret_cast<const double2*>(d.bd + base + i0);
    const double q = __dsub_rn(1.0, d.pc);
    *reinterpret_cast<double2*>(d.bd_o + base + i0) =
        make_double2(__dadd_rn(bd2.x, __dmul_rn(bu[0], q)), __dadd_rn(bd2.y, __dmul_rn(bu[1], q)));
  }
  const size_t tr = static_cast<size_t>(t) * a.n_envs * ncell + base + i0;
  if (d.traj_un) {
    *reinterpret_cast<double2*>(d.traj_un + tr) = un2;
    *reinterpret_cast<double2*>(d.traj_burn + tr) = bu2;
  }
  if (d.traj_lam) *reinterpret_cast<double2*>(d.traj_lam + tr) = make_double2(lam[0], lam[1]);
}

// state_from_fire (engine.cpp:42-52): one-hot planes from the member layers, on the device.
__global__ void k_det_from_fire(const uint8_t* __restrict__ st, double* un, double* bu, double* bd, size_t n) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint8_t s = st[i];
  un[i] = s == 0 ? 1.0 : 0.0;
  bu[i] = s == 1 ? 1.0 : 0.0;
  bd[i] = s == 2 ? 1.0 : 0.0;
}

// Loss (calibrate.hpp:120-146) per env and dL/dpred -> the adjoints of the final state.
// One CTA per env.
#ifndef EBL_DET_LOSS_THREADS
#define EBL_DET_LOSS_THREADS 1024  // one CTA per env: 256 threads took 192 us of a C4 run (1.7 CTAs per SM)
#endif
__global__ void __launch_bounds__(EBL_DET_LOSS_THREADS) k_det_loss(DetArgs d) {
  __shared__ double red[32];
  const StepArgs& a = d.s;
  const int ncell = a.h * a.w;
  const int env = blockIdx.x;
  const size_t base = static_cast<size_t>(env) * ncell;
  const int pool = d.pool;
  const int oh = (a.h + pool - 1) / pool, ow = (a.w + pool - 1) / pool;
  const double eps = 1e-6;  // LossConfig::bce_epsilon
  double bce = 0.0, mse = 0.0;
  for (int i = threadIdx.x; i < ncell; i += blockDim.x) {
    if (d.bce_w == 0.0) {  // the BCE term is bce_w * (finite) = +0 exactly: skip its two fp64 logs
      d.A_burn[base + i] = 0.0;
      continue;
    }
    const double pred = d.burn[base + i] + d.bd[base + i];
    const double m = d.mask[base + i];
    const double p = fmin(fmax(pred, eps), 1.0 - eps);
    bce += -(m * log(p) + (1.0 - m) * log(1.0 - p));
    double g = 0.0;  // max/min pass the derivative on ties to pred (dual.hpp:180-193)
    if (pred >= eps && pred <= 1.0 - eps) g = (-(m / p) + (1.0 - m) / (1.0 - p)) / ncell;
    d.A_burn[base + i] = d.bce_w * g;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < oh * ow; q += blockDim.x) {
    const int pr = q / ow, pc = q - pr * ow;
    double sp = 0.0, sm = 0.0;
    int cnt = 0;
    for (int r = pr * pool; r < (pr + 1) * pool && r < a.h; ++r)
      for (int c = pc * pool; c < (pc + 1) * pool && c < a.w; ++c) {
        const size_t i = base + r * a.w + c;
        sp += d.burn[i] + d.bd[i];
        sm += d.mask[i];
        ++cnt;
      }
    const double diff = sp / cnt - sm / cnt;
    mse += diff * diff;
    const double g = d.mse_w * 2.0 * diff / (static_cast<double>(oh) * ow) / cnt;
    for (int r = pr * pool; r < (pr + 1) * pool && r < a.h; ++r)
      for (int c = pc * pool; c < (pc + 1) * pool && c < a.w; ++c) d.A_burn[base + r * a.w + c] += g;
  }
  bce = block_sum_d(bce, red);
  mse = block_sum_d(mse, red);
  if (threadIdx.x == 0)
    d.loss[env] = d.bce_w * (bce / ncell) + d.mse_w * (mse / (static_cast<double>(oh) * ow));
  __syncthreads();
  for (int i = threadIdx.x; i < ncell; i += blockDim.x) {
    d.A_bd[base + i] = d.A_burn[base + i];  // pred = p_burn + p_bd
    d.A_un[base + i] = 0.0;
  }
}

// back1: lambda, a_lambda, A_un update, gamma / p_continue gradients.
__global__ void k_det_back1(DetArgs d, int t) {
  __shared__ double red[2 * 32];
  const StepArgs& a = d.s;
  const int ncell = a.h * a.w;
  const int env = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const size_t base = static_cast<size_t>(env) * ncell;
  const size_t tb = static_cast<size_t>(env) * d.tab_stride;
  const size_t tr = static_cast<size_t>(t) * a.n_envs * ncell + base;
  double g_gamma = 0.0, g_pc = 0.0;
  if (i < ncell) {
    const double lam = d.traj_lam[tr + i];  // bit-identical to re-folding traj_burn * pot
    const double gam = gamma_at(d, tb, env, i);
    const double x = __dmul_rn(gam, lam);
    const double e = exp_neg(x);
    const double p_ig = __dsub_rn(1.0, e);
    const double un = d.traj_un[tr + i], bu = d.traj_burn[tr + i];
    const double Au = d.A_un[base + i], Ab = d.A_burn[base + i], Ad = d.A_bd[base + i];
    const double a_newly = Ab - Au;
    const double a_x = a_newly * un * e;  // dp_ig/dx = e^{-x} (Dual's exp)
    d.a_lam[base + i] = a_x * gam;
    d.A_un[base + i] = Au + a_newly * p_ig;
    const double F = d.fac_F ? d.fac_F[tb + i] : a.pal64[768 + a.fuel[static_cast<size_t>(env) * a.ter_stride + i]];
    g_gamma = a_x * lam * F;  // dgamma/dalpha_gamma = F(v)
    g_pc = bu * (Ab - Ad);
  }
  double g2[2] = {g_gamma, g_pc};
  block_sum_n<2>(g2, red);
  if (threadIdx.x == 0) {
    double* acc = d.acc + (static_cast<size_t>(env) * gridDim.x + blockIdx.x) * 8;
    acc[4] += g2[0];
    acc[5] += g2[1];
  }
}

// back2: A_burn update and the pot-parameter gradients (gather over each source cell's targets).
__global__ void k_det_back2(DetArgs d, int t) {
  __shared__ double red[4 * 32];
  const StepArgs& a = d.s;
  const int ncell = a.h * a.w;
  const int env = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const size_t base = static_cast<size_t>(env) * ncell;
  const size_t tb = static_cast<size_t>(env) * d.tab_stride;
  const size_t tr = static_cast<size_t>(t) * a.n_envs * ncell + base;
  double gp = 0.0, gw1 = 0.0, gw2 = 0.0, gs = 0.0;
  if (i < ncell) {
    const int r = i / a.w, c = i - r * a.w;
    const double bu = d.traj_burn[tr + i];
    double acc_burn = d.A_burn[base + i] * d.pc + d.A_bd[base + i] * (1.0 - d.pc);
    if (bu != 0.0 && d.fac_pb) {  // general form: host-built derivative factors
      const size_t o = tb + i;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int vr = r + kDy[k], vc = c + kDx[k];
        if (vr < 0 || vr >= a.h || vc < 0 || vc >= a.w) continue;
        const double al = d.a_lam[base + vr * a.w + vc];
        if (al == 0.0) continue;
        const double pot = d.pot[o * 8 + k];
        acc_burn += al * pot;
        const double ab = al * bu;
        gp += ab * d.fac_pb[o * 8 + k];
        gw1 += ab * pot * d.fac_V[o];
        gw2 += ab * pot * d.fac_Va[o * 8 + k];
        gs += ab * pot * d.fac_S[o * 8 + k];
      }
    } else if (bu != 0.0) {
      const TerrainView tv = terrain_view(a, env);
      const float* slope = a.slope32 ? a.slope32 + static_cast<size_t>(env) * a.ter_stride * 8 : nullptr;
      const double V = d.V[env * d.wind_stride];
      const float zu = tv.elev[i];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int vr = r + kDy[k], vc = c + kDx[k];
        if (vr < 0 || vr >= a.h || vc < 0 || vc >= a.w) continue;
        const double al = d.a_lam[base + vr * a.w + vc];
        if (al == 0.0) continue;
        const double pot = d.pot[(tb + i) * 8 + k];
        acc_burn += al * pot;
        // pot = p_base F kw ks (kernel.hpp:21-45): dpot/dp_base = F kw ks, dpot/dalpha_w1 = pot V,
        // dpot/dalpha_w2 = pot V (cos - 1), dpot/dalpha_s = pot S
        // S in fp32 (relative error ~1e-7, far inside the 1e-4 gradient bar); fp32 elevations
        // differ exactly in fp32 unless they are ~2^24 apart in magnitude
        // the slope table holds exactly this fp32 value (record of the target v, direction k)
        double S;
        if (slope) {
          S = static_cast<double>(slope[static_cast<size_t>(vr * a.w + vc) * 8 + k]);
        } else {
          const float dz = tv.elev[vr * a.w + vc] - zu;
          S = dz == dz ? static_cast<double>(atanf(dz * tv.inv_dist32[k & 1])) : 0.0;  // nodata: 0
        }
        const double ab = al * bu;
        gp += ab * (pot * d.inv_p_base);
        gw1 += ab * pot * V;
        gw2 += ab * pot * V * d.align[env * d.wind_stride * 8 + k];
        gs += ab * pot * S;
      }
    }
    d.A_burn[base + i] = acc_burn;  // A_bd is unchanged (bd' = bd + ...)
  }
  double g4[4] = {gp, gw1, gw2, gs};
  block_sum_n<4>(g4, red);
  if (threadIdx.x == 0) {
    double* acc = d.acc + (static_cast<size_t>(env) * gridDim.x + blockIdx.x) * 8;
    acc[0] += g4[0];
    acc[1] += g4[1];
    acc[2] += g4[2];
    acc[3] += g4[3];
  }
}


// back1 + back2 fused per 32 x 8 tile (one launch per step): a_lambda of the tile and its 1-cell
// ring in shared memory (the ring's back1 is recomputed from the same inputs, bit-identical), then
// the gather of back2.  The adjoints are double-buffered (A_un / A_burn read, A_un_o / A_burn_o
// written) because neighbouring tiles read the old values of this tile's ring.  The slope of the
// direction-k pot derivative is the source's own record of the opposite direction, negated
// (atan is odd and fp32 negation exact): 32 contiguous bytes instead of 8 scattered records.
#ifndef EBL_DET_CPT
#define EBL_DET_CPT 2  // cells per thread (rows kBackTy apart): more loads in flight, a thinner ring
#endif
constexpr int kBackTx = 32, kBackTy = 8, kCpt = EBL_DET_CPT, kBackRows = kBackTy * kCpt;

template <int FORM>  // 0: decided at run time, 1: terrain layers (palette gamma), 2: general layers
__device__ __forceinline__ double back1_alam(const DetArgs& d, size_t base, size_t tb, size_t tr, int i, double& lam,
                                             double& e, double& p_ig, double& a_newly, double& un) {
  lam = d.traj_lam[tr + i];
  const int env = static_cast<int>(blockIdx.y);
  const double gam = FORM == 1 ? d.s.pal64[256 + d.s.fuel[static_cast<size_t>(env) * d.s.ter_stride + i]]
                     : FORM == 2 ? d.gam[tb + i] : gamma_at(d, tb, env, i);
  const double x = __dmul_rn(gam, lam);
  e = exp_neg(x);
  p_ig = __dsub_rn(1.0, e);
  un = d.traj_un[tr + i];
  a_newly = d.A_burn[base + i] - d.A_un[base + i];
  const double a_x = a_newly * un * e;  // dp_ig/dx = e^{-x} (Dual's exp)
  return a_x * gam;
}

#ifndef EBL_DET_BACK_MINB
#define EBL_DET_BACK_MINB 5  // 48 registers: 5 CTAs per SM (kCpt 2: a few spilled bytes, still faster than 4 CTAs)
#endif
// Tile of 32 x (8 kCpt) cells, 256 threads; thread (tx, ty) owns rows ty, ty + 8, ... (C4 backward:
// kCpt 1 23.3 ms, 2 20.8 ms, 4 21.0 ms per run)
template <int FORM>
__global__ void __launch_bounds__(kBackTx * kBackTy, EBL_DET_BACK_MINB) k_det_back(DetArgs d, int t) {
  __shared__ double red[6 * 32];
  __shared__ double s_al[kBackRows + 2][kBackTx + 2];
  const StepArgs& a = d.s;
  const int h = a.h, w = a.w, ncell = h * w;
  const int env = blockIdx.y;
  const int tiles_x = (w + kBackTx - 1) / kBackTx;
  const int c0 = (blockIdx.x % tiles_x) * kBackTx, r0 = (blockIdx.x / tiles_x) * kBackRows;
  const int tx = threadIdx.x & (kBackTx - 1), ty = threadIdx.x / kBackTx;
  const int c = c0 + tx;
  const size_t base = static_cast<size_t>(env) * ncell;
  const size_t tb = static_cast<size_t>(env) * d.tab_stride;
  const size_t tr = static_cast<size_t>(t) * a.n_envs * ncell + base;
  double g_gamma = 0.0, g_pc = 0.0, bu[kCpt], Ab[kCpt], Ad[kCpt];
  // ---- back1 of the own cells ----
#pragma unroll
  for (int q = 0; q < kCpt; ++q) {
    const int r = r0 + ty + kBackTy * q, i = r * w + c;
    double al = 0.0;
    bu[q] = Ab[q] = Ad[q] = 0.0;
    if (r < h && c < w) {
      double lam, e, p_ig, a_newly, un;
      al = back1_alam<FORM>(d, base, tb, tr, i, lam, e, p_ig, a_newly, un);
      bu[q] = d.traj_burn[tr + i];
      Ab[q] = d.A_burn[base + i];
      Ad[q] = d.A_bd[base + i];
      d.A_un_o[base + i] = d.A_un[base + i] + a_newly * p_ig;
      const double F = FORM == 2 ? d.fac_F[tb + i] : a.pal64[768 + a.fuel[static_cast<size_t>(env) * a.ter_stride + i]];
      g_gamma += (a_newly * un * e) * lam * F;  // dgamma/dalpha_gamma = F(v)
      g_pc += bu[q] * (Ab[q] - Ad[q]);
    }
    s_al[ty + kBackTy * q + 1][tx + 1] = al;
  }
  // ---- back1 of the ring (a_lambda only) ----
  constexpr int kRing = 2 * (kBackTx + 2) + 2 * kBackRows;
  for (int q = threadIdx.x; q < kRing; q += blockDim.x) {
    int sy, sx;
    if (q < kBackTx + 2) sy = 0, sx = q;
    else if (q < 2 * (kBackTx + 2)) sy = kBackRows + 1, sx = q - (kBackTx + 2);
    else sy = 1 + ((q - 2 * (kBackTx + 2)) >> 1), sx = ((q - 2 * (kBackTx + 2)) & 1) ? kBackTx + 1 : 0;
    const int vr = r0 + sy - 1, vc = c0 + sx - 1;
    double al = 0.0;
    if (vr >= 0 && vr < h && vc >= 0 && vc < w) {
      double lam, e, p_ig, a_newly, un;
      al = back1_alam<FORM>(d, base, tb, tr, vr * w + vc, lam, e, p_ig, a_newly, un);
    }
    s_al[sy][sx] = al;
  }
  __syncthreads();
  // ---- back2 of the own cells (source u = (r, c), targets u + d_k) ----
  double gp = 0.0, gw1 = 0.0, gw2 = 0.0, gs = 0.0;
#pragma unroll
  for (int q = 0; q < kCpt; ++q) {
    const int r = r0 + ty + kBackTy * q, i = r * w + c, sy = ty + kBackTy * q + 1, sx = tx + 1;
    if (r >= h || c >= w) continue;
    double acc_burn = Ab[q] * d.pc + Ad[q] * (1.0 - d.pc);
    if (FORM == 2 && bu[q] != 0.0) {  // general form: host-built derivative factors
      const size_t o = tb + i;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int vr = r + kDy[k], vc = c + kDx[k];
        if (vr < 0 || vr >= h || vc < 0 || vc >= w) continue;
        const double al = s_al[sy + kDy[k]][sx + kDx[k]];
        if (al == 0.0) continue;
        const double pot = d.pot[o * 8 + k];
        acc_burn += al * pot;
        const double ab = al * bu[q];
        gp += ab * d.fac_pb[o * 8 + k];
        gw1 += ab * pot * d.fac_V[o];
        gw2 += ab * pot * d.fac_Va[o * 8 + k];
        gs += ab * pot * d.fac_S[o * 8 + k];
      }
    } else if (FORM == 1 && bu[q] != 0.0) {
      const TerrainView tv = terrain_view(a, env);
      const float* slope = a.slope32 ? a.slope32 + static_cast<size_t>(env) * a.ter_stride * 8 : nullptr;
      const double V = d.V[env * d.wind_stride];
      double potk[8];  // the source's 8 pot entries, 64 contiguous bytes requested at once
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        const double2 pp = *reinterpret_cast<const double2*>(d.pot + (tb + i) * 8 + k);
        potk[k] = pp.x;
        potk[k + 1] = pp.y;
      }
      float sown[8];
      if (slope) {
        const float4 s0 = *reinterpret_cast<const float4*>(slope + static_cast<size_t>(i) * 8);
        const float4 s1 = *reinterpret_cast<const float4*>(slope + static_cast<size_t>(i) * 8 + 4);
        sown[0] = s0.x, sown[1] = s0.y, sown[2] = s0.z, sown[3] = s0.w;
        sown[4] = s1.x, sown[5] = s1.y, sown[6] = s1.z, sown[7] = s1.w;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int vr = r + kDy[k], vc = c + kDx[k];
        if (vr < 0 || vr >= h || vc < 0 || vc >= w) continue;
        const double al = s_al[sy + kDy[k]][sx + kDx[k]];
        if (al == 0.0) continue;
        const double pot = potk[k];
        acc_burn += al * pot;
        // pot = p_base F kw ks (kernel.hpp:21-45): dpot/dp_base = F kw ks, dpot/dalpha_w1 = pot V,
        // dpot/dalpha_w2 = pot V (cos - 1), dpot/dalpha_s = pot S; S in fp32 (relative error ~1e-7,
        // far inside the 1e-4 gradient bar)
        double S;
        if (slope) {
          S = -static_cast<double>(sown[(k + 4) & 7]);  // u's record, direction k+4: source v
        } else {
          const float dz = tv.elev[vr * w + vc] - tv.elev[i];
          S = dz == dz ? static_cast<double>(atanf(dz * tv.inv_dist32[k & 1])) : 0.0;  // nodata: 0
        }
        const double ab = al * bu[q];
        gp += ab * (pot * d.inv_p_base);
        gw1 += ab * pot * V;
        gw2 += ab * pot * V * d.align[env * d.wind_stride * 8 + k];
        gs += ab * pot * S;
      }
    }
    d.A_burn_o[base + i] = acc_burn;  // A_bd is unchanged (bd' = bd + ...)
  }
  double g6[6] = {gp, gw1, gw2, gs, g_gamma, g_pc};
  block_sum_n<6>(g6, red);
  if (threadIdx.x == 0) {
    double* acc = d.acc + (static_cast<size_t>(env) * gridDim.x + blockIdx.x) * 8;
#pragma unroll
    for (int k = 0; k < 6; ++k) acc[k] += g6[k];
  }
}

#ifndef EBL_DET_STREAM
#define EBL_DET_STREAM 1  // row-streaming backward with bulk asynchronous copies (terrain layers)
#endif

// ---- row-streaming backward (terrain layers, W <= 128, W % 16 == 0) ----------------------------
// One CTA per (env, band of kSB rows), one thread per column.  The dense per-cell inputs of every
// row (lambda, p_un, p_burn of step t, the three adjoints, the fuel class) are streamed into a ring
// of shared-memory stages by bulk asynchronous copies (cp.async.bulk, completion on an mbarrier)
// kSD rows ahead, so the SM keeps ~tens of KB in flight without per-thread loads; each source's pot
// and slope records (needed only where p_burn != 0) are requested one step of the loop early.  Row
// q: back1 (a_lambda into a 3-row ring, A_un' of band rows), then back2 of row q-1 (A_burn', the
// pot-parameter gradients).  Same arithmetic per cell as k_det_back; the band's halo rows get
// their a_lambda recomputed (bit-identical inputs).  Gradient partials per (env, band), reduced in
// a fixed order by k_det_reduce.
#ifndef EBL_DET_SB
#define EBL_DET_SB 16  // C4 at 1 row ahead: 16 rows 15.07 ms, 10: 15.29, 13: 15.49, 21: 16.19, 26: 16.68, 32: 15.11
#endif
constexpr int kSB = EBL_DET_SB;  // rows per band
#ifndef EBL_DET_SD
#define EBL_DET_SD 1  // C4 run: 1 row (7 CTAs/SM) 15.07 ms, 2 rows (6 CTAs/SM) 15.80-16.15, 3 rows 17.6, 4 rows 19.2
#endif
constexpr int kSD = EBL_DET_SD;  // rows requested ahead
constexpr int kSlots = kSD + 3;  // + the rows back1 and back2 read, + the one refilled this iteration
constexpr int kAl = 4;        // a_lambda ring: back2 of row q-1 reads rows q-2..q while back1 writes q+1
constexpr int kSW = 128;      // max columns
struct StreamRow {
  double lam[kSW], un[kSW], burn[kSW], au[kSW], ab[kSW], ad[kSW];
  uint8_t fuel[kSW];
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_addr(bar)),
      "r"(phase)
      : "memory");
}

__global__ void __launch_bounds__(kSW, EBL_DET_SD <= 1 ? 7 : (EBL_DET_SD <= 2 ? 6 : 5)) k_det_back_stream(DetArgs d, int t) {
  pdl_enter();
  extern __shared__ __align__(128) uint8_t dsm[];
  StreamRow* const st = reinterpret_cast<StreamRow*>(dsm);
  double (*const alam)[kSW + 2] = reinterpret_cast<double (*)[kSW + 2]>(dsm + kSlots * sizeof(StreamRow));
  auto al_row = [&](int q) { return alam[(q + kAl) % kAl]; };
  __shared__ __align__(8) uint64_t bar[kSlots];
  __shared__ double red[6 * 32];
  const StepArgs& a = d.s;
  const int h = a.h, w = a.w, ncell = h * w;
  const int env = blockIdx.y;
  const int r0 = blockIdx.x * kSB, r1 = min(h, r0 + kSB);
  const int qa = max(0, r0 - 1), qb = min(h - 1, r1);  // rows whose a_lambda the band needs
  const int c = threadIdx.x;
  const bool col = c < w;
  const size_t base = static_cast<size_t>(env) * ncell;
  const size_t tr = static_cast<size_t>(t) * a.n_envs * ncell + base;
  const uint8_t* fuel = a.fuel + static_cast<size_t>(env) * a.ter_stride;
  const unsigned rowb = static_cast<unsigned>(w) * 8u;
  auto issue = [&](int q) {  // one thread: the stage of row q (6 dense rows + the fuel row)
    const int slot = (q - qa) % kSlots;
    StreamRow& S = st[slot];
    const size_t o = static_cast<size_t>(q) * w;
    mbar_expect_tx(&bar[slot], 6 * rowb + static_cast<unsigned>(w));
    bulk_g2s(S.lam, d.traj_lam + tr + o, rowb, &bar[slot]);
    bulk_g2s(S.un, d.traj_un + tr + o, rowb, &bar[slot]);
    bulk_g2s(S.burn, d.traj_burn + tr + o, rowb, &bar[slot]);
    bulk_g2s(S.au, d.A_un + base + o, rowb, &bar[slot]);
    bulk_g2s(S.ab, d.A_burn + base + o, rowb, &bar[slot]);
    bulk_g2s(S.ad, d.A_bd + base + o, rowb, &bar[slot]);
    bulk_g2s(S.fuel, fuel + o, static_cast<unsigned>(w), &bar[slot]);
  };
  if (c < kSlots) mbar_init(&bar[c], 1);
  for (int i = c; i < kAl * (kSW + 2); i += blockDim.x) (&alam[0][0])[i] = 0.0;  // OOB rows / columns
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  if (c == 0)
    for (int q = qa; q <= qb && q < qa + kSlots; ++q) issue(q);

  const double pc = d.pc, qc = 1.0 - d.pc;
  const double V = d.V[env * d.wind_stride];
  const double* align = d.align + env * d.wind_stride * 8;
  const float* slope = a.slope32 + static_cast<size_t>(env) * a.ter_stride * 8;
  const double* pot = d.pot + static_cast<size_t>(env) * d.tab_stride * 8;
  double g_gamma = 0.0, g_pc = 0.0, gp = 0.0, gw1 = 0.0, gw2 = 0.0, gs = 0.0;
  double potk[8];
  float sown[8];
  for (int q = qa; q <= r1; ++q) {
    // ---- the source records of row q-1 (back2 below), requested before this row's wait ----
    const int rs = q - 1;
    const bool b2 = rs >= r0 && rs < r1;
    double bu = 0.0;
    if (b2 && col) {
      bu = st[(rs - qa) % kSlots].burn[c];
      if (bu != 0.0) {  // into L1 now (two lines of pot, one of slope), read after back1
        const size_t i = static_cast<size_t>(rs) * w + c;
        asm volatile("prefetch.global.L1 [%0];" ::"l"(pot + i * 8));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(pot + i * 8 + 4));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(slope + i * 8));
      }
    }
    // ---- back1 of row q (a real row), or an all-zero a_lambda row below the landscape ----
    double* al_q = al_row(q);
    if (q <= qb) {
      const int slot = (q - qa) % kSlots;
      mbar_wait(&bar[slot], static_cast<unsigned>(((q - qa) / kSlots) & 1));
      const StreamRow& S = st[slot];
      double al = 0.0;
      if (col) {
        const int f = S.fuel[c];
        const double lam = S.lam[c], gam = a.pal64[256 + f];
        const double x = __dmul_rn(gam, lam);
        const double e = exp_neg(x);
        const double p_ig = __dsub_rn(1.0, e);
        const double un = S.un[c];
        const double a_newly = S.ab[c] - S.au[c];
        const double a_x = a_newly * un * e;  // dp_ig/dx = e^{-x} (Dual's exp)
        al = a_x * gam;
        if (q >= r0 && q < r1) {
          d.A_un_o[base + static_cast<size_t>(q) * w + c] = S.au[c] + a_newly * p_ig;
          g_gamma += a_x * lam * a.pal64[768 + f];  // dgamma/dalpha_gamma = F(v)
          g_pc += S.burn[c] * (S.ab[c] - S.ad[c]);
        }
      }
      al_q[c + 1] = al;
    } else {
      al_q[c + 1] = 0.0;
    }
    __syncthreads();  // a_lambda of rows q-2 .. q complete; every thread is past back2 of row q-2
    if (c == 0 && q - 2 >= qa) {  // the stage of row q-2 is free: refill it kSlots rows later
      const int nq = q - 2 + kSlots;
      if (nq <= qb) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(nq);
      }
    }
    // ---- back2 of row q-1 (source u = (rs, c), targets u + d_k) ----
    if (b2 && col) {
      const StreamRow& S = st[(rs - qa) % kSlots];
      double acc_burn = S.ab[c] * pc + S.ad[c] * qc;
      if (bu != 0.0) {
        const size_t i = static_cast<size_t>(rs) * w + c;
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
          const double2 pp = __ldg(reinterpret_cast<const double2*>(pot + i * 8 + k));
          potk[k] = pp.x;
          potk[k + 1] = pp.y;
        }
        const float4 s0 = __ldg(reinterpret_cast<const float4*>(slope + i * 8));
        const float4 s1 = __ldg(reinterpret_cast<const float4*>(slope + i * 8 + 4));
        sown[0] = s0.x, sown[1] = s0.y, sown[2] = s0.z, sown[3] = s0.w;
        sown[4] = s1.x, sown[5] = s1.y, sown[6] = s1.z, sown[7] = s1.w;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int vr = rs + kDy[k], vc = c + kDx[k];
          if (vr < 0 || vr >= h || vc < 0 || vc >= w) continue;
          const double al = al_row(vr)[vc + 1];
          if (al == 0.0) continue;
          const double pt = potk[k];
          acc_burn += al * pt;
          // dpot/dp_base = pot / p_base, dpot/dalpha_w1 = pot V, dpot/dalpha_w2 = pot V (cos - 1),
          // dpot/dalpha_s = pot S; S of direction k = the source's own record of k + 4, negated
          const double S_k = -static_cast<double>(sown[(k + 4) & 7]);
          const double ab = al * bu;
          gp += ab * (pt * d.inv_p_base);
          gw1 += ab * pt * V;
          gw2 += ab * pt * V * align[k];
          gs += ab * pt * S_k;
        }
      }
      d.A_burn_o[base + static_cast<size_t>(rs) * w + c] = acc_burn;  // A_bd is unchanged
    }
  }
  double g6[6] = {gp, gw1, gw2, gs, g_gamma, g_pc};
  block_sum_n<6>(g6, red);
  if (threadIdx.x == 0) {
    double* acc = d.acc + (static_cast<size_t>(env) * gridDim.x + blockIdx.x) * 8;
#pragma unroll
    for (int k = 0; k < 6; ++k) acc[k] += g6[k];
  }
}


bool det_stream_ok(const DetArgs& d) {  // terrain layers, whole rows of <= 128 cells, 16-byte rows
  return !d.fac_pb && d.s.fuel && d.s.slope32 && d.s.w <= kSW && (d.s.w % 16) == 0;
}

size_t det_stream_smem() { return kSlots * sizeof(StreamRow) + kAl * (kSW + 2) * sizeof(double); }

int det_blocks_per_env_stream(int h) { return (h + kSB - 1) / kSB; }

// SpreadTables<double>::pot of terrain layers built on the device (engine.hpp:88-107 /
// build_terrain_tables): pot[t][cell][k] = (source(class) kappa_wind_t(k)) exp(alpha_s S[g][cell][k])
// with S the cached config-free slopes (host atan, once per terrain), source the palette's fp64
// value and exp the restatement of the reference's libm exp (ember_exp.cuh): bit-identical to the
// host-built table, so a config change (every calibration iteration) needs no host rebuild.
__device__ const uint64_t kExpTabDev[256] = EBL_EXP_TAB_INIT;

__global__ void k_det_tables_terrain(const double* __restrict__ S, const uint8_t* __restrict__ fuel,
                                     const double* __restrict__ pal64, const double* __restrict__ kw64, double alpha_s,
                                     int n_tables, size_t ncell, size_t grid_stride, int wind_stride, double* pot) {
  __shared__ uint64_t tab[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) tab[i] = kExpTabDev[i];
  __syncthreads();
  const size_t total = static_cast<size_t>(n_tables) * ncell * 8;
  for (size_t j = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < total;
       j += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t tcell = j >> 3;
    const int k = static_cast<int>(j & 7);
    const int t = static_cast<int>(tcell / ncell);
    const size_t cell = tcell - static_cast<size_t>(t) * ncell;
    const size_t g = grid_stride ? static_cast<size_t>(t) : 0;  // grid of table t
    const double src = pal64[fuel[g * ncell + cell]];
    const double kw = kw64[static_cast<size_t>(t) * wind_stride * 8 + k];
    bool exact = true;
    const double ks = exp_glibc(__dmul_rn(alpha_s, S[(g * ncell + cell) * 8 + k]), tab, &exact);
    pot[j] = __dmul_rn(__dmul_rn(src, kw), ks);
  }
}

cudaError_t launch_det_tables_terrain(const double* S, const uint8_t* fuel, const double* pal64, const double* kw64,
                                      double alpha_s, int n_tables, size_t ncell, size_t grid_stride, int wind_stride,
                                      double* pot, cudaStream_t s) {
  const size_t total = static_cast<size_t>(n_tables) * ncell * 8;
  const unsigned blocks = static_cast<unsigned>(std::min<size_t>((total + 255) / 256, 148 * 8));
  k_det_tables_terrain<<<blocks, 256, 0, s>>>(S, fuel, pal64, kw64, alpha_s, n_tables, ncell, grid_stride, wind_stride,
                                              pot);
  return cudaGetLastError();
}

int det_blocks_per_env(int h, int w) {
  return ((w + kBackTx - 1) / kBackTx) * ((h + kBackRows - 1) / kBackRows);
}

__global__ void k_det_reduce(DetArgs d, int blocks_per_env) {
  const int env = blockIdx.x;
  const int k = threadIdx.x;
  if (k >= 6) return;
  double s = 0.0;
  for (int b = 0; b < blocks_per_env; ++b) s += d.acc[(static_cast<size_t>(env) * blocks_per_env + b) * 8 + k];
  d.grad[env * 6 + k] = s;
}

// p_bd of a recorded run (record mode): p_bd never feeds back into the dynamics, so
// the forward steps skip it (16 B per cell-step) and this pass replays the reference's per-step
// update p_bd += p_burn(t) (1 - p_continue) (engine.hpp:164-167) over the recorded p_burn planes, in
// step order -- the same fp64 operations in the same order, so the same bits.
__global__ void k_det_bd_run(const double* __restrict__ bd0, double* bd_out, const double* __restrict__ traj_burn,
                             size_t n, int n_steps, double pc) {
  pdl_enter();
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double q = __dsub_rn(1.0, pc);
  double bd = bd0[i];
#pragma unroll 8
  for (int t = 0; t < n_steps; ++t) bd = __dadd_rn(bd, __dmul_rn(__ldg(traj_burn + static_cast<size_t>(t) * n + i), q));
  bd_out[i] = bd;
}

cudaError_t launch_det_bd_run(const double* bd0, double* bd_out, const double* traj_burn, size_t n, int n_steps,
                              double pc, cudaStream_t s) {
  return launch_pdl(k_det_bd_run, dim3(static_cast<unsigned>((n + 255) / 256)), dim3(256), 0, s, bd0, bd_out,
                    traj_burn, n, n_steps, pc);
}

cudaError_t launch_det_forward(const DetArgs& d, int t, cudaStream_t s) {
  const int ncell = d.s.h * d.s.w;
  if (EBL_DET_FWD2 && d.potT && (d.s.w % 2) == 0) {
    return launch_pdl(k_det_forward2, dim3((ncell / 2 + EBL_DET_FWD_THREADS - 1) / EBL_DET_FWD_THREADS, d.s.n_envs),
                      dim3(EBL_DET_FWD_THREADS), 0, s, d, t);
  }
  k_det_forward<<<dim3((ncell + 255) / 256, d.s.n_envs), 256, 0, s>>>(d, t);
  return cudaGetLastError();
}

cudaError_t launch_det_from_fire(const uint8_t* st, double* un, double* bu, double* bd, size_t n,
                                 cudaStream_t s) {
  k_det_from_fire<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(st, un, bu, bd, n);
  return cudaGetLastError();
}

cudaError_t launch_det_loss(const DetArgs& d, cudaStream_t s) {
  k_det_loss<<<d.s.n_envs, EBL_DET_LOSS_THREADS, 0, s>>>(d);
  return cudaGetLastError();
}

cudaError_t launch_det_backward(const DetArgs& d, int t, cudaStream_t s) {
  const int ncell = d.s.h * d.s.w;
  const dim3 grid((ncell + 255) / 256, d.s.n_envs);
  if (EBL_DET_STREAM && det_stream_ok(d) && d.A_un_o) {
    const size_t sm = det_stream_smem();
    cudaError_t e = smem_opt_in(reinterpret_cast<const void*>(k_det_back_stream), sm);
    if (e != cudaSuccess) return e;
    return launch_pdl(k_det_back_stream, dim3(det_blocks_per_env_stream(d.s.h), d.s.n_envs), dim3(kSW), sm, s, d, t);
  }
  if (d.A_un_o) {  // fused, double-buffered adjoints
    const dim3 g(det_blocks_per_env(d.s.h, d.s.w), d.s.n_envs);
    if (d.fac_pb) k_det_back<2><<<g, kBackTx * kBackTy, 0, s>>>(d, t);  // general layers
    else k_det_back<1><<<g, kBackTx * kBackTy, 0, s>>>(d, t);           // terrain layers
    return cudaGetLastError();
  }
  k_det_back1<<<grid, 256, 0, s>>>(d, t);
  k_det_back2<<<grid, 256, 0, s>>>(d, t);
  return cudaGetLastError();
}

cudaError_t launch_det_reduce(const DetArgs& d, cudaStream_t s) {
  const int ncell = d.s.h * d.s.w;
  const int bpe = EBL_DET_STREAM && det_stream_ok(d) && d.A_un_o ? det_blocks_per_env_stream(d.s.h)
                  : d.A_un_o ? det_blocks_per_env(d.s.h, d.s.w) : (ncell + 255) / 256;
  k_det_reduce<<<d.s.n_envs, 32, 0, s>>>(d, bpe);
  return cudaGetLastError();
}

}  // namespace ebl
