// Kernels of the stochastic CA step (general tiled path), the intensity probe,
// per-env statistics and the RL step.  See DESIGN.md for layout and rooflines.
#include <cuda_runtime.h>

#include <cstdint>

#include "ember_device.cuh"
#include "ember_kernels.h"
#include "ember_params.h"

namespace ebl {

// Block-wide sum of 4 counters, then one atomicAdd each into counts[env].
__device__ __forceinline__ void flush_counts(int32_t* counts, int env, int32_t v0, int32_t v1,
                                             int32_t v2, int32_t v3) {
  __shared__ int32_t red[4];
  if (threadIdx.x < 4) red[threadIdx.x] = 0;
  __syncthreads();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v0 += __shfl_xor_sync(0xffffffffu, v0, o);
    v1 += __shfl_xor_sync(0xffffffffu, v1, o);
    v2 += __shfl_xor_sync(0xffffffffu, v2, o);
    v3 += __shfl_xor_sync(0xffffffffu, v3, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&red[0], v0);
    atomicAdd(&red[1], v1);
    atomicAdd(&red[2], v2);
    atomicAdd(&red[3], v3);
  }
  __syncthreads();
  if (threadIdx.x < 4) atomicAdd(counts + env * 4 + threadIdx.x, red[threadIdx.x]);
}

// ---------------------------------------------------------------------------------
// General tiled step: one launch = one synchronous step of every env
// (step_stochastic_into, engine.cpp:28-38, over the batch as step_batch does,
// engine.cpp:134-159).  CTA = TILE_H x TILE_W cells of one env; the tile plus a
// 1-cell halo of states is staged in shared memory so each state byte is read
// from HBM ~once; OOB halo cells are staged as Unburned, which is exactly the
// reference's "skip out-of-bounds neighbour" (kernel.hpp:61).
// ---------------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(kTileThreads) k_step_tile(StepArgs a) {
  __shared__ uint8_t tile[kTileH + 2][kTileW + 4];
  const int env = blockIdx.z;
  const int r0 = blockIdx.y * kTileH, c0 = blockIdx.x * kTileW;
  const int H = a.h, W = a.w;
  const size_t ncell = static_cast<size_t>(H) * W;
  const uint8_t* __restrict__ in = a.in + env * ncell;
  uint8_t* __restrict__ out = a.out + env * ncell;

  for (int idx = threadIdx.x; idx < (kTileH + 2) * (kTileW + 2); idx += kTileThreads) {
    const int rr = idx / (kTileW + 2), cc = idx - rr * (kTileW + 2);
    const int gr = r0 - 1 + rr, gc = c0 - 1 + cc;
    uint8_t v = 0;
    if (gr >= 0 && gr < H && gc >= 0 && gc < W) v = in[static_cast<size_t>(gr) * W + gc];
    tile[rr][cc] = v;
  }
  __syncthreads();

  const uint64_t prefix = key_prefix(a.seed, a.streams[env], a.step);
  const DiagCounters dg{a.diag};
  int32_t nU = 0, nB = 0, nX = 0, nNew = 0;
  const int lc = threadIdx.x % kTileW;
#pragma unroll
  for (int j = 0; j < kTileH * kTileW / kTileThreads; ++j) {
    const int lr = threadIdx.x / kTileW + j * (kTileThreads / kTileW);
    const int r = r0 + lr, c = c0 + lc;
    if (r >= H || c >= W) continue;
    const uint8_t s = tile[lr + 1][lc + 1];
    uint8_t ns = 2;
    if (s == 1) {
      ns = cell_bits53(prefix, static_cast<uint64_t>(a.row_off + r) * W + c, 0) < a.pc_thr ? 1 : 2;
    } else if (s != 2) {  // any other byte takes the Unburned path (engine.cpp:15-25)
      uint32_t nb = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) nb |= static_cast<uint32_t>(tile[lr + 1 - kDy[k]][lc + 1 - kDx[k]] == 1) << k;
      ns = 0;
      if (nb) {
        const uint64_t m = cell_bits53(prefix, static_cast<uint64_t>(a.row_off + r) * W + c, 0);
        ns = ignite<MODE>(a, env, r, c, nb, m, dg, sched_row(a, a.step)) ? 1 : 0;
        nNew += ns;
      }
    }
    out[static_cast<size_t>(r) * W + c] = ns;
    nU += ns == 0;
    nB += ns == 1;
    nX += ns == 2;
  }
  if (a.counts) flush_counts(a.counts, env, nU, nB, nX, nNew);
}

// Intensity / probability probe (kernel.hpp:53-78) of the current state; tables
// form reports the fp64 values rounded to float, terrain the fp32 fast path.
template <int MODE>
__global__ void k_intensity(StepArgs a, float* lam_out, float* p_out) {
  const size_t ncell = static_cast<size_t>(a.h) * a.w;
  const size_t total = ncell * a.n_envs;
  for (size_t g = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int env = static_cast<int>(g / ncell);
    const int i = static_cast<int>(g - env * ncell);
    const int r = i / a.w, c = i - r * a.w;
    const uint8_t* st = a.in + env * ncell;
    uint32_t nb = 0;
    for (int k = 0; k < 8; ++k) {
      const int ur = r - kDy[k], uc = c - kDx[k];
      if (ur < 0 || ur >= a.h || uc < 0 || uc >= a.w) continue;
      nb |= static_cast<uint32_t>(st[ur * a.w + uc] == 1) << k;
    }
    float lam = 0.f, p = 0.f;
    if constexpr (MODE == kStaticTables) {
      const size_t base = static_cast<size_t>(env) * a.tab_stride;
      const double* pot = a.pot + static_cast<size_t>(sched_row(a, a.step)) * a.pot_sched_stride;
      double l = 0.0;
      for (int k = 0; k < 8; ++k)
        if (nb & (1u << k))
          l = __dadd_rn(l, pot[(base + (r - kDy[k]) * a.w + (c - kDx[k])) * 8 + k]);
      lam = static_cast<float>(l);
      p = static_cast<float>(__dsub_rn(1.0, exp(-__dmul_rn(a.gamma[base + i], l))));
    } else {
      const TerrainView t = terrain_view(a, env, sched_row(a, a.step));
      if (a.nfuel && a.slope32 && a.n_pal <= 32 && a.rec_probe) {
        // the resident kernels' form (ember_device.cuh terrain_lambda32_rec): slope + source-class
        // records, src32 * kappa_wind32 products, 2^(alpha_s log2e S)
        float srckw[32 * 8];
        for (int q = 0; q < a.n_pal * 8; ++q) srckw[q] = t.pal_src32[q >> 3] * t.kw32[q & 7];
        lam = terrain_lambda32_rec(a.slope32 + static_cast<size_t>(env) * a.ter_stride * 8,
                                   a.nfuel + static_cast<size_t>(env) * a.ter_stride, srckw, a.alpha_s_l2, i, nb);
        p = p_ignite32(t.pal_gam32[t.fuel[i]] * lam);  // the warp kernels' p
      } else {
        lam = terrain_lambda32(t, a.w, r, c, nb);
        p = -expm1f(-t.pal_gam32[t.fuel[i]] * lam);
      }
    }
    lam_out[g] = lam;
    p_out[g] = p;
  }
}

__global__ void k_counts(const uint8_t* __restrict__ st, int ncell, int32_t* counts) {
  const int env = blockIdx.x;
  int32_t nU = 0, nB = 0, nX = 0;
  for (int i = threadIdx.x; i < ncell; i += blockDim.x) {
    const uint8_t s = st[static_cast<size_t>(env) * ncell + i];
    nU += s == 0;
    nB += s == 1;
    nX += s == 2;
  }
  flush_counts(counts, env, nU, nB, nX, 0);
}

// ---------------------------------------------------------------------------------
// RL step kernels: one CTA per env, the env's layer resident in shared memory.
// ---------------------------------------------------------------------------------
template <int MODE>
__device__ __forceinline__ uint8_t rl_cell(const StepArgs& a, int env, const uint8_t* cur, int r,
                                           int c, uint64_t prefix, const DiagCounters& dg) {
  const int W = a.w, H = a.h;
  const uint8_t s = cur[r * W + c];
  if (s == 2) return 2;
  if (s == 1) return cell_bits53(prefix, static_cast<uint64_t>(r) * W + c, 0) < a.pc_thr ? 1 : 2;
  uint32_t nb = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int ur = r - kDy[k], uc = c - kDx[k];
    if (ur < 0 || ur >= H || uc < 0 || uc >= W) continue;
    nb |= static_cast<uint32_t>(cur[ur * W + uc] == 1) << k;
  }
  if (!nb) return 0;
  const uint64_t m = cell_bits53(prefix, static_cast<uint64_t>(r) * W + c, 0);
  return ignite<MODE>(a, env, r, c, nb, m, dg) ? 1 : 0;
}

__device__ __forceinline__ int block_sum(int v) {
  __shared__ int red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  int t = 0;
  for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) t += red[i];
  return t;
}

// FireSuppressionEnv::step (rl_env.cpp:172-210), one env per CTA.
template <int MODE>
__global__ void __launch_bounds__(kRlThreads) k_rl_ref_step(RlArgs g) {
  extern __shared__ uint8_t smem[];
  const StepArgs& a = g.s;
  const int env = blockIdx.x;
  const int H = a.h, W = a.w, n = H * W;
  uint8_t* cur = smem;
  uint8_t* st = g.state + static_cast<size_t>(env) * n;
  RlEnv e = g.env[env];
  if (e.done) {  // logic_error in the reference; leave the env untouched
    if (threadIdx.x == 0) atomicExch(g.error, 1);
    return;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) cur[i] = st[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    const int act = g.actions ? g.actions[env]
                              : static_cast<int>(below(cell_bits53(key_prefix(e.seed, e.stream,
                                                                              static_cast<uint64_t>(e.step)),
                                                                   0, 2),
                                                       10));
    const int move = act / 2, open = act % 2;
    if (move == 0) e.row = min(e.row + 1, H - 1);
    else if (move == 1) e.row = max(e.row - 1, 0);
    else if (move == 2) e.col = min(e.col + 1, W - 1);
    else if (move == 3) e.col = max(e.col - 1, 0);
    if (open && e.water > 0) {
      const int ai = e.row * W + e.col;
      const bool on_fire = cur[ai] == 1;
      if (on_fire) cur[ai] = 2;
      if (on_fire || g.waste_water) e.water -= 1;
    }
  }
  __syncthreads();
  const uint64_t prefix = key_prefix(e.seed, e.stream, static_cast<uint64_t>(e.step));
  const DiagCounters dg{a.diag};
  int burning = 0, touched = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const uint8_t v = rl_cell<MODE>(a, env, cur, i / W, i % W, prefix, dg);
    st[i] = v;
    burning += v == 1;
    touched += v != 0;
  }
  burning = block_sum(burning);
  touched = block_sum(touched);
  if (threadIdx.x == 0) {
    e.step += 1;
    double reward = -g.burn_penalty * static_cast<double>(burning);
    if (burning == 0 && touched > 0) reward += 10.0;  // kTerminalBonus (rl_env.hpp:42)
    e.done = (burning == 0 || e.step >= g.max_episode_steps) ? 1 : 0;
    g.env[env] = e;
    if (g.reward) g.reward[env] = reward;
    if (g.done) g.done[env] = static_cast<uint8_t>(e.done);
  }
}

// Observation (rl_env.cpp:147-170): one thread per (env, output slot).
__global__ void k_rl_observe(const uint8_t* state, const RlEnv* envs, int n_envs, int H, int W,
                             int radius, int capacity, double* obs) {
  const int side = 2 * radius + 1;
  const int osz = 3 * side * side + 3;
  const size_t total = static_cast<size_t>(n_envs) * osz;
  for (size_t g = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int env = static_cast<int>(g / osz);
    const int o = static_cast<int>(g - static_cast<size_t>(env) * osz);
    const RlEnv e = envs[env];
    double v = 0.0;
    if (o < 3 * side * side) {
      const int cellw = o / 3, ch = o % 3;
      const int dy = radius - cellw / side, dx = cellw % side - radius;
      const int row = e.row + dy, col = e.col + dx;
      if (row >= 0 && row < H && col >= 0 && col < W)
        v = state[static_cast<size_t>(env) * H * W + row * W + col] == ch ? 1.0 : 0.0;
    } else if (o == 3 * side * side) {
      v = static_cast<double>(e.water) / capacity;
    } else if (o == 3 * side * side + 1) {
      v = H > 1 ? static_cast<double>(e.row) / (H - 1) : 0.0;
    } else {
      v = W > 1 ? static_cast<double>(e.col) / (W - 1) : 0.0;
    }
    obs[g] = v;
  }
}

// ---- tanker (BASELINE C2) ---------------------------------------------------------
__device__ __forceinline__ uint64_t tanker_stream(uint32_t env_id, uint32_t episode) {
  return (static_cast<uint64_t>(episode) << 32) | env_id;
}

template <int MODE>
__device__ __forceinline__ bool burnable_cell(const StepArgs& a, int env, int i) {
  if constexpr (MODE == kStaticTerrain) {
    const uint8_t cls = a.fuel[static_cast<size_t>(env) * a.ter_stride + i];
    return a.pal64[512 + cls] > 0.5;  // (1+veg)*(1+den) > 0, precomputed per class
  } else {
    return a.gamma[static_cast<size_t>(env) * a.tab_stride + i] > 0.0;
  }
}

// Reset of one env into shared memory (cur, wet): thread 0 draws the ignitions
// exactly like ebo_tanker_reset.  Caller syncs.
template <int MODE>
__device__ void tanker_reset(const RlArgs& g, int env, RlEnv& e, uint8_t* cur, uint8_t* wet, int n,
                             uint32_t episode, int* s_burning) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    cur[i] = 0;
    wet[i] = 0;
  }
  const uint64_t stream = tanker_stream(g.env_id0 + env, episode);
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t prefix = key_prefix(g.seed, stream, 0);
    uint64_t counter = 0;
    const uint64_t max_draws = 64ull * n;
    int placed = 0;
    while (placed < g.ignitions && counter < max_draws) {
      const int cell = static_cast<int>(below(cell_bits53(prefix, counter++, 1), n));
      if (cur[cell] == 1 || !burnable_cell<MODE>(g.s, env, cell)) continue;
      cur[cell] = 1;
      ++placed;
    }
    *s_burning = placed;
  }
  __syncthreads();
  // every thread holds its own copy of the env record: update all copies uniformly
  e.step = 0;
  e.episode = episode;
  e.stream = stream;
  e.done = *s_burning == 0;
}

// n_steps tanker steps of one env per CTA (n_steps = 1 for the per-step API).
template <int MODE>
__global__ void __launch_bounds__(kRlThreads) k_rl_tanker(RlArgs g) {
  extern __shared__ uint8_t smem[];
  __shared__ int s_burning;
  __shared__ int s_action;
  const StepArgs& a = g.s;
  const int env = blockIdx.x;
  const int H = a.h, W = a.w, n = H * W;
  uint8_t* cur = smem;
  uint8_t* wet = smem + n;
  uint8_t* nxt = smem + 2 * n;
  uint8_t* st = g.state + static_cast<size_t>(env) * n;
  uint8_t* wt = g.wet + static_cast<size_t>(env) * n;
  RlEnv e = g.env[env];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    cur[i] = st[i];
    wet[i] = wt[i];
  }
  __syncthreads();
  const DiagCounters dg{a.diag};
  double rsum = 0.0;
  int32_t finished = 0;
  for (int t = 0; t < g.n_steps; ++t) {
    // 1) action (device random policy: rng_below(key{seed,step,stream}, 0, kDrawPolicy, n))
    if (threadIdx.x == 0) {
      s_action = g.actions ? g.actions[env]
                           : static_cast<int>(below(cell_bits53(key_prefix(g.seed, e.stream,
                                                                           static_cast<uint64_t>(e.step)),
                                                                0, 2),
                                                    n));
    }
    __syncthreads();
    // 2) extinguish + wet the 3x3 patch
    if (threadIdx.x < 9) {
      const int r = s_action / W + static_cast<int>(threadIdx.x) / 3 - 1;
      const int c = s_action % W + static_cast<int>(threadIdx.x) % 3 - 1;
      if (r >= 0 && r < H && c >= 0 && c < W) {
        const int i = r * W + c;
        if (cur[i] == 1) cur[i] = 2;
        else if (cur[i] == 0) wet[i] = 1;
      }
    }
    __syncthreads();
    // 3) fire step; wet Unburned cells never ignite
    const uint64_t prefix = key_prefix(g.seed, e.stream, static_cast<uint64_t>(e.step));
    int burning = 0, newly = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const uint8_t s = cur[i];
      uint8_t v = 0;
      if (!(s == 0 && wet[i])) v = rl_cell<MODE>(a, env, cur, i / W, i % W, prefix, dg);
      nxt[i] = v;
      burning += v == 1;
      newly += (s == 0 && v == 1);
    }
    burning = block_sum(burning);
    newly = block_sum(newly);
    for (int i = threadIdx.x; i < n; i += blockDim.x) cur[i] = nxt[i];
    e.step += 1;
    const double reward = -static_cast<double>(newly);
    const bool done = burning == 0 || e.step >= g.max_steps;
    rsum += reward;
    if (g.n_steps == 1 && threadIdx.x == 0) {
      if (g.reward) g.reward[env] = reward;
      if (g.done) g.done[env] = done ? 1 : 0;
    }
    __syncthreads();
    if (done) {
      ++finished;
      tanker_reset<MODE>(g, env, e, cur, wet, n, e.episode + 1, &s_burning);
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    st[i] = cur[i];
    wt[i] = wet[i];
  }
  if (threadIdx.x == 0) {
    g.env[env] = e;
    if (g.reward_sum) g.reward_sum[env] += rsum;
    if (g.episodes) g.episodes[env] += finished;
  }
}

// Reset kernel (both variants' episode start for the tanker).
template <int MODE>
__global__ void __launch_bounds__(kRlThreads) k_rl_tanker_reset(RlArgs g, const uint8_t* mask) {
  extern __shared__ uint8_t smem[];
  __shared__ int s_burning;
  const int env = blockIdx.x;
  if (mask && !mask[env]) return;
  const int n = g.s.h * g.s.w;
  uint8_t* cur = smem;
  uint8_t* wet = smem + n;
  RlEnv e = g.env[env];
  tanker_reset<MODE>(g, env, e, cur, wet, n, 0u, &s_burning);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    g.state[static_cast<size_t>(env) * n + i] = cur[i];
    g.wet[static_cast<size_t>(env) * n + i] = wet[i];
  }
  if (threadIdx.x == 0) g.env[env] = e;
}

__global__ void k_rng_probe(int n, const uint64_t* keys5, uint64_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t* k = keys5 + 5 * i;
  out[i] = mix64(mix64(key_prefix(k[0], k[2], k[1]) ^ k[3]) ^ k[4]);
}

// ---------------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------------
cudaError_t launch_rng_probe(int n, const uint64_t* keys5, uint64_t* out, cudaStream_t s) {
  k_rng_probe<<<(n + 255) / 256, 256, 0, s>>>(n, keys5, out);
  return cudaGetLastError();
}

cudaError_t launch_step_tile(const StepArgs& a, int mode, cudaStream_t s) {
  const dim3 grid((a.w + kTileW - 1) / kTileW, (a.h + kTileH - 1) / kTileH, a.n_envs);
  if (mode == kStaticTables) k_step_tile<kStaticTables><<<grid, kTileThreads, 0, s>>>(a);
  else k_step_tile<kStaticTerrain><<<grid, kTileThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_intensity(const StepArgs& a, int mode, float* lam, float* p, cudaStream_t s) {
  const size_t total = static_cast<size_t>(a.h) * a.w * a.n_envs;
  const int blocks = static_cast<int>((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
  if (mode == kStaticTables) k_intensity<kStaticTables><<<blocks, 256, 0, s>>>(a, lam, p);
  else k_intensity<kStaticTerrain><<<blocks, 256, 0, s>>>(a, lam, p);
  return cudaGetLastError();
}

cudaError_t launch_counts(const uint8_t* st, int n_envs, int ncell, int32_t* counts, cudaStream_t s) {
  k_counts<<<n_envs, 256, 0, s>>>(st, ncell, counts);
  return cudaGetLastError();
}

cudaError_t launch_rl_ref_step(const RlArgs& g, int mode, cudaStream_t s) {
  const size_t sm = static_cast<size_t>(g.s.h) * g.s.w;
  if (mode == kStaticTables) k_rl_ref_step<kStaticTables><<<g.s.n_envs, kRlThreads, sm, s>>>(g);
  else k_rl_ref_step<kStaticTerrain><<<g.s.n_envs, kRlThreads, sm, s>>>(g);
  return cudaGetLastError();
}

cudaError_t launch_rl_observe(const uint8_t* state, const RlEnv* envs, int n_envs, int h, int w,
                              int radius, int capacity, double* obs, cudaStream_t s) {
  const int side = 2 * radius + 1;
  const size_t total = static_cast<size_t>(n_envs) * (3 * side * side + 3);
  const int blocks = static_cast<int>((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
  k_rl_observe<<<blocks, 256, 0, s>>>(state, envs, n_envs, h, w, radius, capacity, obs);
  return cudaGetLastError();
}

cudaError_t launch_rl_tanker(const RlArgs& g, int mode, cudaStream_t s) {
  const size_t sm = 3 * static_cast<size_t>(g.s.h) * g.s.w;
  if (mode == kStaticTables) k_rl_tanker<kStaticTables><<<g.s.n_envs, kRlThreads, sm, s>>>(g);
  else k_rl_tanker<kStaticTerrain><<<g.s.n_envs, kRlThreads, sm, s>>>(g);
  return cudaGetLastError();
}

cudaError_t launch_rl_tanker_reset(const RlArgs& g, int mode, const uint8_t* mask, cudaStream_t s) {
  const size_t sm = 2 * static_cast<size_t>(g.s.h) * g.s.w;
  if (mode == kStaticTables) k_rl_tanker_reset<kStaticTables><<<g.s.n_envs, kRlThreads, sm, s>>>(g, mask);
  else k_rl_tanker_reset<kStaticTerrain><<<g.s.n_envs, kRlThreads, sm, s>>>(g, mask);
  return cudaGetLastError();
}

}  // namespace ebl
