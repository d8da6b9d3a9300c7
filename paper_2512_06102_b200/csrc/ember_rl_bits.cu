// Bit-plane air-tanker RL kernel (BASELINE C2): one CTA per env, the env's layer as bit-planes
// in shared memory for the whole launch (n_steps = 1 for the per-step API, or a fused rollout
// with the device random policy).  Per step:
//   drop   the action's 3x3 patch: Burning -> Burned, Unburned -> wet (never ignites again);
//   step   the blocked kernel's bit-sliced CA step (ember_blocked.cu) with candidates masked
//          by ~wet, RNG key {seed, episode step, stream}, every cell updated;
//   reward -(cells ignited this step); done = no cell burning or step == max_steps;
//   reset  on done, in place: episode+1, stream = episode << 32 | env id, ignitions drawn
//          with rng_below(key{seed,0,stream}, counter++, kDrawEnvSetup, H*W) at burnable cells.
// Identical semantics to the byte kernel k_rl_tanker.
#include <cuda_runtime.h>

#include <cstdint>

#include "ember_bits.cuh"
#include "ember_device.cuh"
#include "ember_kernels.h"
#include "ember_params.h"

namespace ebl {

template <int MODE>
__global__ void __launch_bounds__(kRlBitsThreads, 8) k_rl_tanker_bits(RlArgs g) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int s_total[2], s_newly[2], s_burn[2];
  __shared__ int s_action, s_placed;
  __shared__ float s_pal[MODE == kStaticTerrain ? 512 : 1];  // terrain palette: fp32 src, gam
  __shared__ float s_kw[8];                                   // kappa_wind of this env

  const StepArgs& a = g.s;
  const int env = blockIdx.x;
  const int H = a.h, W = a.w, n = H * W;
  const int wpr = (W + 31) >> 5;
  const int nwords = H * wpr;
  const int pw = (H + 2) * wpr;
  uint32_t* Bp[2];
  Bp[0] = reinterpret_cast<uint32_t*>(smem);
  Bp[1] = Bp[0] + pw;
  uint32_t* X = Bp[1] + pw;
  uint32_t* WET = X + nwords;
  uint32_t* ACT = WET + nwords;
  uint16_t* list = reinterpret_cast<uint16_t*>(ACT + nwords);
  const int cap = n;
  const int lane = threadIdx.x & 31;
  const bool vec = (W & 31) == 0;

  uint8_t* st = g.state + static_cast<size_t>(env) * n;
  uint8_t* wt = g.wet + static_cast<size_t>(env) * n;
  for (int i = threadIdx.x; i < wpr; i += blockDim.x) {
    Bp[0][i] = Bp[1][i] = 0u;
    Bp[0][(H + 1) * wpr + i] = Bp[1][(H + 1) * wpr + i] = 0u;
  }
  if (threadIdx.x < 2) s_total[threadIdx.x] = s_newly[threadIdx.x] = s_burn[threadIdx.x] = 0;
  if constexpr (MODE == kStaticTerrain) {
    for (int i = threadIdx.x; i < 512; i += blockDim.x) s_pal[i] = __ldg(a.pal32 + i);
    if (threadIdx.x < 8) s_kw[threadIdx.x] = __ldg(a.kw32 + static_cast<size_t>(env) * a.kw_stride + threadIdx.x);
  }
  for (WordIter it(wpr, nwords); it.ok(); it.next()) {
    const uint8_t* src = st + it.r * W + 32 * it.j;
    const uint8_t* wsrc = wt + it.r * W + 32 * it.j;
    const int nc = min(32, W - 32 * it.j);
    uint32_t b = 0u, x = 0u, wb = 0u;
    if (vec) {
      bytes_to_bits(src, b, x);
      uint32_t w1, w2;
      bytes_to_bits(wsrc, w1, w2);  // wet bytes are 0/1
      wb = w1;
    } else {
      for (int k = 0; k < nc; ++k) {
        b |= static_cast<uint32_t>(src[k] == 1) << k;
        x |= static_cast<uint32_t>(src[k] == 2) << k;
        wb |= static_cast<uint32_t>(wsrc[k] != 0) << k;
      }
    }
    Bp[0][(it.r + 1) * wpr + it.j] = b;
    X[it.idx] = x;
    WET[it.idx] = wb;
  }
  __syncthreads();

  RlEnv e = g.env[env];
  const DiagCounters dg{a.diag};
  double rsum = 0.0;
  int32_t finished = 0;
  int cur = 0;
  for (int t = 0; t < g.n_steps; ++t) {
    const int par = t & 1;
    uint32_t* B = Bp[cur];
    uint32_t* Bn = Bp[cur ^ 1];
    // ---- action + drop -------------------------------------------------------------------
    if (threadIdx.x == 0) {
      s_total[par ^ 1] = s_newly[par ^ 1] = s_burn[par ^ 1] = 0;
      s_action = g.actions ? g.actions[env]
                           : static_cast<int>(below(cell_bits53(key_prefix(g.seed, e.stream,
                                                                           static_cast<uint64_t>(e.step)),
                                                                0, 2),
                                                    n));
    }
    __syncthreads();
    if (threadIdx.x < 9) {
      const int r = s_action / W + static_cast<int>(threadIdx.x) / 3 - 1;
      const int c = s_action % W + static_cast<int>(threadIdx.x) % 3 - 1;
      if (r >= 0 && r < H && c >= 0 && c < W) {
        const int wi = r * wpr + (c >> 5);
        const uint32_t bit = 1u << (c & 31);
        if (B[wi + wpr] & bit) {  // extinguish
          atomicAnd(B + wi + wpr, ~bit);
          atomicOr(X + wi, bit);
        } else if (!(X[wi] & bit)) {  // wet
          atomicOr(WET + wi, bit);
        }
      }
    }
    __syncthreads();
    // ---- P1: dilation, copy, candidates (not wet) ------------------------------------------
    const uint64_t prefix = key_prefix(g.seed, e.stream, static_cast<uint64_t>(e.step));
    int cnt = 0;
    for (WordIter it(wpr, nwords); it.ok(); it.next()) {
      const int j = it.j;
      const uint32_t* up = B + (it.r + 2) * wpr;
      const uint32_t* mid = B + (it.r + 1) * wpr;
      const uint32_t* dn = B + it.r * wpr;
      const uint32_t any = up[j] | west_of(up, j) | east_of(up, j, wpr) | dn[j] | west_of(dn, j) |
                           east_of(dn, j, wpr) | west_of(mid, j) | east_of(mid, j, wpr);
      const uint32_t b = mid[j];
      Bn[(it.r + 1) * wpr + j] = b;
      const uint32_t act = ((~(b | X[it.idx] | WET[it.idx]) & low_mask(W - 32 * j)) & any) | b;
      ACT[it.idx] = act;
      cnt += __popc(act);
    }
    if (__ballot_sync(0xffffffffu, cnt > 0)) {
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int base = 0;
      if (lane == 31) base = atomicAdd(&s_total[par], incl);
      base = __shfl_sync(0xffffffffu, base, 31) + incl - cnt;
      if (cnt > 0)
        for (WordIter it(wpr, nwords); it.ok(); it.next()) {
          uint32_t act = ACT[it.idx];
          const int cell0 = it.r * W + 32 * it.j;
          while (act) {
            const int bit = __ffs(act) - 1;
            act &= act - 1;
            list[base++] = static_cast<uint16_t>(cell0 + bit);
          }
        }
    }
    __syncthreads();
    // ---- P2: decisions ------------------------------------------------------------------------
    int newly = 0;
    for (int i = threadIdx.x; i < s_total[par]; i += blockDim.x) {
      const int cell = list[i];
      const int r = cell / W, c = cell - r * W;
      const int wi = (r + 1) * wpr + (c >> 5);
      const uint32_t bit = 1u << (c & 31);
      const uint64_t m = cell_bits53(prefix, static_cast<uint64_t>(cell), 0);
      if (B[wi] & bit) {
        if (m >= a.pc_thr) {
          atomicAnd(Bn + wi, ~bit);
          atomicOr(X + r * wpr + (c >> 5), bit);
        }
      } else {
        // burning-source mask from 3-cell windows of the rows below / at / above (ember_blocked.cu)
        const int j = c >> 5, b = c & 31;
        auto win3 = [&](const uint32_t* row) -> uint32_t {
          const uint32_t wj = row[j];
          uint32_t v = b > 0 ? wj >> (b - 1) : ((j > 0 ? row[j - 1] >> 31 : 0u) | (wj << 1));
          if (b == 31) v = (v & 3u) | ((j + 1 < wpr ? row[j + 1] & 1u : 0u) << 2);
          return v & 7u;
        };
        const uint32_t mid = win3(B + (r + 1) * wpr), dnw = win3(B + r * wpr), upw = win3(B + (r + 2) * wpr);
        const uint32_t nb = (mid & 1u) | (dnw << 1) | ((mid >> 2) << 4) | ((upw >> 2) << 5) |
                            ((upw & 2u) << 5) | ((upw & 1u) << 7);
        bool ig;
        if constexpr (MODE == kStaticTerrain)
          ig = ignite_terrain_tab(terrain_view(a, env), a.slope32 + static_cast<size_t>(env) * a.ter_stride * 8,
                                  s_pal, s_kw, W, H, r, c, nb, m, dg);
        else
          ig = ignite<MODE>(a, env, r, c, nb, m, dg);
        if (ig) {
          atomicOr(Bn + wi, bit);
          ++newly;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) newly += __shfl_xor_sync(0xffffffffu, newly, o);
    if (lane == 0 && newly) atomicAdd(&s_newly[par], newly);
    __syncthreads();
    cur ^= 1;
    // ---- burning count, reward, done -----------------------------------------------------------
    int burning = 0;
    for (WordIter it(wpr, nwords); it.ok(); it.next()) burning += __popc(Bn[(it.r + 1) * wpr + it.j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) burning += __shfl_xor_sync(0xffffffffu, burning, o);
    if (lane == 0 && burning) atomicAdd(&s_burn[par], burning);
    __syncthreads();
    e.step += 1;
    const double reward = -static_cast<double>(s_newly[par]);
    const bool done = s_burn[par] == 0 || e.step >= g.max_steps;
    rsum += reward;
    if (g.n_steps == 1 && threadIdx.x == 0) {
      if (g.reward) g.reward[env] = reward;
      if (g.done) g.done[env] = done ? 1 : 0;
    }
    if (done) {  // auto-reset in place (block-uniform branch)
      ++finished;
      for (int i = threadIdx.x; i < pw; i += blockDim.x) Bn[i] = 0u;
      for (int i = threadIdx.x; i < nwords; i += blockDim.x) X[i] = WET[i] = 0u;
      const uint32_t episode = e.episode + 1;
      const uint64_t stream = (static_cast<uint64_t>(episode) << 32) | (g.env_id0 + env);
      __syncthreads();
      if (threadIdx.x == 0) {
        const uint64_t pre = key_prefix(g.seed, stream, 0);
        const uint8_t* fuel = a.fuel + static_cast<size_t>(env) * a.ter_stride;
        uint64_t counter = 0;
        int placed = 0;
        while (placed < g.ignitions && counter < 64ull * n) {
          const int cell = static_cast<int>(below(cell_bits53(pre, counter++, 1), n));
          const int wi = (cell / W + 1) * wpr + ((cell % W) >> 5);
          const uint32_t bit = 1u << ((cell % W) & 31);
          const bool burnable = MODE == kStaticTerrain ? a.pal64[512 + fuel[cell]] > 0.5
                                                       : a.gamma[static_cast<size_t>(env) * a.tab_stride + cell] > 0.0;
          if ((Bn[wi] & bit) || !burnable) continue;
          Bn[wi] |= bit;
          ++placed;
        }
        s_placed = placed;
      }
      __syncthreads();
      e.step = 0;
      e.episode = episode;
      e.stream = stream;
      e.done = s_placed == 0;
    }
  }
  // ---- store ----------------------------------------------------------------------------------
  const uint32_t* B = Bp[cur];
  for (WordIter it(wpr, nwords); it.ok(); it.next()) {
    const uint32_t b = B[(it.r + 1) * wpr + it.j], x = X[it.idx], wb = WET[it.idx];
    uint8_t* dst = st + it.r * W + 32 * it.j;
    uint8_t* wdst = wt + it.r * W + 32 * it.j;
    if (vec) {
      bits_to_bytes(b, x, dst);
      bits_to_bytes(wb, 0u, wdst);
    } else {
      const int nc = min(32, W - 32 * it.j);
      for (int k = 0; k < nc; ++k) {
        dst[k] = static_cast<uint8_t>(((b >> k) & 1u) | (((x >> k) & 1u) << 1));
        wdst[k] = static_cast<uint8_t>((wb >> k) & 1u);
      }
    }
  }
  if (threadIdx.x == 0) {
    g.env[env] = e;
    if (g.reward_sum) g.reward_sum[env] += rsum;
    if (g.episodes) g.episodes[env] += finished;
  }
}

size_t rl_bits_smem_bytes(int h, int w) {
  const size_t wpr = (w + 31) / 32;
  return (2 * (static_cast<size_t>(h) + 2) + 3 * static_cast<size_t>(h)) * wpr * 4 +
         ((static_cast<size_t>(h) * w * 2 + 15) & ~size_t(15));
}

bool rl_bits_fits(int h, int w) {
  return static_cast<size_t>(h) * w <= 65536 && rl_bits_smem_bytes(h, w) <= kResMaxSmem;
}

cudaError_t launch_rl_tanker_bits(const RlArgs& g, int mode, cudaStream_t s) {
  const size_t sm = rl_bits_smem_bytes(g.s.h, g.s.w);
  cudaError_t e;
  if (mode == kStaticTables) {
    e = cudaFuncSetAttribute(k_rl_tanker_bits<kStaticTables>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sm));
    if (e != cudaSuccess) return e;
    k_rl_tanker_bits<kStaticTables><<<g.s.n_envs, kRlBitsThreads, sm, s>>>(g);
  } else {
    e = cudaFuncSetAttribute(k_rl_tanker_bits<kStaticTerrain>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sm));
    if (e != cudaSuccess) return e;
    k_rl_tanker_bits<kStaticTerrain><<<g.s.n_envs, kRlBitsThreads, sm, s>>>(g);
  }
  return cudaGetLastError();
}

}  // namespace ebl
