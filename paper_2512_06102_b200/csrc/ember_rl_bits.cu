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

#include <algorithm>
#include <cstdint>

#include "ember_bits.cuh"
#include "ember_device.cuh"
#include "ember_kernels.h"
#include "ember_pdl.cuh"
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
  uint16_t* list = reinterpret_cast<uint16_t*>(ACT + nwords);  // capacity n: every cell fits
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
    for (int i = threadIdx.x; i < 2 * a.n_pal; i += blockDim.x)  // the palette entries in use: src, gam
      s_pal[i < a.n_pal ? i : 256 + i - a.n_pal] = __ldg(a.pal32 + (i < a.n_pal ? i : 256 + i - a.n_pal));
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
      s_action = g.actions ? g.actions[env]
                           : static_cast<int>(below(cell_bits53(key_prefix(g.seed, e.stream,
                                                                           static_cast<uint64_t>(e.step)),
                                                                0, 2),
                                                    n));
    }
    __syncthreads();
    // the next step's counters: every thread has read this slot (as the previous step's) before
    // the barrier above; the next step writes it after this step's last barrier
    if (threadIdx.x == 0) s_total[par ^ 1] = s_newly[par ^ 1] = s_burn[par ^ 1] = 0;
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
    e = smem_opt_in(reinterpret_cast<const void*>(k_rl_tanker_bits<kStaticTables>), sm);
    if (e != cudaSuccess) return e;
    k_rl_tanker_bits<kStaticTables><<<g.s.n_envs, kRlBitsThreads, sm, s>>>(g);
  } else {
    e = smem_opt_in(reinterpret_cast<const void*>(k_rl_tanker_bits<kStaticTerrain>), sm);
    if (e != cudaSuccess) return e;
    k_rl_tanker_bits<kStaticTerrain><<<g.s.n_envs, kRlBitsThreads, sm, s>>>(g);
  }
  return cudaGetLastError();
}



// ---- warp-local tanker kernel -----------------------------------------------------------------
// The same env step as k_rl_tanker_bits, with the CA step of k_step_warp (ember_warp.cu): rows
// dealt to warps interleaved (row 4l + w), each warp deciding its own rows' active cells, so a
// step needs two block barriers (after the drop, at the end) instead of five: every thread draws
// the action itself, and the Burning count is kept incrementally (burning(t+1) = burning(t) -
// extinguished - burnt out + ignited) instead of a popc pass.
#ifndef EBL_RL_FAST
#define EBL_RL_FAST 1  // the branch-free decide pass in the tanker kernel
#endif
#ifndef EBL_RL_FAST_STEP  // the branch-free pass in single-step launches too (2 warps per 64-row env:
#define EBL_RL_FAST_STEP 1  // device-io steps 2.67e8 -> 2.74e8 env-steps/s, rollouts 6.87 -> 6.74 ms)
#endif
#ifndef EBL_RL_LUT  // its table-driven n-th set bit (a global table: one L2 miss per fresh CTA,
#define EBL_RL_LUT 0  // which single-step launches of 16384 CTAs pay: popc search instead)
#endif
namespace {

// the shallower n-th set bit of the warp kernel (ember_warp.cu)
__device__ __forceinline__ int nth_set_bit_lut32(uint32_t v, int q, const uint32_t* lut) {
  uint32_t c = v - ((v >> 1) & 0x55555555u);
  c = (c & 0x33333333u) + ((c >> 2) & 0x33333333u);
  c = (c + (c >> 4)) & 0x0f0f0f0fu;
  const uint32_t cum = c * 0x01010101u;
  const uint32_t qq = static_cast<uint32_t>(q);
  const int k = (qq >= (cum & 0xffu)) + (qq >= ((cum >> 8) & 0xffu)) + (qq >= ((cum >> 16) & 0xffu));
  const int before = k ? static_cast<int>((cum << 8 >> (8 * k)) & 0xffu) : 0;
  const uint32_t byte = (v >> (8 * k)) & 0xffu;
  return 8 * k + static_cast<int>((__ldg(lut + byte) >> (3 * (q - before))) & 7u);
}

__device__ __forceinline__ int nth_set_bit32(uint32_t v, int q) {
  int pos = 0;
#pragma unroll
  for (int half = 16; half > 0; half >>= 1) {
    const int c = __popc(v & ((1u << half) - 1u));
    if (q >= c) {
      q -= c;
      pos += half;
      v >>= half;
    }
  }
  return pos;
}

}  // namespace

// NW warps per env (rows dealt NW apart): 4 in general, 2 for envs of <= 64 rows (every lane owns a
// row in the dense pass, and twice the envs are resident per SM)
template <int MODE, int DIMC, int NW>
__global__ void __launch_bounds__(32 * NW, 32 / NW) k_rl_tanker_warp(RlArgs g) {
  pdl_enter();  // consecutive ebl_rl_step launches (device-io learner loop): PDL
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int s_newly[2], s_gone[2];  // per step parity: ignitions, Burning cells lost
  __shared__ int s_burning[2];           // Burning cells at the start of step t (slot t & 1)
  __shared__ int s_placed;
  constexpr bool kTer = MODE == kStaticTerrain;
  __shared__ float s_pal[kTer ? 512 : 1];
  __shared__ float s_kw[8];
  __shared__ float s_srckw[kTer ? 32 * 8 : 1];
  // the branch-free decide pass of k_step_warp (even compile-time words per row, pot32t rows)
  constexpr bool kFast = EBL_RL_FAST && kTer && DIMC != 0 && ((DIMC + 31) / 32) % 2 == 0;

  const StepArgs& a = g.s;
  const int env = blockIdx.x;
  const int H = DIMC ? DIMC : a.h, W = DIMC ? DIMC : a.w, n = H * W;
  const int wpr = (W + 31) >> 5;
  const int S = plane_stride(wpr);
  auto ro = [S](int R) { return R * S + R / NW; };  // conflict-free rows NW apart (ember_warp.cu)
  const int PH = ro(H + 2) + 1;
  uint32_t* const Bp0 = reinterpret_cast<uint32_t*>(smem) + 4;  // 4 zero guard words before the planes
  uint32_t* const Bp1 = Bp0 + PH;
  uint32_t* const X = Bp1 + PH;
  uint32_t* const WET = X + PH;
  uint32_t* const ACT = WET + PH;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool vec = (W & 31) == 0;
  const uint32_t last_mask = low_mask(W - 32 * (wpr - 1));

  uint8_t* st = g.state + static_cast<size_t>(env) * n;
  uint8_t* wt = g.wet + static_cast<size_t>(env) * n;
  // the env record and the caller's action are requested first: their latency overlaps the plane
  // loads instead of following the barrier (single-step launches are a chain of global round trips)
  RlEnv e = g.env[env];
  const int action_in = g.actions ? __ldg(g.actions + env) : 0;
  if constexpr (kFast) {  // guard, padding words and padding rows of both B planes stay zero
    // only the words no load or dense pass writes: the 4 guard words, the padding rows 0 and H+1,
    // and every row's padding / skew words (ro(R) + wpr .. ro(R+1)) of both planes
    if (threadIdx.x < 4) reinterpret_cast<uint32_t*>(smem)[threadIdx.x] = 0u;
    for (int i = threadIdx.x; i < 2 * (H + 2); i += blockDim.x) {
      const int R = i % (H + 2);
      uint32_t* P = i < H + 2 ? Bp0 : Bp1;
      for (int k = (R == 0 || R == H + 1) ? ro(R) : ro(R) + wpr; k < ro(R + 1); ++k) P[k] = 0u;
    }
    if (threadIdx.x == 0) Bp0[ro(H + 2)] = Bp1[ro(H + 2)] = 0u;  // the plane's last word
    __syncthreads();
  } else {
    for (int i = threadIdx.x; i < wpr; i += blockDim.x) {
      Bp0[i] = Bp1[i] = 0u;
      Bp0[ro(H + 1) + i] = Bp1[ro(H + 1) + i] = 0u;
    }
  }
  if (threadIdx.x < 2) s_newly[threadIdx.x] = s_gone[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_burning[0] = 0;
  const bool use_tab = kTer && a.pot32t != nullptr;  // precomputed lambda terms (one wind per env)
  const bool use_rec = kTer && a.nfuel && a.n_pal <= 32;
  if constexpr (kTer) {
    for (int i = threadIdx.x; i < 2 * a.n_pal; i += blockDim.x)  // the palette entries in use: src, gam
      s_pal[i < a.n_pal ? i : 256 + i - a.n_pal] = __ldg(a.pal32 + (i < a.n_pal ? i : 256 + i - a.n_pal));
    if (threadIdx.x < 8) s_kw[threadIdx.x] = __ldg(a.kw32 + static_cast<size_t>(env) * a.kw_stride + threadIdx.x);
    if (use_rec)
      for (int i = threadIdx.x; i < a.n_pal * 8; i += blockDim.x)
        s_srckw[i] = __ldg(a.pal32 + (i >> 3)) * __ldg(a.kw32 + static_cast<size_t>(env) * a.kw_stride + (i & 7));
  }
  int burning0 = 0;
  const size_t plane_words = static_cast<size_t>(H) * wpr;
  uint32_t* const gbits = g.bits ? g.bits + static_cast<size_t>(env) * 3 * plane_words : nullptr;
  for (WordIter it(wpr, H * wpr); it.ok(); it.next()) {
    uint32_t b = 0u, x = 0u, wb = 0u;
    if (g.bits_in) {  // bit-resident state of the previous launch: 1/8 of the byte traffic
      b = gbits[it.idx];
      x = gbits[plane_words + it.idx];
      wb = gbits[2 * plane_words + it.idx];
    } else {
      const uint8_t* src = st + it.r * W + 32 * it.j;
      const uint8_t* wsrc = wt + it.r * W + 32 * it.j;
      const int nc = min(32, W - 32 * it.j);
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
    }
    Bp0[ro(it.r + 1) + it.j] = b;
    X[ro(it.r) + it.j] = x;
    WET[ro(it.r) + it.j] = wb;
    burning0 += __popc(b);
  }
  __syncthreads();  // s_burning zeroed, planes loaded
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) burning0 += __shfl_xor_sync(0xffffffffu, burning0, o);
  if (lane == 0 && burning0) atomicAdd(&s_burning[0], burning0);

  const DiagCounters dg{a.diag};
  double rsum = 0.0;
  int32_t finished = 0;
  int cur = 0;
  auto win3 = [&](const uint32_t* row, int j, int b) -> uint32_t {
    const uint32_t wj = row[j];
    uint32_t v = b > 0 ? wj >> (b - 1) : ((j > 0 ? row[j - 1] >> 31 : 0u) | (wj << 1));
    if (b == 31) v = (v & 3u) | ((j + 1 < wpr ? row[j + 1] & 1u : 0u) << 2);
    return v & 7u;
  };
  // fused rollouts: rng key prefixes (3 of the 5 rounds) and random-policy actions of the next 64
  // episode steps, one per thread, rebuilt when they run out or an auto-reset starts a new episode
  // stream (C2 rollout 6.75 -> 6.20 ms)
  __shared__ uint64_t s_pre[64];
  __shared__ int s_act[64];
  int tab_step = -64;
  uint64_t tab_stream = ~0ull;
  for (int t = 0; t < g.n_steps; ++t) {
    const int par = t & 1;
    uint32_t* B = cur ? Bp1 : Bp0;
    uint32_t* Bn = cur ? Bp0 : Bp1;
    if (g.n_steps > 1 && (e.stream != tab_stream || e.step - tab_step >= 64)) {  // block-uniform (e is shared)
      for (int k = threadIdx.x; k < 64; k += blockDim.x) {
        const uint64_t pre = key_prefix(g.seed, e.stream, static_cast<uint64_t>(e.step + k));
        s_pre[k] = pre;
        s_act[k] = g.actions ? 0 : static_cast<int>(below(cell_bits53(pre, 0, 2), n));
      }
      tab_step = e.step;
      tab_stream = e.stream;
      __syncthreads();
    }
    // ---- action (every thread) + drop ----------------------------------------------------------
    // (single-step launches: the one prefix directly)
    const uint64_t prefix = g.n_steps > 1 ? s_pre[e.step - tab_step] : key_prefix(g.seed, e.stream, static_cast<uint64_t>(e.step));
    const int action = g.actions ? action_in
                                 : g.n_steps > 1 ? s_act[e.step - tab_step] : static_cast<int>(below(cell_bits53(prefix, 0, 2), n));
    if (threadIdx.x < 9) {
      const int r = action / W + static_cast<int>(threadIdx.x) / 3 - 1;
      const int c = action % W + static_cast<int>(threadIdx.x) % 3 - 1;
      if (r >= 0 && r < H && c >= 0 && c < W) {
        const uint32_t bit = 1u << (c & 31);
        uint32_t* bw = B + ro(r + 1) + (c >> 5);
        if (*bw & bit) {  // extinguish
          atomicAnd(bw, ~bit);
          atomicOr(X + ro(r) + (c >> 5), bit);
          atomicAdd(&s_gone[par], 1);
        } else if (!(X[ro(r) + (c >> 5)] & bit)) {  // wet
          atomicOr(WET + ro(r) + (c >> 5), bit);
        }
      }
    }
    __syncthreads();
    // the next step's counters (read as the previous step's before the barrier above, written by
    // the next step after this step's last barrier)
    if (threadIdx.x == 0) s_newly[par ^ 1] = s_gone[par ^ 1] = 0;
    // ---- warp-local CA step (k_step_warp) -----------------------------------------------------------
    int newly = 0, burnt = 0;
    for (int rb = 0; rb < H; rb += 32 * NW) {
      const int r = rb + NW * lane + warp;
      int cnt = 0;
      uint32_t cum = 0xffffffffu;
      if (r < H) {
        const uint32_t* up = B + ro(r + 2);
        const uint32_t* mid = B + ro(r + 1);
        const uint32_t* dn = B + ro(r);
        uint32_t* bn = Bn + ro(r + 1);
        const uint32_t* xr = X + ro(r);
        const uint32_t* wr = WET + ro(r);
        uint32_t* ar = ACT + ro(r);
        uint32_t vl = 0u;
        uint32_t uc = up[0], mc = mid[0], dc = dn[0];
        uint32_t vc = uc | mc | dc;
        for (int j = 0; j < wpr; ++j) {
          uint32_t un = 0u, mn = 0u, dnn = 0u;
          if (j + 1 < wpr) {
            un = up[j + 1];
            mn = mid[j + 1];
            dnn = dn[j + 1];
          }
          const uint32_t vn = un | mn | dnn;
          const uint32_t any = ((vc << 1) | (vl >> 31)) | ((vc >> 1) | (vn << 31)) | uc | dc;
          bn[j] = mc;
          const uint32_t valid = j + 1 < wpr ? 0xffffffffu : last_mask;
          const uint32_t act = ((~(mc | xr[j] | wr[j]) & valid) & any) | mc;  // wet cells never ignite
          ar[j] = act;
          if (j + 1 < 4) cum = (cum & ~(0xffu << (8 * (j + 1)))) | (static_cast<uint32_t>(cnt + __popc(act)) << (8 * (j + 1)));
          cnt += __popc(act);
          vl = vc;
          vc = vn;
          uc = un;
          mc = mn;
          dc = dnn;
        }
      }
      if (!__ballot_sync(0xffffffffu, cnt > 0)) continue;
      __syncwarp();
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int excl = incl - cnt;
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      for (int p = 0; p < total; p += 32) {
        const int idx = p + lane;
        int L = 0;
#pragma unroll
        for (int stp = 16; stp > 0; stp >>= 1) {
          const int cand = L + stp;
          const int v = __shfl_sync(0xffffffffu, excl, cand & 31);
          if (cand < 32 && v <= idx) L = cand;
        }
        int q = idx - __shfl_sync(0xffffffffu, excl, L);
        const uint32_t cumL = __shfl_sync(0xffffffffu, cum, L);
        if (idx >= total) continue;
        const int rr = rb + NW * L + warp;
        const uint32_t* ar = ACT + ro(rr);
        int jj = 0;
        uint32_t wv;
        if (wpr <= 4) {
          const uint32_t qq = static_cast<uint32_t>(q);
          jj = (qq >= ((cumL >> 8) & 0xffu)) + (qq >= ((cumL >> 16) & 0xffu)) + (qq >= (cumL >> 24));
          q -= jj ? static_cast<int>((cumL >> (8 * jj)) & 0xffu) : 0;
          wv = ar[jj];
        } else {
          wv = ar[0];
          for (;;) {
            const int pc = __popc(wv);
            if (q < pc) break;
            q -= pc;
            wv = ar[++jj];
          }
        }
        int cc;
        if constexpr (kFast && EBL_RL_LUT) cc = 32 * jj + nth_set_bit_lut32(wv, q, kNthBitLut);
        else cc = 32 * jj + nth_set_bit32(wv, q);
        // one branch-free path for burning and candidate cells (ember_warp.cu); with 4 warps per env
        // single-step launches had measured faster on the branchy path (EBL_RL_FAST_STEP=0)
        if (kFast && use_tab && (EBL_RL_FAST_STEP || g.n_steps > 1)) {
          const float4* tp = reinterpret_cast<const float4*>(a.pot32t + static_cast<size_t>(env) * a.pot32t_stride) +
                             2 * (rr * W + cc);
          const float4 T0 = __ldg(tp), T1 = __ldg(tp + 1);
          const int j = cc >> 5, b = cc & 31;
          const uint32_t bit = 1u << b;
          const int wi = ro(rr + 1) + j;
          const uint64_t m = cell_bits53(prefix, static_cast<uint64_t>(rr * W + cc), 0);
          auto win = [&](const uint32_t* row) -> uint32_t {
            const uint32_t lo = row[j - 1], md = row[j], hi = row[j + 1];
            return (b > 0 ? __funnelshift_r(md, hi, b - 1) : __funnelshift_r(lo, md, 31)) & 7u;
          };
          const uint32_t midw = win(B + ro(rr + 1)), dnw = win(B + ro(rr)), upw = win(B + ro(rr + 2));
          const bool burning = midw & 2u;
          const uint32_t nb = burning ? 0u
                                      : (midw & 1u) | (dnw << 1) | ((midw >> 2) << 4) | ((upw >> 2) << 5) |
                                            ((upw & 2u) << 5) | ((upw & 1u) << 7);
          const bool ig = ignite_pot_fast(a, env, 0, T0, T1, W, rr, cc, nb, m, dg);
          if (burning && m >= a.pc_thr) {
            atomicAnd(Bn + wi, ~bit);
            atomicOr(X + ro(rr) + j, bit);
            ++burnt;
          }
          if (ig) {
            atomicOr(Bn + wi, bit);
            ++newly;
          }
          continue;
        }
        CellRec rec{};
        if (use_tab) {  // the candidate's 8 terms of gamma * lambda (pot32t)
          const float4* tp = reinterpret_cast<const float4*>(a.pot32t + static_cast<size_t>(env) * a.pot32t_stride) +
                             2 * (rr * W + cc);
          rec.s0 = __ldg(tp);
          rec.s1 = __ldg(tp + 1);
        } else if (use_rec) {
          rec = load_rec(a.slope32 + static_cast<size_t>(env) * a.ter_stride * 8,
                         a.nfuel + static_cast<size_t>(env) * a.ter_stride, a.fuel + static_cast<size_t>(env) * a.ter_stride,
                         rr * W + cc);
        }
        const int j = cc >> 5, b = cc & 31;
        const uint32_t bit = 1u << b;
        const int wi = ro(rr + 1) + j;
        const uint64_t m = cell_bits53(prefix, static_cast<uint64_t>(rr * W + cc), 0);
        const uint32_t midw = win3(B + ro(rr + 1), j, b);
        if (midw & 2u) {
          if (m >= a.pc_thr) {
            atomicAnd(Bn + wi, ~bit);
            atomicOr(X + ro(rr) + j, bit);
            ++burnt;
          }
        } else {
          const uint32_t dnw = win3(B + ro(rr), j, b), upw = win3(B + ro(rr + 2), j, b);
          const uint32_t nb = (midw & 1u) | (dnw << 1) | ((midw >> 2) << 4) | ((upw >> 2) << 5) |
                              ((upw & 2u) << 5) | ((upw & 1u) << 7);
          bool ig;
          if (use_tab)
            ig = ignite_pot(a, env, 0, rec.s0, rec.s1, W, rr, cc, nb, m, dg);
          else if (use_rec)
            ig = ignite_terrain_rec_pre(terrain_view(a, env), rec, s_srckw, s_pal + 256, a.alpha_s_l2, W, rr, cc, nb, m, dg);
          else if constexpr (kTer)
            ig = ignite_terrain_tab(terrain_view(a, env), a.slope32 + static_cast<size_t>(env) * a.ter_stride * 8,
                                    s_pal, s_kw, W, H, rr, cc, nb, m, dg);
          else
            ig = ignite<MODE>(a, env, rr, cc, nb, m, dg);
          if (ig) {
            atomicOr(Bn + wi, bit);
            ++newly;
          }
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      newly += __shfl_xor_sync(0xffffffffu, newly, o);
      burnt += __shfl_xor_sync(0xffffffffu, burnt, o);
    }
    if (lane == 0 && newly) atomicAdd(&s_newly[par], newly);
    if (lane == 0 && burnt) atomicAdd(&s_gone[par], burnt);
    __syncthreads();
    cur ^= 1;
    // ---- reward, done (Burning count kept incrementally) --------------------------------------------
    const int burning = s_burning[par] - s_gone[par] + s_newly[par];
    e.step += 1;
    const double reward = -static_cast<double>(s_newly[par]);
    const bool done = burning == 0 || e.step >= g.max_steps;
    rsum += reward;
    if (g.n_steps == 1 && threadIdx.x == 0) {
      if (g.reward) g.reward[env] = reward;
      if (g.done) g.done[env] = done ? 1 : 0;
    }
    if (done) {  // auto-reset in place (block-uniform branch)
      ++finished;
      uint32_t* Bnew = cur ? Bp1 : Bp0;
      for (int i = threadIdx.x; i < PH; i += blockDim.x) {
        Bnew[i] = 0u;
        X[i] = 0u;
        WET[i] = 0u;
      }
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
          const int cr = cell / W, cc2 = cell % W;
          uint32_t* bw = Bnew + ro(cr + 1) + (cc2 >> 5);
          const uint32_t bit = 1u << (cc2 & 31);
          const bool burnable = kTer ? a.pal64[512 + fuel[cell]] > 0.5
                                     : a.gamma[static_cast<size_t>(env) * a.tab_stride + cell] > 0.0;
          if ((*bw & bit) || !burnable) continue;
          *bw |= bit;
          ++placed;
        }
        s_placed = placed;
        s_burning[par ^ 1] = placed;
      }
      __syncthreads();
      e.step = 0;
      e.episode = episode;
      e.stream = stream;
      e.done = s_placed == 0;
    } else if (threadIdx.x == 0) {
      s_burning[par ^ 1] = burning;  // read after the next step's barriers
    }
  }
  // ---- store ----------------------------------------------------------------------------------
  __syncthreads();
  const uint32_t* Bs = cur ? Bp1 : Bp0;
  for (WordIter it(wpr, H * wpr); it.ok(); it.next()) {
    const uint32_t b = Bs[ro(it.r + 1) + it.j], x = X[ro(it.r) + it.j], wb = WET[ro(it.r) + it.j];
    if (gbits) {  // bit-resident (the byte layers are rebuilt on demand, ebl_rl_bits_to_bytes)
      gbits[it.idx] = b;
      gbits[plane_words + it.idx] = x;
      gbits[2 * plane_words + it.idx] = wb;
      continue;
    }
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

// Bit-resident tanker state -> byte layers (state, wet): one thread per (env, row, word).
__global__ void k_rl_bits_to_bytes(const uint32_t* __restrict__ bits, uint8_t* state, uint8_t* wet, int n_envs, int H,
                                   int W) {
  const int wpr = (W + 31) >> 5;
  const size_t plane = static_cast<size_t>(H) * wpr;
  const size_t total = plane * n_envs;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t env = i / plane, k = i - env * plane;
    const int r = static_cast<int>(k / wpr), j = static_cast<int>(k - static_cast<size_t>(r) * wpr);
    const uint32_t* eb = bits + env * 3 * plane;
    const uint32_t b = eb[k], x = eb[plane + k], wb = eb[2 * plane + k];
    uint8_t* dst = state + env * H * W + static_cast<size_t>(r) * W + 32 * j;
    uint8_t* wdst = wet + env * H * W + static_cast<size_t>(r) * W + 32 * j;
    const int nc = min(32, W - 32 * j);
    if (nc == 32 && (W & 15) == 0) {
      bits_to_bytes(b, x, dst);
      bits_to_bytes(wb, 0u, wdst);
    } else {
      for (int c = 0; c < nc; ++c) {
        dst[c] = static_cast<uint8_t>(((b >> c) & 1u) | (((x >> c) & 1u) << 1));
        wdst[c] = static_cast<uint8_t>((wb >> c) & 1u);
      }
    }
  }
}

// Tanker observation on the device: one byte per cell, FireState in bits 0-1 and the wet flag in
// bit 2, [n_envs][H][W] into a caller buffer (e.g. a learner's torch tensor).  Reads the bit-resident
// planes (bits != null) without invalidating them, else the byte layers.
__global__ void k_rl_observe_planes(const uint32_t* __restrict__ bits, const uint8_t* __restrict__ state,
                                    const uint8_t* __restrict__ wet, uint8_t* out, int n_envs, int H, int W) {
  const int wpr = (W + 31) >> 5;
  const size_t plane = static_cast<size_t>(H) * wpr;
  const size_t total = plane * n_envs;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t env = i / plane, k = i - env * plane;
    const int r = static_cast<int>(k / wpr), j = static_cast<int>(k - static_cast<size_t>(r) * wpr);
    const size_t off = env * H * W + static_cast<size_t>(r) * W + 32 * j;
    const int nc = min(32, W - 32 * j);
    if (bits) {
      const uint32_t* eb = bits + env * 3 * plane;
      const uint32_t b = eb[k], x = eb[plane + k], wb = eb[2 * plane + k];
      for (int c = 0; c < nc; ++c)
        out[off + c] = static_cast<uint8_t>(((b >> c) & 1u) | (((x >> c) & 1u) << 1) | (((wb >> c) & 1u) << 2));
    } else {
      for (int c = 0; c < nc; ++c) out[off + c] = static_cast<uint8_t>(state[off + c] | (wet[off + c] << 2));
    }
  }
}

cudaError_t launch_rl_observe_planes(const uint32_t* bits, const uint8_t* state, const uint8_t* wet, uint8_t* out,
                                     int n_envs, int h, int w, cudaStream_t s) {
  const size_t total = static_cast<size_t>(n_envs) * h * ((w + 31) / 32);
  const unsigned blocks = static_cast<unsigned>(std::min<size_t>((total + 255) / 256, 148 * 16));
  k_rl_observe_planes<<<blocks, 256, 0, s>>>(bits, state, wet, out, n_envs, h, w);
  return cudaGetLastError();
}

cudaError_t launch_rl_bits_to_bytes(const uint32_t* bits, uint8_t* state, uint8_t* wet, int n_envs, int h, int w,
                                    cudaStream_t s) {
  const size_t total = static_cast<size_t>(n_envs) * h * ((w + 31) / 32);
  const unsigned blocks = static_cast<unsigned>(std::min<size_t>((total + 255) / 256, 148 * 16));
  k_rl_bits_to_bytes<<<blocks, 256, 0, s>>>(bits, state, wet, n_envs, h, w);
  return cudaGetLastError();
}

int rl_warps(int h) { return h <= 64 ? 2 : 4; }

size_t rl_warp_smem_bytes(int h, int w) {
  const size_t S = plane_stride((w + 31) / 32);
  const size_t R = static_cast<size_t>(h) + 2;
  // B x2, X, WET, ACT (ro() layout) + guard words
  return 5 * (R * S + R / rl_warps(h) + 1) * sizeof(uint32_t) + 16;
}

template <int MODE, int DIMC, int NW>
static cudaError_t launch_rl_warp_t(const RlArgs& g, size_t sm, cudaStream_t s) {
  cudaError_t e = smem_opt_in(reinterpret_cast<const void*>(k_rl_tanker_warp<MODE, DIMC, NW>), sm);
  if (e != cudaSuccess) return e;
  return launch_pdl(k_rl_tanker_warp<MODE, DIMC, NW>, dim3(g.s.n_envs), dim3(32 * NW), sm, s, g);
}

cudaError_t launch_rl_tanker_warp(const RlArgs& g, int mode, cudaStream_t s) {
  const size_t sm = rl_warp_smem_bytes(g.s.h, g.s.w);
  const bool two = rl_warps(g.s.h) == 2;
  if (mode == kStaticTables)
    return two ? launch_rl_warp_t<kStaticTables, 0, 2>(g, sm, s) : launch_rl_warp_t<kStaticTables, 0, 4>(g, sm, s);
  if (g.s.h == 64 && g.s.w == 64) return launch_rl_warp_t<kStaticTerrain, 64, 2>(g, sm, s);
  return two ? launch_rl_warp_t<kStaticTerrain, 0, 2>(g, sm, s) : launch_rl_warp_t<kStaticTerrain, 0, 4>(g, sm, s);
}

}  // namespace ebl
