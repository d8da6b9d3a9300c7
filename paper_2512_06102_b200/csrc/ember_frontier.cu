// Frontier kernel — the resident-env throughput path (whole env per CTA, all steps fused).
//
// Same transition as k_step_blocked (engine.cpp:12-38, next_fire_cell), organised around the
// *active list* instead of a dense pass: only Burning cells and Unburned cells with a burning
// neighbour can change (an Unburned cell without one has p = 0, a Burned cell is absorbing,
// engine.cpp:16-25), and the list of step t+1 follows from the decisions of step t, so a step
// touches only its list:
//   decide  one thread per list entry, reading the state of step t: Burning -> survive test
//           (integer form of u < p_continue), candidate -> burning-source mask from three 3-cell
//           windows of B, slope-table fp32 lambda with the fp64 guard (ember_device.cuh);
//           the outcome (ignite / burn out / keep burning / none) is written into the entry;
//   --- barrier ---
//   apply   the outcomes are applied in place to the single B / X planes, and every cell burning
//           at t+1 (survivor or ignition) claims itself and its unburned neighbours in the listed
//           bitmap L[t+1] (one atomicOr per row of its 3x3 window); the newly claimed cells are
//           appended to the list of t+1 (one warp-aggregated reservation per warp);
//   --- barrier ---
// Races in apply are benign: a neighbour read as Unburned that is igniting or burning out in the
// same phase is listed anyway (burning cells list themselves) or decides "no change" at t+1
// (Burned cells are absorbing; a candidate without a burning source has lambda = 0).
// The list of step 0 is built densely at launch.  When the list of a step would exceed its
// capacity the CTA stores the state of that step and records it in a.resume[env]; the blocked
// kernel launched after this one continues those envs from there (launch_step_frontier), so the
// result never depends on the capacity.  Results are bit-identical to k_step_blocked.
#include <cuda_runtime.h>

#include <cstdint>

#include "ember_bits.cuh"
#include "ember_device.cuh"
#include "ember_kernels.h"
#include "ember_params.h"

#ifndef EBL_PHASE_PROF
#define EBL_PHASE_PROF 0
#endif

namespace ebl {

namespace {

constexpr int kFrThreads = 128;
constexpr uint16_t kOutNone = 0, kOutIgnite = 1, kOutBurnout = 2, kOutKeep = 3;

template <int MODE, int WPRC>
__global__ void __launch_bounds__(kFrThreads, 8) k_step_frontier(StepArgs a, int n_steps, int cap) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int s_n[2];       // list sizes (step parity)
  __shared__ int s_ovf;        // list of the next step overflowed
  __shared__ int s_newly;
  __shared__ int s_cnt[3];
  __shared__ uint64_t s_prefix[128];  // rng key prefixes, slot t & 127, refilled 64 steps at a time
  __shared__ float s_pal[MODE == kStaticTerrain ? 512 : 1];
  __shared__ float s_kw[8];

  const int env = blockIdx.x;
  const int H = a.h, W = a.w;
  const int wpr = WPRC ? WPRC : (W + 31) >> 5;
  const int S = plane_stride(wpr);
  uint32_t* const B = reinterpret_cast<uint32_t*>(smem);  // (H + 2) rows, zero padding rows 0, H+1
  uint32_t* const X = B + (H + 2) * S;                    // H rows
  uint32_t* const L0 = X + H * S;                          // listed bitmaps of the two step parities
  uint16_t* const list0 = reinterpret_cast<uint16_t*>(L0 + 2 * H * S);  // 2 x cap entries
  const size_t ncell = static_cast<size_t>(H) * W;
  const bool vec = (W & 15) == 0;
  const int lane = threadIdx.x & 31;
  const uint32_t last_mask = low_mask(W - 32 * (wpr - 1));
  // cell -> row: exact reciprocal division (cell * W < 2^32 here); W == 1 needs none
  const uint32_t magic = W > 1 ? static_cast<uint32_t>((0x100000000ull + W - 1) / W) : 0u;
  auto row_of = [&](uint32_t cell) -> int { return W > 1 ? static_cast<int>(__umulhi(cell, magic)) : static_cast<int>(cell); };

  // ---- load ----------------------------------------------------------------------------------
  for (int i = threadIdx.x; i < wpr; i += blockDim.x) {
    B[i] = 0u;
    B[(H + 1) * S + i] = 0u;
  }
  const uint8_t* __restrict__ in = a.in + env * ncell;
  for (WordIter it(wpr, H * wpr); it.ok(); it.next()) {
    const int nc = min(32, W - 32 * it.j);
    uint32_t b = 0u, x = 0u;
    const uint8_t* src = in + static_cast<size_t>(it.r) * W + 32 * it.j;
    if (nc == 32 && vec) {
      bytes_to_bits(src, b, x);
    } else {
      for (int k = 0; k < nc; ++k) {
        const uint8_t v = src[k];
        b |= static_cast<uint32_t>(v == 1) << k;
        x |= static_cast<uint32_t>(v == 2) << k;
      }
    }
    B[(it.r + 1) * S + it.j] = b;
    X[it.r * S + it.j] = x;
  }
  if constexpr (MODE == kStaticTerrain) {
    for (int i = threadIdx.x; i < 2 * a.n_pal; i += blockDim.x)  // the palette entries in use: src, gam
      s_pal[i < a.n_pal ? i : 256 + i - a.n_pal] = __ldg(a.pal32 + (i < a.n_pal ? i : 256 + i - a.n_pal));
    if (threadIdx.x < 8)  // the wind of step 0; a wind schedule reloads it per step
      s_kw[threadIdx.x] = __ldg(a.kw32 + static_cast<size_t>(sched_row(a, a.step)) * a.kw_sched_stride +
                                static_cast<size_t>(env) * a.kw_stride + threadIdx.x);
  }
  if (threadIdx.x < 2) s_n[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    s_ovf = 0;
    s_newly = 0;
  }
  if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0;
  const uint64_t stream = a.streams[env];
  for (int k = threadIdx.x; k < 64; k += blockDim.x) s_prefix[k] = key_prefix(a.seed, stream, a.step + k);
  __syncthreads();

  // ---- list of step 0 (dense, once): Burning cells and Unburned cells next to one ----------------
  {
    uint32_t* L = L0;
    int cnt = 0;
    for (int r = threadIdx.x; r < H; r += blockDim.x) {
      const uint32_t* up = B + (r + 2) * S;
      const uint32_t* mid = B + (r + 1) * S;
      const uint32_t* dn = B + r * S;
      for (int j = 0; j < wpr; ++j) {
        const uint32_t any = up[j] | west_of(up, j) | east_of(up, j, wpr) | dn[j] | west_of(dn, j) |
                             east_of(dn, j, wpr) | west_of(mid, j) | east_of(mid, j, wpr);
        const uint32_t valid = j + 1 < wpr ? 0xffffffffu : last_mask;
        const uint32_t act = ((~(mid[j] | X[r * S + j]) & valid) & any) | mid[j];
        L[r * S + j] = act;
        L[H * S + r * S + j] = 0u;  // the other parity starts empty
        cnt += __popc(act);
      }
    }
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int base = 0;
    if (lane == 31) base = atomicAdd(&s_n[0], incl);
    base = __shfl_sync(0xffffffffu, base, 31) + incl - cnt;
    for (int r = threadIdx.x; r < H; r += blockDim.x)
      for (int j = 0; j < wpr; ++j) {
        uint32_t rest = L[r * S + j];
        while (rest) {
          const int bit = __ffs(rest) - 1;
          rest &= rest - 1;
          if (base < cap) list0[base] = static_cast<uint16_t>(r * W + 32 * j + bit);
          ++base;
        }
      }
  }
  __syncthreads();
  int t = 0;
  if (s_n[0] > cap) s_ovf = 1;  // (read by all; thread-uniform) the dense list did not fit
  __syncthreads();

  const DiagCounters dg{a.diag};
  const uint64_t gbase = static_cast<uint64_t>(a.row_off) * W;
  auto win3 = [&](const uint32_t* row, int j, int b) -> uint32_t {  // columns c-1, c, c+1 -> bits 0..2
    const uint32_t wj = row[j];
    uint32_t v = b > 0 ? wj >> (b - 1) : ((j > 0 ? row[j - 1] >> 31 : 0u) | (wj << 1));
    if (b == 31) v = (v & 3u) | ((j + 1 < wpr ? row[j + 1] & 1u : 0u) << 2);
    return v & 7u;
  };

#if EBL_PHASE_PROF
  long long pr_t0 = 0, pr[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  __shared__ long long s_pa[3][kFrThreads / 32];
#endif
  for (; t < n_steps && !s_ovf; ++t) {
    const int par = t & 1;
#if EBL_PHASE_PROF
    if (a.prof && threadIdx.x == 0) {
      pr_t0 = clock64();
      pr[2] += s_n[par];
    }
#endif
    uint16_t* const list = list0 + par * cap;
    uint16_t* const nlist = list0 + (par ^ 1) * cap;
    uint32_t* const L = L0 + par * H * S;
    uint32_t* const Ln = L0 + (par ^ 1) * H * S;
    const int n = s_n[par];
    const int srow = sched_row(a, a.step + static_cast<uint64_t>(t));
    if constexpr (MODE == kStaticTerrain) {
      if (a.sched_len > 1) {  // CTA-uniform: time-varying wind
        if (threadIdx.x < 8)
          s_kw[threadIdx.x] = __ldg(a.kw32 + static_cast<size_t>(srow) * a.kw_sched_stride +
                                    static_cast<size_t>(env) * a.kw_stride + threadIdx.x);
        __syncthreads();
      }
    }
    // ---- decide ------------------------------------------------------------------------------
    const uint64_t prefix = s_prefix[t & 127];
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int cell = list[i];
      const int r = row_of(static_cast<uint32_t>(cell)), c = cell - r * W;
      const int j = c >> 5, b = c & 31;
      const uint32_t bit = 1u << b;
      uint16_t out = kOutNone;
      const uint32_t mid = win3(B + (r + 1) * S, j, b);
      if (!(X[r * S + j] & bit)) {
        const uint64_t m = cell_bits53(prefix, gbase + static_cast<uint64_t>(cell), 0);
        if (mid & 2u) {
          out = m >= a.pc_thr ? kOutBurnout : kOutKeep;
        } else {
          const uint32_t dnw = win3(B + r * S, j, b), upw = win3(B + (r + 2) * S, j, b);
          const uint32_t nb = (mid & 1u) | (dnw << 1) | ((mid >> 2) << 4) | ((upw >> 2) << 5) |
                              ((upw & 2u) << 5) | ((upw & 1u) << 7);
          if (nb) {
            bool ig;
            if constexpr (MODE == kStaticTerrain)
              ig = ignite_terrain_tab(terrain_view(a, env, srow), a.slope32 + static_cast<size_t>(env) * a.ter_stride * 8,
                                      s_pal, s_kw, W, H, r, c, nb, m, dg);
            else
              ig = ignite<MODE>(a, env, r, c, nb, m, dg, srow);
            if (ig) out = kOutIgnite;
          }
        }
      }
      list[i] = static_cast<uint16_t>(cell | (out << 14));
    }
    if (((t & 63) == 63) && t + 1 < n_steps) {  // refill the prefix ring with steps t+1 .. t+64
      for (int k = threadIdx.x; k < 64; k += blockDim.x)
        s_prefix[(t + 1 + k) & 127] = key_prefix(a.seed, stream, a.step + static_cast<uint64_t>(t + 1 + k));
    }
    if (threadIdx.x == 0) s_n[par ^ 1] = 0;
    __syncthreads();
#if EBL_PHASE_PROF
    if (a.prof && threadIdx.x == 0) {
      const long long t1 = clock64();
      pr[1] += t1 - pr_t0;  // decide (reported as P2)
      pr_t0 = t1;
    }
#endif
    // ---- apply + next list ---------------------------------------------------------------------
#if EBL_PHASE_PROF
    long long pa0 = 0, pa1 = 0, pa2 = 0;
    if (a.prof && lane == 0) pa0 = clock64();
#endif
    int newly = 0;
    for (int base0 = 0; base0 < n; base0 += blockDim.x) {  // CTA-uniform trip count (warp scans)
      const int i = base0 + threadIdx.x;
      uint32_t claim[3] = {0u, 0u, 0u};  // newly listed cells per row r-1, r, r+1 (bits: c-1, c, c+1)
      int r = 0, c = 0;
      if (i < n) {
        const uint16_t e = list[i];
        const int cell = e & 0x3fff, out = e >> 14;
        r = row_of(static_cast<uint32_t>(cell));
        c = cell - r * W;
        const int j = c >> 5, b = c & 31;
        const uint32_t bit = 1u << b;
        L[r * S + j] = 0u;  // L[t] is all-zero again after this phase (its bits are list t's entries)
        if (out == kOutIgnite) {
          atomicOr(B + (r + 1) * S + j, bit);
          ++newly;
        } else if (out == kOutBurnout) {
          atomicAnd(B + (r + 1) * S + j, ~bit);
          atomicOr(X + r * S + j, bit);
        }
        if (out == kOutIgnite || out == kOutKeep) {
          // claim the cell and its unburned neighbours for the list of t+1
#pragma unroll
          for (int d = -1; d <= 1; ++d) {
            const int rr = r + d;
            if (rr < 0 || rr >= H) continue;
            const uint32_t unb = ~(win3(B + (rr + 1) * S, j, b) | win3(X + rr * S, j, b)) & 7u;
            uint32_t want = d == 0 ? (unb | 2u) : unb;
            if (c == 0) want &= 6u;
            if (c == W - 1) want &= 3u;
            if (!want) continue;
            // bits c-1..c+1 of row rr in words j-1 / j / j+1
            uint32_t got = 0u;
            uint32_t* Lr = Ln + rr * S;
            if (b > 0 && b < 31) {
              const uint32_t msk = want << (b - 1);
              got = (msk & ~atomicOr(Lr + j, msk)) >> (b - 1);
            } else if (b == 0) {
              const uint32_t mw = (want >> 1) & 3u;  // c, c+1 in word j
              uint32_t g = mw ? (mw & ~atomicOr(Lr + j, mw)) << 1 : 0u;
              if (want & 1u) g |= (atomicOr(Lr + j - 1, 0x80000000u) & 0x80000000u) ? 0u : 1u;
              got = g;
            } else {  // b == 31
              const uint32_t mw = want & 3u;  // c-1, c in word j (bits 30, 31)
              uint32_t g = mw ? (((mw << 30) & ~atomicOr(Lr + j, mw << 30)) >> 30) : 0u;
              if (want & 4u) g |= (atomicOr(Lr + j + 1, 1u) & 1u) ? 0u : 4u;
              got = g;
            }
            claim[d + 1] = got;
          }
        }
      }
#if EBL_PHASE_PROF
      __syncwarp();
      if (a.prof && lane == 0) pa1 += clock64() - pa0;
#endif
      const int mine = __popc(claim[0]) + __popc(claim[1]) + __popc(claim[2]);
      int incl = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int pos = 0;
      if (lane == 31 && incl) pos = atomicAdd(&s_n[par ^ 1], incl);
      pos = __shfl_sync(0xffffffffu, pos, 31) + incl - mine;
#if EBL_PHASE_PROF
      if (a.prof && lane == 0) pa2 += clock64() - pa0;
#endif
      if (mine) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          uint32_t g = claim[d];
          while (g) {
            const int k = __ffs(g) - 1;
            g &= g - 1;
            if (pos < cap) nlist[pos] = static_cast<uint16_t>((r + d - 1) * W + c + k - 1);
            ++pos;
          }
        }
      }
    }
    if (t == n_steps - 1) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) newly += __shfl_xor_sync(0xffffffffu, newly, o);
      if (lane == 0 && newly) atomicAdd(&s_newly, newly);
    }
#if EBL_PHASE_PROF
    __syncwarp();
    if (a.prof && lane == 0) {
      s_pa[0][threadIdx.x >> 5] = pa1;
      s_pa[1][threadIdx.x >> 5] = pa2;
      s_pa[2][threadIdx.x >> 5] = clock64() - pa0;
    }
#endif
    __syncthreads();
#if EBL_PHASE_PROF
    if (a.prof && threadIdx.x == 0) {
      pr[0] += clock64() - pr_t0;  // apply + list (reported as P1)
      long long m0 = 0, m1 = 0, m2 = 0;
      for (int q = 0; q < kFrThreads / 32; ++q) {
        m0 = max(m0, s_pa[0][q]);
        m1 = max(m1, s_pa[1][q]);
        m2 = max(m2, s_pa[2][q]);
      }
      pr[4] += m0;  // reported as "dense": entries applied + claims
      pr[5] += m2;  // reported as "build": whole apply phase of the slowest warp
      pr[8] += m0;
      pr[9] += m1;  // reserve done
    }
#endif
    if (threadIdx.x == 0 && s_n[par ^ 1] > cap) s_ovf = 1;
    if (a.traj) {  // record (run_stochastic(record=true), engine.cpp:116): the layer after this step
      uint8_t* dst = a.traj + ((a.traj_t0 + t) * a.n_envs + env) * ncell;
      for (WordIter it(wpr, H * wpr); it.ok(); it.next()) {
        const uint32_t bb = B[(it.r + 1) * S + it.j], xx = X[it.r * S + it.j];
        uint8_t* o = dst + static_cast<size_t>(it.r) * W + 32 * it.j;
        const int nc = min(32, W - 32 * it.j);
        if (nc == 32 && vec) bits_to_bytes(bb, xx, o);
        else
          for (int k = 0; k < nc; ++k) o[k] = static_cast<uint8_t>(((bb >> k) & 1u) | (((xx >> k) & 1u) << 1));
      }
    }
    __syncthreads();  // s_ovf
  }

#if EBL_PHASE_PROF
  if (a.prof && threadIdx.x == 0) {
    pr[3] = t;
    for (int q = 0; q < 10; ++q) a.prof[env * 10 + q] = pr[q];
  }
#endif
  // ---- store: the state after step t (t == n_steps, or the hand-over step) -----------------------
  uint8_t* __restrict__ outp = a.out + env * ncell;
  int cu = 0, cb = 0, cx = 0;
  for (WordIter it(wpr, H * wpr); it.ok(); it.next()) {
    const uint32_t bb = B[(it.r + 1) * S + it.j], xx = X[it.r * S + it.j];
    const int nc = min(32, W - 32 * it.j);
    cu += nc - __popc(bb) - __popc(xx);
    cb += __popc(bb);
    cx += __popc(xx);
    uint8_t* o = outp + static_cast<size_t>(it.r) * W + 32 * it.j;
    if (nc == 32 && vec) bits_to_bytes(bb, xx, o);
    else
      for (int k = 0; k < nc; ++k) o[k] = static_cast<uint8_t>(((bb >> k) & 1u) | (((xx >> k) & 1u) << 1));
  }
  if (threadIdx.x == 0) a.resume[env] = t;  // t < n_steps: the blocked kernel continues this env
  if (t < n_steps || !a.counts) return;   // counts come from the continuation
  atomicAdd(&s_cnt[0], cu);
  atomicAdd(&s_cnt[1], cb);
  atomicAdd(&s_cnt[2], cx);
  __syncthreads();
  if (threadIdx.x < 3) atomicAdd(a.counts + env * 4 + threadIdx.x, s_cnt[threadIdx.x]);
  if (threadIdx.x == 3) atomicAdd(a.counts + env * 4 + 3, s_newly);
}

template <int MODE, int WPRC>
cudaError_t launch_fr(const StepArgs& a, int n_steps, int cap, size_t sm, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(k_step_frontier<MODE, WPRC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(sm));
  if (e != cudaSuccess) return e;
  k_step_frontier<MODE, WPRC><<<a.n_envs, kFrThreads, sm, s>>>(a, n_steps, cap);
  return cudaGetLastError();
}

}  // namespace

int frontier_cap(int h, int w) {
  const int cells = h * w;
  return cells <= 4096 ? cells : (cells / 8 > 2048 ? cells / 8 : 2048);
}

size_t frontier_smem_bytes(int h, int w) {
  const size_t S = plane_stride((w + 31) / 32);
  return ((static_cast<size_t>(h) + 2) + 3 * static_cast<size_t>(h)) * S * sizeof(uint32_t) +
         2 * static_cast<size_t>(frontier_cap(h, w)) * sizeof(uint16_t);
}

bool frontier_fits(int h, int w) {
  return static_cast<size_t>(h) * w <= 16384 && frontier_smem_bytes(h, w) <= kResMaxSmem;
}

// Frontier launch, then the blocked kernel for the envs that handed over (a.resume[env] < n).
// a.in / a.out as for the blocked kernel; a.resume must point to n_envs ints of device memory.
cudaError_t launch_step_frontier(const StepArgs& a0, int mode, int n_steps, cudaStream_t s) {
  StepArgs a = a0;
  const int cap = frontier_cap(a.h, a.w);
  const size_t sm = frontier_smem_bytes(a.h, a.w);
  const int wpr = (a.w + 31) / 32;
  cudaError_t e;
  if (mode == kStaticTables)
    e = wpr == 4 ? launch_fr<kStaticTables, 4>(a, n_steps, cap, sm, s)
                 : (wpr == 2 ? launch_fr<kStaticTables, 2>(a, n_steps, cap, sm, s)
                             : launch_fr<kStaticTables, 0>(a, n_steps, cap, sm, s));
  else
    e = wpr == 4 ? launch_fr<kStaticTerrain, 4>(a, n_steps, cap, sm, s)
                 : (wpr == 2 ? launch_fr<kStaticTerrain, 2>(a, n_steps, cap, sm, s)
                             : launch_fr<kStaticTerrain, 0>(a, n_steps, cap, sm, s));
  if (e != cudaSuccess) return e;
  // continuation: the blocked kernel in place on the handed-over envs (others exit at once)
  StepArgs b = a;
  b.in = a.out;
  BlockGeom g = plan_blocks(a.h, a.w, n_steps, false, 0, a.n_envs, 1);
  if (g.tile_h != a.h || g.halo_rows != 0) return cudaErrorInvalidValue;  // resident envs only
  return launch_step_blocked(b, mode, g, s);
}

}  // namespace ebl
