// Bit-sliced, temporally blocked multi-step kernel — the throughput path.
//
// A CTA owns one *tile* of one env layer and advances it n_steps steps per launch:
// the tile plus a halo (K rows above/below, one 32-cell word left/right) is read once
// from HBM (uint8 [row][col]), converted to bit-planes in shared memory, stepped, and
// the tile (not the halo) is written back once.  Cells at distance d from a region
// boundary that is not a grid edge are exact for d steps (the halo is the light cone),
// so n_steps <= K.  With the tile = the whole env (H*W <= 65536 cells) there is no halo
// and n_steps is unbounded: BASELINE C1 runs its 200 steps in ONE launch per env.
//
// Planes: B[2] (Burning, double-buffered, one zero row of padding above/below), X (Burned),
// ACT (per-thread overflow of the active list).  Per step, two block barriers:
//   P1 dense   (32 cells per op, each thread owns fixed words): any = 8-neighbour dilation
//              of B, act = (Unburned & any) | B; Bn[w] = B[w]; active cells appended to a
//              shared list with one warp-aggregated atomic per warp (cells beyond the
//              list capacity stay with their owner thread in ACT);
//   --- barrier ---
//   P2 sparse  one thread per active cell: the last two rng_word rounds on the
//              per-(env,step) prefix; Burning: integer survive test, burn-out clears Bn
//              and sets X; candidate: 8-bit neighbour mask from B, lambda/p in fp32 with the
//              fp64 guard (ember_device.cuh), ignition sets Bn (shared atomics);
//   --- barrier ---, swap B <-> Bn.
// Every cell of the tile is updated every step (quiescent ones by the bit-sliced copy),
// so cell-updates are counted densely as the reference does (emberline_main.cpp:432-433);
// results are bit-identical to k_step_tile and engine.cpp:134-159 by construction.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <algorithm>

#include "ember_bits.cuh"
#include "ember_device.cuh"
#include "ember_kernels.h"
#include "ember_params.h"

#ifndef EBL_PREFETCH
#define EBL_PREFETCH 0    // bulk L2 prefetch of the region's static layers at launch
#endif
#ifndef EBL_PREFETCH_FRONT
#define EBL_PREFETCH_FRONT 0  // prefetch next step's candidate statics at each ignition
#endif
#ifndef EBL_PF
#define EBL_PF prefetch_l2
#endif
#ifndef EBL_PHASE_PROF
#define EBL_PHASE_PROF 0  // per-phase clock64 profile (diagnostic builds: scripts/build_variant.sh)
#endif
#ifndef EBL_LAMBDA_ALL
#define EBL_LAMBDA_ALL 1  // slope-table, branch-free 8-direction lambda (terrain form)
#endif

namespace ebl {


// E envs per CTA (E = 1, or 2 for whole-env residency of envs <= 32768 cells): 128 threads per
// env in P1, one pooled active list in P2, so a heavy env shares its CTA's 128*E threads with a
// lighter one (the batch's kernel time is set by its slowest CTA: measured, scripts/imbalance.py).
// WPRC: words per region row when known at compile time (2: 64-wide, 4: 128-wide envs), else 0.
template <int MODE, int E, int WPRC>
__global__ void __launch_bounds__(kResThreads * E, 8 / E) k_step_blocked(StepArgs a, BlockGeom g) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int s_total[2];
  __shared__ int32_t s_newly[2][E];
  __shared__ int32_t s_cnt[E][4];
  // rng key prefixes (3 of rng_word's 5 rounds) of steps t .. t+63 in a ring, slot t & 127: 64 are
  // computed in parallel every 64 steps instead of one per step on the critical path
  __shared__ uint64_t s_prefix[E][128];
  __shared__ float s_pal[MODE == kStaticTerrain ? 512 : 1];  // terrain palette: fp32 src, gam
  __shared__ float s_kw[MODE == kStaticTerrain ? E : 1][8];    // kappa_wind of the wind in force
  // src32(class) * kappa_wind32(k) of the wind in force, palettes of <= 32 classes
  // (only in the whole-width instantiations: the extra 1 KB costs halo-tile launches occupancy)
  constexpr bool kRec = MODE == kStaticTerrain && WPRC != 0;
  __shared__ float s_srckw[kRec ? E : 1][kRec ? 32 * 8 : 1];
  // source-class records for whole-env regions (C1-like batches: measured faster); halo tiles of
  // large landscapes keep the fuel-byte gathers (their statics stream from DRAM; C3 measured
  // 22.5 ms vs 24.1 ms with the 8-byte records)
  const bool use_rec = kRec && a.nfuel && a.n_pal <= 32 && g.halo_rows == 0 && g.halo_cols == 0;

  const int env0 = blockIdx.z * E;
  constexpr int t_start = 0;
  const int W = a.w, BH = a.h;
  const int r0 = blockIdx.y * g.tile_h, c0 = blockIdx.x * g.tile_w;  // c0 % 32 == 0
  const int R0 = max(0, r0 - g.halo_rows), R1 = min(BH, r0 + g.tile_h + g.halo_rows);
  const int C0 = max(0, c0 - g.halo_cols), C1 = min(W, c0 + g.tile_w + g.halo_cols);
  const int RH = R1 - R0, RW = C1 - C0;
  const int wpr = WPRC ? WPRC : (RW + 31) >> 5;
  const int S = plane_stride(wpr);  // odd row stride: a warp's 32 rows hit 32 distinct banks
  const int PB = (2 * (RH + 2) + 2 * RH) * S;  // words of one env's planes: B[2], X, ACT
  uint32_t* const planes = reinterpret_cast<uint32_t*>(smem);
  // env s's planes: B[c] = planes + s*PB + c*(RH+2)*S, X = + 2*(RH+2)*S, ACT = X + RH*S
  auto Bplane = [&](int sub, int c) { return planes + sub * PB + c * (RH + 2) * S; };
  auto Xplane = [&](int sub) { return planes + sub * PB + 2 * (RH + 2) * S; };
  auto Aplane = [&](int sub) { return planes + sub * PB + (2 * (RH + 2) + RH) * S; };
  uint16_t* list = reinterpret_cast<uint16_t*>(planes + E * PB);
  const int cap = g.list_cap;
  const uint32_t last_mask = low_mask(RW - 32 * (wpr - 1));
  const int rot = wpr >= 32 ? 1 : 32 / wpr;  // list-build word rotation (see P1)
  // list entry -> region row: exact reciprocal division (entry * RW < 2^32)
  const uint32_t rw_magic = RW > 1 ? static_cast<uint32_t>((0x100000000ull + RW - 1) / RW) : 0u;

  const size_t ncell = static_cast<size_t>(BH) * W;
  const bool vec = (W & 15) == 0;  // 16-byte aligned rows (C0 is a multiple of 32)

  // ---- load: uint8 layers -> bit-planes ------------------------------------------------
  for (int sub = 0; sub < E; ++sub) {
    uint32_t* B0 = Bplane(sub, 0);
    uint32_t* B1 = Bplane(sub, 1);
    uint32_t* X = Xplane(sub);
    for (int i = threadIdx.x; i < wpr; i += blockDim.x) {  // zero padding rows of both buffers
      B0[i] = B1[i] = 0u;
      B0[(RH + 1) * S + i] = B1[(RH + 1) * S + i] = 0u;
    }
    const bool live = env0 + sub < a.n_envs;
    const uint8_t* __restrict__ in = a.in + (env0 + sub) * ncell;
    for (WordIter it(wpr, RH * wpr); it.ok(); it.next()) {
      const int nc = min(32, RW - 32 * it.j);
      uint32_t b = 0u, x = 0u;
      if (live) {
        const uint8_t* src = in + static_cast<size_t>(R0 + it.r) * W + C0 + 32 * it.j;
        if (nc == 32 && vec) {
          bytes_to_bits(src, b, x);
        } else {
          for (int k = 0; k < nc; ++k) {
            const uint8_t v = src[k];
            b |= static_cast<uint32_t>(v == 1) << k;
            x |= static_cast<uint32_t>(v == 2) << k;
          }
        }
      }
      B0[(it.r + 1) * S + it.j] = b;
      X[it.r * S + it.j] = x;
    }
  }
  if constexpr (MODE == kStaticTerrain) {
    for (int i = threadIdx.x; i < 2 * a.n_pal; i += blockDim.x)  // the palette entries in use: src, gam
      s_pal[i < a.n_pal ? i : 256 + i - a.n_pal] = __ldg(a.pal32 + (i < a.n_pal ? i : 256 + i - a.n_pal));
#if EBL_PREFETCH
    // the region's static layers are touched only along the fire front: one bulk L2 prefetch per
    // region row (whole env = one contiguous range) hides their first-touch DRAM latency
    const bool whole = RW == W;
    const int n_pf = whole ? E : E * RH;
    for (int i = threadIdx.x; i < n_pf; i += blockDim.x) {
      const int sub = whole ? i : i / RH, rr = whole ? 0 : i % RH;
      if (env0 + sub >= a.n_envs) continue;
      const size_t base = static_cast<size_t>(env0 + sub) * a.ter_stride + static_cast<size_t>(R0 + rr) * W + C0;
      const uint32_t cells = whole ? static_cast<uint32_t>(RH) * W : static_cast<uint32_t>(RW);
      prefetch_l2(a.elev + base, (cells * 4u) & ~15u);
      prefetch_l2(a.fuel + base, cells & ~15u);
    }
#endif
  }
  if (threadIdx.x < 4 * E) s_cnt[threadIdx.x >> 2][threadIdx.x & 3] = 0;
  if (threadIdx.x < 2) s_total[threadIdx.x] = 0;
  if (threadIdx.x < 2 * E) s_newly[threadIdx.x / E][threadIdx.x % E] = 0;
  for (int i = threadIdx.x; i < 64 * E; i += blockDim.x) {
    const int q = i >> 6, k = t_start + (i & 63);
    s_prefix[q][k & 127] = key_prefix(a.seed, a.streams[min(env0 + q, a.n_envs - 1)], a.step + static_cast<uint64_t>(k));
  }
  __syncthreads();

  const DiagCounters dg{a.diag};
  const uint64_t gbase = static_cast<uint64_t>(a.row_off + R0) * W + C0;  // RNG index of region (0,0)
  const int lane = threadIdx.x & 31;
  const int my_sub = E > 1 ? static_cast<int>(threadIdx.x) / kResThreads : 0;  // P1 ownership
  const int lt = E > 1 ? static_cast<int>(threadIdx.x) % kResThreads : static_cast<int>(threadIdx.x);
  // newly-ignited cells are counted only inside the output tile
  const int tr0 = r0 - R0, tr1 = min(r0 + g.tile_h, BH) - R0;
  const int tc0 = c0 - C0, tc1 = min(c0 + g.tile_w, W) - C0;
  int cur = 0;
  const int tj0 = tc0 >> 5, tj1 = (tc1 + 31) >> 5;
  const int twords = tj1 - tj0;
  // bit-planes of the output tile -> uint8 layer at `layer` (+ U/B/X counts when cnt3)
  // bit-planes of the output tile -> uint8 layer at `layer` (+ U/B/X counts when cnt3); rows
  // outside [row_lo, row_hi) (layer rows) are skipped
  auto store_tile = [&](const uint32_t* Bs, const uint32_t* X, uint8_t* __restrict__ layer, int32_t* cnt3,
                        int row_lo, int row_hi, int dst_shift) {
    for (WordIter it(twords, (tr1 - tr0) * twords); it.ok(); it.next()) {
      const int rr = tr0 + it.r, j = tj0 + it.j;
      const int lrow = R0 + rr;
      if (lrow < row_lo || lrow >= row_hi) continue;
      const uint32_t b = Bs[(rr + 1) * S + j], x = X[rr * S + j];
      const int nc = min(32, RW - 32 * j);
      if (cnt3) {
        cnt3[0] += nc - __popc(b) - __popc(x);
        cnt3[1] += __popc(b);
        cnt3[2] += __popc(x);
      }
      uint8_t* dst = layer + static_cast<size_t>(lrow + dst_shift) * W + C0 + 32 * j;
      if (nc == 32 && vec) {
        bits_to_bytes(b, x, dst);
      } else {
        for (int k = 0; k < nc; ++k) dst[k] = static_cast<uint8_t>(((b >> k) & 1u) | (((x >> k) & 1u) << 1));
      }
    }
  };

#if EBL_PHASE_PROF
  // phase profile: thread 0 times the barrier-to-barrier phases; each warp's lane 0 times its own
  // dense pass, list build and P2 work; the slowest warp's times are accumulated
  __shared__ long long s_pw[5][kResThreads * E / 32];
  __shared__ int s_ncand;
  long long pr_t0 = 0, pr[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, pw0 = 0, pw1 = 0;
  if (threadIdx.x == 0) s_ncand = 0;
  if (threadIdx.x < 5 * (kResThreads * E / 32)) (&s_pw[0][0])[threadIdx.x] = 0;
#define EBL_PW_MARK(v) \
  if (a.prof && lane == 0) v = clock64();
#else
#define EBL_PW_MARK(v)
#endif
  for (int t = t_start; t < g.n_steps; ++t) {
    const int par = t & 1;
#if EBL_PHASE_PROF
    if (a.prof && threadIdx.x == 0) pr_t0 = clock64();
    EBL_PW_MARK(pw0)
#endif
    if (threadIdx.x == 0) s_total[par ^ 1] = 0;  // the other parity's counters are free until the next step
    if (threadIdx.x < E) s_newly[par ^ 1][threadIdx.x] = 0;
    const int srow = sched_row(a, a.step + static_cast<uint64_t>(t));  // wind in force
    if constexpr (MODE == kStaticTerrain) {  // read by P2, after the first barrier
      if ((t == t_start || a.sched_len > 1) && threadIdx.x < 8 * E) {
        const int q = threadIdx.x >> 3;
        s_kw[q][threadIdx.x & 7] = __ldg(a.kw32 + static_cast<size_t>(srow) * a.kw_sched_stride +
                                         static_cast<size_t>(min(env0 + q, a.n_envs - 1)) * a.kw_stride +
                                         (threadIdx.x & 7));
      }
      if (use_rec && (t == t_start || a.sched_len > 1)) {
        for (int i = threadIdx.x; i < E * a.n_pal * 8; i += blockDim.x) {
          const int q = i / (a.n_pal * 8), ck = i - q * a.n_pal * 8;
          const float kw = __ldg(a.kw32 + static_cast<size_t>(srow) * a.kw_sched_stride +
                                 static_cast<size_t>(min(env0 + q, a.n_envs - 1)) * a.kw_stride + (ck & 7));
          s_srckw[q][ck] = s_pal[ck >> 3] * kw;  // the same product terrain_lambda32 forms
        }
      }
    }
    // ---- P1: each thread owns whole rows of one env; the 3x3 dilation slides along the row in
    //      registers (3 shared loads per word: north, own, south) ------------------------------
    int cnt = 0;
    bool ovf = false;
    {
      const uint32_t* B = Bplane(my_sub, cur);
      uint32_t* Bn = Bplane(my_sub, cur ^ 1);
      const uint32_t* X = Xplane(my_sub);
      uint32_t* ACT = Aplane(my_sub);
      uint32_t* const ACT_P1 = ACT;
      for (int r = lt; r < RH; r += kResThreads) {
        const uint32_t* up = B + (r + 2) * S;
        const uint32_t* mid = B + (r + 1) * S;
        const uint32_t* dn = B + r * S;
        uint32_t* bn = Bn + (r + 1) * S;
        const uint32_t* xr = X + r * S;
        uint32_t* ar = ACT + r * S;
        uint32_t vl = 0u;                            // column j-1: north | own | south
        uint32_t uc = up[0], mc = mid[0], dc = dn[0];
        uint32_t vc = uc | mc | dc;
#pragma unroll 4
        for (int j = 0; j < wpr; ++j) {
          uint32_t un = 0u, mn = 0u, dnn = 0u;
          if (j + 1 < wpr) {
            un = up[j + 1];
            mn = mid[j + 1];
            dnn = dn[j + 1];
          }
          const uint32_t vn = un | mn | dnn;
          // west/east neighbours of all three rows, plus north/south of the own column
          const uint32_t any = ((vc << 1) | (vl >> 31)) | ((vc >> 1) | (vn << 31)) | uc | dc;
          bn[j] = mc;
          const uint32_t valid = j + 1 < wpr ? 0xffffffffu : last_mask;
          const uint32_t act = ((~(mc | xr[j]) & valid) & any) | mc;
          ar[j] = act;
          cnt += __popc(act);
          vl = vc;
          vc = vn;
          uc = un;
          mc = mn;
          dc = dnn;
        }
      }
#if EBL_PHASE_PROF
      if (a.prof && lane == 0) { pw1 = clock64(); s_pw[0][threadIdx.x >> 5] = pw1 - pw0; }
#endif
      // List build, one warp-aggregated reservation per warp and step (skipped by quiet warps).
      // The warp's ACT words are re-dealt to its lanes so that a row with a long front is spread
      // over several lanes: in 128-row block rb, lane l extracts word j of row rb + ((l + rot*j) & 31)
      // (a rotation per word column: every (row, word) exactly once).  ovf words stay with that lane.
      if (__ballot_sync(0xffffffffu, cnt > 0)) {
        __syncwarp();  // the warp's ACT rows (its own dense-pass output) are visible to all lanes
        int c2 = 0;
        for (int rb = lt & ~31; rb < RH; rb += kResThreads)
          for (int j = 0; j < wpr; ++j) {
            const int r = rb + ((lane + rot * j) & 31);
            if (r < RH) c2 += __popc(ACT_P1[r * S + j]);
          }
#if EBL_PHASE_PROF
        if (a.prof && lane == 0) s_pw[3][threadIdx.x >> 5] = clock64() - pw1;
#endif
        int incl = c2;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        int base = 0;
        if (lane == 31) base = atomicAdd(&s_total[par], incl);
        base = __shfl_sync(0xffffffffu, base, 31) + incl - c2;
#if EBL_PHASE_PROF
        if (a.prof && lane == 0) s_pw[4][threadIdx.x >> 5] = clock64() - pw1;
#endif
        if (c2 > 0) {
          const int tag = E > 1 ? (my_sub << 15) : 0;
          for (int rb = lt & ~31; rb < RH; rb += kResThreads)
            for (int j = 0; j < wpr; ++j) {
              const int r = rb + ((lane + rot * j) & 31);
              if (r >= RH) continue;
              uint32_t rest = ACT_P1[r * S + j];
              if (!rest) continue;
              const int cell0 = r * RW + 32 * j;
              while (rest && base < cap) {
                const int bit = __ffs(rest) - 1;
                rest &= rest - 1;
                list[base++] = static_cast<uint16_t>((cell0 + bit) | tag);
              }
              ACT_P1[r * S + j] = rest;  // overflow beyond the list capacity: done by this lane in P2
              ovf |= rest != 0u;
            }
        }
      }
    }
#if EBL_PHASE_PROF
    if (a.prof) {
      __syncwarp();
      if (lane == 0) s_pw[1][threadIdx.x >> 5] = clock64() - pw1;
    }
#endif
    __syncthreads();
#if EBL_PHASE_PROF
    if (a.prof && threadIdx.x == 0) {
      const long long t1 = clock64();
      pr[0] += t1 - pr_t0;
      pr_t0 = t1;
      pr[2] += s_total[par];
      long long m0 = 0, m1 = 0, m3 = 0, m4 = 0;
      for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) {
        m0 = max(m0, s_pw[0][q]);
        m1 = max(m1, s_pw[1][q]);
        m3 = max(m3, s_pw[3][q]);
        m4 = max(m4, s_pw[4][q]);
        s_pw[3][q] = s_pw[4][q] = 0;
      }
      pr[4] += m0;
      pr[5] += m1;
      pr[8] += m3;
      pr[9] += m4;
    }
    EBL_PW_MARK(pw0)
#endif
    // ---- P2: sparse decisions over the pooled list ------------------------------------------
    int newly[E];
#pragma unroll
    for (int q = 0; q < E; ++q) newly[q] = 0;
    const int total = min(s_total[par], cap);
    if (((t - t_start) & 63) == 63 && t + 1 < g.n_steps) {  // refill the ring with steps t+1 .. t+64
      for (int i = threadIdx.x; i < 64 * E; i += blockDim.x) {
        const int q = i >> 6, k = i & 63;
        s_prefix[q][(t + 1 + k) & 127] = key_prefix(a.seed, a.streams[min(env0 + q, a.n_envs - 1)],
                                                   a.step + static_cast<uint64_t>(t + 1 + k));
      }
    }
    auto decide = [&](int sub, int lc) {
      const uint32_t* B = Bplane(sub, cur);
      uint32_t* Bn = Bplane(sub, cur ^ 1);
      const int rr = RW > 1 ? static_cast<int>(__umulhi(static_cast<uint32_t>(lc), rw_magic)) : lc, cc = lc - rr * RW;
      const int wi = (rr + 1) * S + (cc >> 5);
      const uint32_t bit = 1u << (cc & 31);
      const uint64_t m = cell_bits53(s_prefix[sub][t & 127], gbase + static_cast<uint64_t>(rr) * W + cc, 0);
      // 3-cell windows (columns cc-1, cc, cc+1 -> bits 0..2) of the rows below, at and above the
      // cell; padding rows cover rr-1 = -1 and rr+1 = RH, bits past RW are never set
      const int j = cc >> 5, b = cc & 31;
      auto win3 = [&](const uint32_t* row) -> uint32_t {
        const uint32_t wj = row[j];
        uint32_t v = b > 0 ? wj >> (b - 1) : ((j > 0 ? row[j - 1] >> 31 : 0u) | (wj << 1));
        if (b == 31) v = (v & 3u) | ((j + 1 < wpr ? row[j + 1] & 1u : 0u) << 2);
        return v & 7u;
      };
      const uint32_t mid = win3(B + (rr + 1) * S);
      if (mid & 2u) {
        if (m >= a.pc_thr) {
          atomicAnd(Bn + wi, ~bit);
          atomicOr(Xplane(sub) + rr * S + (cc >> 5), bit);
        }
      } else {
        // burning-source mask in kNeighborOffsets order (u_k = v - d_k): E <- (r, c-1),
        // NE <- (r-1, c-1), N <- (r-1, c), NW <- (r-1, c+1), W <- (r, c+1), SW <- (r+1, c+1),
        // S <- (r+1, c), SE <- (r+1, c-1)
        const uint32_t dnw = win3(B + rr * S), upw = win3(B + (rr + 2) * S);
        const uint32_t nb = (mid & 1u) | (dnw << 1) | ((mid >> 2) << 4) | ((upw >> 2) << 5) |
                            ((upw & 2u) << 5) | ((upw & 1u) << 7);
#if EBL_PHASE_PROF
        if (a.prof) atomicAdd(&s_ncand, 1);
#endif
        bool ig;
        if (use_rec)
          ig = ignite_terrain_rec(terrain_view(a, env0 + sub, srow),
                                  a.slope32 + static_cast<size_t>(env0 + sub) * a.ter_stride * 8,
                                  a.nfuel + static_cast<size_t>(env0 + sub) * a.ter_stride, s_srckw[sub], s_pal + 256,
                                  a.alpha_s_l2, W, R0 + rr, C0 + cc, nb, m, dg);
        else if constexpr (MODE == kStaticTerrain && EBL_LAMBDA_ALL)
          ig = ignite_terrain_tab(terrain_view(a, env0 + sub, srow),
                                  a.slope32 + static_cast<size_t>(env0 + sub) * a.ter_stride * 8, s_pal, s_kw[sub],
                                  W, BH, R0 + rr, C0 + cc, nb, m, dg);
        else
          ig = ignite<MODE>(a, env0 + sub, R0 + rr, C0 + cc, nb, m, dg, srow);
        if (ig) {
          atomicOr(Bn + wi, bit);
#if EBL_PREFETCH_FRONT
          if (use_rec) {
            // the ignited cell's unburned neighbours are next step's candidates: pull their slope
            // and source-class records (rows r-1..r+1, 3 cells each) toward the SM meanwhile
            const int gr = R0 + rr, gc = C0 + cc;
            const size_t eb = static_cast<size_t>(env0 + sub) * a.ter_stride;
            const int c0 = max(gc - 1, 0), c1 = min(gc + 1, W - 1);
#pragma unroll
            for (int d = -1; d <= 1; ++d) {
              const int rowp = min(max(gr + d, 0), BH - 1);
              const size_t rb = eb + static_cast<size_t>(rowp) * W;
              EBL_PF(a.slope32 + (rb + c0) * 8);
              EBL_PF(a.slope32 + (rb + c1) * 8 + 7);
              EBL_PF(a.nfuel + rb + c0);
            }
          }
#endif
          const int in_tile = (rr >= tr0 && rr < tr1 && cc >= tc0 && cc < tc1);
#pragma unroll
          for (int q = 0; q < E; ++q) newly[q] += (q == sub) ? in_tile : 0;
        }
      }
    };
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
      const int e = list[i];
      if (E > 1) decide(e >> 15, e & 0x7fff);
      else decide(0, e);
    }
    if (ovf) {
      uint32_t* ACT = Aplane(my_sub);
      for (int rb = lt & ~31; rb < RH; rb += kResThreads)
        for (int j = 0; j < wpr; ++j) {
          const int r = rb + ((lane + rot * j) & 31);
          if (r >= RH) continue;
          uint32_t rest = ACT[r * S + j];
          while (rest) {
            const int bit = __ffs(rest) - 1;
            rest &= rest - 1;
            decide(my_sub, r * RW + 32 * j + bit);
          }
        }
    }
    if (t == g.n_steps - 1) {
#pragma unroll
      for (int q = 0; q < E; ++q) {
        int v = newly[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && v) atomicAdd(&s_newly[par][q], v);
      }
    }
#if EBL_PHASE_PROF
    if (a.prof) {
      __syncwarp();
      if (lane == 0) s_pw[2][threadIdx.x >> 5] = clock64() - pw0;
    }
#endif
    __syncthreads();
#if EBL_PHASE_PROF
    if (a.prof && threadIdx.x == 0) {
      pr[1] += clock64() - pr_t0;
      long long m2 = 0;
      for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) m2 = max(m2, s_pw[2][q]);
      pr[6] += m2;
    }
#endif
    cur ^= 1;
    if (a.traj) {  // record (run_stochastic(record=true), engine.cpp:116): this step's tile
      for (int sub = 0; sub < E; ++sub)
        if (env0 + sub < a.n_envs)
          store_tile(Bplane(sub, cur), Xplane(sub), a.traj + ((a.traj_t0 + t) * a.n_envs + env0 + sub) * ncell,
                     nullptr, 0, BH, 0);
    }
  }

#if EBL_PHASE_PROF
  if (a.prof && threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) {
    pr[3] = g.n_steps;
    pr[7] = s_ncand;
    for (int q = 0; q < 10; ++q) a.prof[env0 * 10 + q] = pr[q];
  }
#endif
  // ---- store the tiles: bit-planes -> uint8, counts -----------------------------------------
  for (int sub = 0; sub < E; ++sub) {
    if (env0 + sub >= a.n_envs) break;
    int32_t cnt3[3] = {0, 0, 0};
    store_tile(Bplane(sub, cur), Xplane(sub), a.out + (env0 + sub) * ncell, cnt3, a.store_lo, a.store_hi, 0);
    if (a.out2)  // the host's buffer directly (mapped pinned memory): no device -> host copy after the launch
      store_tile(Bplane(sub, cur), Xplane(sub), a.out2 + (env0 + sub) * ncell, nullptr, a.store_lo, a.store_hi, 0);
    for (int p = 0; p < a.n_peers; ++p)  // fused halo exchange: owned rows straight into the neighbour
      store_tile(Bplane(sub, cur), Xplane(sub), a.peer_out[p], nullptr,
                 a.peer_lo[p], a.peer_hi[p], a.peer_dst[p] - a.peer_lo[p]);
    if (a.counts) {
      atomicAdd(&s_cnt[sub][0], cnt3[0]);
      atomicAdd(&s_cnt[sub][1], cnt3[1]);
      atomicAdd(&s_cnt[sub][2], cnt3[2]);
    }
  }
  if (a.counts) {
    __syncthreads();
    if (threadIdx.x < 4 * E) {
      const int sub = threadIdx.x >> 2, k = threadIdx.x & 3;
      if (env0 + sub < a.n_envs) {
        if (k < 3) atomicAdd(a.counts + (env0 + sub) * 4 + k, s_cnt[sub][k]);
        else if (g.n_steps > 0) atomicAdd(a.counts + (env0 + sub) * 4 + 3, s_newly[(g.n_steps - 1) & 1][sub]);
      }
    }
  }
}

bool phase_prof_built() { return EBL_PHASE_PROF != 0; }

size_t blocked_smem_bytes(int region_h, int region_w, int list_cap, int envs_per_cta) {
  const size_t S = plane_stride((region_w + 31) / 32);
  const size_t planes = (2 * (static_cast<size_t>(region_h) + 2) + 2 * region_h) * S * sizeof(uint32_t);
  const size_t list = static_cast<size_t>(list_cap) * sizeof(uint16_t);
  return envs_per_cta * planes + ((list + 15) & ~size_t(15));
}

static int list_cap_for(int cells) {
  // active cells are ~1-3% of an env per step; a quarter of the region is ample and an
  // overflow is still exact (owner threads finish the rest)
  const int cap = (cells + 3) / 4;
  return cap < 1024 ? (cells < 1024 ? cells : 1024) : cap;
}

bool resident_fits(int h, int w) {
  return static_cast<size_t>(h) * w <= 65536 &&
         blocked_smem_bytes(h, w, list_cap_for(h * w), 1) <= kResMaxSmem;
}

BlockGeom plan_blocks(int buf_h, int w, int n_steps, bool force_tiles, int row_off, int n_envs,
                      int envs_per_cta) {
  BlockGeom g{};
  g.row_off = row_off;
  g.envs_per_cta = 1;
  if (!force_tiles && resident_fits(buf_h, w)) {  // whole env per CTA, all steps fused
    g.tile_h = buf_h;
    g.tile_w = ((w + 31) / 32) * 32;
    g.halo_rows = 0;
    g.halo_cols = 0;
    g.n_steps = n_steps;
  } else {
    // tile geometry of halo-tiled runs (EBL_TILE_H / EBL_TILE_W override, multiples of 32 columns)
    static const int tile_h_env = [] {
      const char* e = std::getenv("EBL_TILE_H");
      return e ? std::max(1, std::atoi(e)) : kBlockTileH;
    }();
    static const int tile_w_env = [] {
      const char* e = std::getenv("EBL_TILE_W");
      return e ? std::max(32, std::atoi(e) / 32 * 32) : kBlockTileW;
    }();
    static const int halo_env = [] {  // EBL_TILE_HALO: rows of light-cone halo = steps per launch
      const char* e = std::getenv("EBL_TILE_HALO");
      return e ? std::max(1, std::min(32, std::atoi(e))) : kBlockHalo;
    }();
    g.halo_rows = halo_env;
    g.tile_w = w <= tile_w_env + 64 ? ((w + 31) / 32) * 32 : tile_w_env;
    g.halo_cols = g.tile_w >= w ? 0 : 32;
    g.tile_h = tile_h_env;
    if (g.tile_h >= buf_h) {
      g.tile_h = buf_h;
      g.halo_rows = 0;
    }
    const bool fuzzy = g.halo_rows > 0 || g.halo_cols > 0;
    const int lim = g.halo_rows > 0 ? g.halo_rows : kBlockHalo;  // steps per launch <= the light-cone halo
    g.n_steps = !fuzzy ? n_steps : (n_steps < lim ? n_steps : lim);
  }
  const int rh = g.tile_h + 2 * g.halo_rows, rw = g.tile_w + 2 * g.halo_cols;
  g.list_cap = g.envs_per_cta * list_cap_for((rh < buf_h ? rh : buf_h) * (rw < w ? rw : w));
  return g;
}

template <int MODE, int E, int WPRC>
static cudaError_t launch_blocked_w(const StepArgs& a, const BlockGeom& g, size_t sm, cudaStream_t s) {
  cudaError_t e = smem_opt_in(reinterpret_cast<const void*>(k_step_blocked<MODE, E, WPRC>), sm);
  if (e != cudaSuccess) return e;
  const dim3 grid((a.w + g.tile_w - 1) / g.tile_w, (a.h + g.tile_h - 1) / g.tile_h, (a.n_envs + E - 1) / E);
  k_step_blocked<MODE, E, WPRC><<<grid, kResThreads * E, sm, s>>>(a, g);
  return cudaGetLastError();
}

template <int MODE, int E>
static cudaError_t launch_blocked_t(const StepArgs& a, const BlockGeom& g, size_t sm, cudaStream_t s) {
  // compile-time words per row only when every region spans the full width (edge tiles of a
  // column-tiled grid are narrower; their last-word mask depends on the true word count)
  if (g.tile_w >= a.w) {
    const int wpr = (a.w + 31) / 32;
    if (wpr == 4) return launch_blocked_w<MODE, E, 4>(a, g, sm, s);
    if (wpr == 2) return launch_blocked_w<MODE, E, 2>(a, g, sm, s);
  }
  return launch_blocked_w<MODE, E, 0>(a, g, sm, s);
}

cudaError_t launch_step_blocked(const StepArgs& a, int mode, const BlockGeom& g, cudaStream_t s) {
  const int rh = g.tile_h + 2 * g.halo_rows, rw = g.tile_w + 2 * g.halo_cols;
  const size_t sm = blocked_smem_bytes(rh < a.h ? rh : a.h, rw < a.w ? rw : a.w, g.list_cap, 1);
  if (mode == kStaticTables) return launch_blocked_t<kStaticTables, 1>(a, g, sm, s);
  return launch_blocked_t<kStaticTerrain, 1>(a, g, sm, s);
}

}  // namespace ebl
