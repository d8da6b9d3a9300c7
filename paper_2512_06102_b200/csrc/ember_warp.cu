// Warp-local resident kernel: whole env per CTA, all steps fused, ONE block barrier per step.
//
// Same transition as k_step_blocked (engine.cpp:12-38, next_fire_cell) and the same bit-planes
// (B double-buffered with zero padding rows, X), but no CTA-wide active list: rows are dealt to
// warps interleaved (block rb, lane l of warp w owns row rb + 4l + w, so a front spanning a few
// rows is shared by all four warps), and each warp decides the active cells of its own rows:
//   dense   per lane, its row: 8-neighbour dilation of B, Bn = B, act = (Unburned & any) | B
//           (stored to the lane's ACT row), cnt = popc(act);
//   warp    inclusive scan of cnt; pass p: lane l takes the warp's active cell p*32 + l, finds
//           the owning lane by a 5-step shuffle search of the exclusive counts and the bit by
//           popc over that row's ACT words + fns; decides it (survive test / slope-table lambda
//           with the fp64 guard, ember_device.cuh) and updates Bn / X of that row (only this
//           warp writes those words in this step);
//   --- one barrier ---, swap B / Bn.
// The pooled list of k_step_blocked costs a barrier and a per-bit list build per step; here a
// warp only waits for itself until the end of the step.  Bit-identical results (decisions are
// per cell; the RNG is counter-based).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <mutex>
#include <unordered_map>

#include "ember_bits.cuh"
#include "ember_device.cuh"
#include "ember_kernels.h"
#include "ember_pdl.cuh"
#include "ember_params.h"

#ifndef EBL_PHASE_PROF
#define EBL_PHASE_PROF 0
#endif

#ifndef EBL_WARP_UNROLL2  // step loop unrolled by two (B / Bn roles alternate)
#define EBL_WARP_UNROLL2 1  // C1 kernel 0.524 -> 0.509 ms (a few spilled bytes)
#endif
#ifndef EBL_WARP_MICRO  // newly-ignited counts from the planes at the store (not per ignition),
#define EBL_WARP_MICRO 1  // schedule / record branches hoisted out of the step loop
#endif
#ifndef EBL_WARP_FAST  // decide passes without divergent branches: branch-free neighbour windows
#define EBL_WARP_FAST 1  // (zeroed guard words), SWAR + table n-th set bit, burning and candidate
#endif                   // cells through one code path (even compile-time words per row, pot32t)
#ifndef EBL_WARP_POT  // lambda terms from the pot32t table (0: slope + source-class records)
#define EBL_WARP_POT 1
#endif

namespace ebl {

namespace {

constexpr int kWpThreads = 128;  // 4 warps

#if EBL_PHASE_PROF
__device__ __forceinline__ long long pw_wait_dummy(long long v) { return v; }
#endif

// Position of the q-th (0-based) set bit of v (q < popc(v)): popc binary search, 5 levels.
__device__ __forceinline__ int nth_set_bit(uint32_t v, int q) {
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

// Position of the q-th (0-based) set bit of v (q < popc(v)) with a shallower dependency chain:
// SWAR byte counts, their inclusive prefix in one multiply, the byte by three compares, the bit
// from a 256-entry table of packed 3-bit positions (kNthBitLut, read-only cache).
__device__ __forceinline__ int nth_set_bit_lut(uint32_t v, int q, const uint32_t* lut) {
  uint32_t c = v - ((v >> 1) & 0x55555555u);
  c = (c & 0x33333333u) + ((c >> 2) & 0x33333333u);
  c = (c + (c >> 4)) & 0x0f0f0f0fu;
  const uint32_t cum = c * 0x01010101u;  // byte k: set bits in bytes 0..k
  const uint32_t qq = static_cast<uint32_t>(q);
  const int k = (qq >= (cum & 0xffu)) + (qq >= ((cum >> 8) & 0xffu)) + (qq >= ((cum >> 16) & 0xffu));
  const int before = k ? static_cast<int>((cum << 8 >> (8 * k)) & 0xffu) : 0;
  const uint32_t byte = (v >> (8 * k)) & 0xffu;
  return 8 * k + static_cast<int>((__ldg(lut + byte) >> (3 * (q - before))) & 7u);
}

// DIMC: the env's side when the env is a DIMC x DIMC square known at compile time (128: C1, 64:
// C2-sized), else 0; WPRC: words per row when known (2, 4), else 0.
#ifndef EBL_WARP_MINB
#define EBL_WARP_MINB 8  // 64 registers; 7 (72 registers, still one wave for C1): same C1, slower C3
#endif
// One region: one tile of one env's layer plus its light-cone halo (the whole env for resident
// launches); H x RW region cells, layer BH x W.  Grid launches run the CTA's own region, work-list
// launches (a.list_mode == 2) loop over the listed tiles (k_step_warp below).  Whole-env
// instantiations pass compile-time tile coordinates.
template <int MODE, int WPRC, int DIMC, bool EXIT = false>
__device__ __forceinline__ void warp_region(const StepArgs& a, const BlockGeom& g, const int env, const int bxi,
                                            const int byi, const int ntx, const int nty) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int32_t s_cnt[3];
  __shared__ int32_t s_newly;
  __shared__ uint64_t s_prefix[128];  // rng key prefixes, slot t & 127, refilled 64 steps at a time
  constexpr bool kTer = MODE == kStaticTerrain;
  __shared__ float s_pal[kTer ? 512 : 1];
  __shared__ float s_kw[8];
  __shared__ float s_srckw[kTer ? 32 * 8 : 1];
  // the fast decide path: even compile-time words per row leave a zero padding word after every
  // plane row (stride wpr | 1), so the neighbour windows need no bounds branches
  constexpr bool kFast = EBL_WARP_FAST && EBL_WARP_MICRO && kTer && WPRC != 0 && (WPRC & 1) == 0;

  const int n_steps = g.n_steps;
  const int BH = DIMC ? DIMC : a.h, W = DIMC ? DIMC : a.w;
  const int r0 = DIMC ? 0 : byi * g.tile_h, c0 = DIMC ? 0 : bxi * g.tile_w;  // c0 % 32 == 0
  // fixed regions: (tile + 2 halo) rows / columns for every tile, clamped inside the layer
  const bool fixed = !DIMC && g.fixed_region;
  const int frh = g.tile_h + 2 * g.halo_rows, frw = g.tile_w + 2 * g.halo_cols;
  const int R0 = DIMC ? 0 : fixed ? min(max(0, r0 - g.halo_rows), BH - frh) : max(0, r0 - g.halo_rows);
  const int R1 = DIMC ? BH : fixed ? R0 + frh : min(BH, r0 + g.tile_h + g.halo_rows);
  const int C0 = DIMC ? 0 : fixed ? min(max(0, c0 - g.halo_cols), W - frw) : max(0, c0 - g.halo_cols);
  const int C1 = DIMC ? W : fixed ? C0 + frw : min(W, c0 + g.tile_w + g.halo_cols);
  const int H = R1 - R0, RW = C1 - C0;
  const int wpr = WPRC ? WPRC : (RW + 31) >> 5;
  const int S = plane_stride(wpr);
  // plane row R starts at word R*S + (R >> 2): the 32 lanes of a warp own rows 4 apart, and the
  // extra word every 4 rows makes their stride 4S+1 (odd) -> 32 distinct banks
  auto ro = [S](int R) { return R * S + (R >> 2); };
  const int PH = ro(H + 2) + 1;  // words of a B plane (H + 2 rows)
  uint32_t* const Bp0 = reinterpret_cast<uint32_t*>(smem) + 4;  // 4 zero guard words before the planes
  uint32_t* const Bp1 = Bp0 + PH;
  uint32_t* const X = Bp1 + PH;
  uint32_t* const ACT = X + PH;
  const size_t ncell = static_cast<size_t>(BH) * W;
  const bool vec = (W & 15) == 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t last_mask = low_mask(RW - 32 * (wpr - 1));
  // the output tile inside the region (rows tr0..tr1, words tj0..tj1)
  const int tr0 = r0 - R0, tr1 = (DIMC ? BH : min(r0 + g.tile_h, BH)) - R0;
  const int tc0 = c0 - C0, tc1 = (DIMC ? W : min(c0 + g.tile_w, W)) - C0;
  const int tj0 = tc0 >> 5, tj1 = (tc1 + 31) >> 5, twords = tj1 - tj0;

  // ---- quiet tiles of a halo-tiled run: skipped outright -----------------------------------------
  // A tile whose own and 8 neighbours' output tiles had no burning cell after the previous launch
  // has a quiet region (the halo lies in the neighbours); after two quiet launches both layer
  // buffers hold its (canonical) bytes, so there is nothing to load, step or store.
  const size_t tile_id = (static_cast<size_t>(env) * nty + byi) * ntx + bxi;
  int streak0 = 0;
  // work-list launches (C3, one batch): the in-place record of this tile gives its quiet streak;
  // listed tiles always run (the list holds exactly the tiles the skip rule would not skip)
  if (a.list_mode == 2) streak0 = (reinterpret_cast<const int4*>(a.trec)[tile_id].x >> 1) & 3;
  const int4* const tf_in = reinterpret_cast<const int4*>(a.tflag_in);
  int4* const tf_out = reinterpret_cast<int4*>(a.tflag_out);
  if (tf_in) {
    __shared__ int s_skip;
    if (threadIdx.x == 0) {
      const int4 me = tf_in[tile_id];
      bool quiet = true;
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const int ty = byi + dy, tx = bxi + dx;
          if (ty >= 0 && ty < nty && tx >= 0 && tx < ntx)
            quiet &= !(tf_in[(static_cast<size_t>(env) * nty + ty) * ntx + tx].x & 1);
        }
      // tiles holding halo rows a neighbour shard writes are never skipped outright unless those
      // writes mark the records (halo_marked); DESIGN.md §6 gives the distance argument that keeps
      // the other tiles' skip decisions exact
      const bool exposed = !a.halo_marked && (r0 < a.keep_lo || r0 + g.tile_h > a.keep_hi);
      s_skip = quiet && ((me.x >> 1) & 3) >= 2 && !exposed;
      if (s_skip) {
        tf_out[tile_id] = me;
        if (a.counts) {
          atomicAdd(a.counts + env * 4 + 0, me.y);
          atomicAdd(a.counts + env * 4 + 2, me.w);
        }
      }
    }
    __syncthreads();
    if (s_skip) {
      if (threadIdx.x == 0 && a.diag) atomicAdd(a.diag + 3, 1ull);
      return;
    }
    streak0 = (tf_in[tile_id].x >> 1) & 3;
  }
  if (threadIdx.x == 0 && a.diag) {  // tile statistics: processed / launched regions
    atomicAdd(a.diag + 2, 1ull);
    if (a.list_mode != 2) atomicAdd(a.diag + 3, 1ull);
  }
  // ---- load ----------------------------------------------------------------------------------
  if constexpr (kFast) {  // guard words, padding words and padding rows of both B planes: zero
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
  const uint8_t* __restrict__ in = a.in + env * ncell;
  uint32_t any_b = 0u;  // a burning cell anywhere in the region
  uint32_t noncanon = 0u;  // (records) a byte that is not a FireState in the region
  for (WordIter it(wpr, H * wpr); it.ok(); it.next()) {
    const int nc = min(32, RW - 32 * it.j);
    uint32_t b = 0u, x = 0u;
    const uint8_t* src = in + static_cast<size_t>(R0 + it.r) * W + C0 + 32 * it.j;
    if (nc == 32 && vec) {
      if (DIMC) bytes_to_bits(src, b, x);
      else bytes_to_bits_nc(src, b, x, noncanon);
    } else {
      for (int k = 0; k < nc; ++k) {
        const uint8_t v = src[k];
        b |= static_cast<uint32_t>(v == 1) << k;
        x |= static_cast<uint32_t>(v == 2) << k;
        noncanon |= v > 2;
      }
    }
    Bp0[ro(it.r + 1) + it.j] = b;
    X[ro(it.r) + it.j] = x;
    any_b |= b;
  }
  const bool use_tab = kTer && a.pot32t && EBL_WARP_POT;  // one wind for all steps: precomputed terms
  const bool use_rec = kTer && a.nfuel && a.n_pal <= 32;
  auto load_wind = [&](int srow) {  // kappa_wind of the wind in force (+ the src * kappa_wind table)
    if constexpr (kTer) {
      if (threadIdx.x < 8)
        s_kw[threadIdx.x] = __ldg(a.kw32 + static_cast<size_t>(srow) * a.kw_sched_stride +
                                  static_cast<size_t>(env) * a.kw_stride + threadIdx.x);
      if (use_rec)
        for (int i = threadIdx.x; i < a.n_pal * 8; i += blockDim.x)
          s_srckw[i] = __ldg(a.pal32 + (i >> 3)) *
                       __ldg(a.kw32 + static_cast<size_t>(srow) * a.kw_sched_stride +
                             static_cast<size_t>(env) * a.kw_stride + (i & 7));
    }
  };
  if constexpr (kTer)
    for (int i = threadIdx.x; i < 2 * a.n_pal; i += blockDim.x)  // the palette entries in use: src, gam
      s_pal[i < a.n_pal ? i : 256 + i - a.n_pal] = __ldg(a.pal32 + (i < a.n_pal ? i : 256 + i - a.n_pal));
  load_wind(sched_row(a, a.step));
  if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_newly = 0;
  const uint64_t stream = a.streams[env];
  for (int k = threadIdx.x; k < 64; k += blockDim.x) s_prefix[k] = key_prefix(a.seed, stream, a.step + k);
  // a region without a burning cell does not change in n_steps <= halo steps (no draw can flip an
  // Unburned cell without a burning neighbour; the light cone of outside fire stays in the halo):
  // straight to the store (which maps other byte values to Unburned as a step does)
  const int n_run = __syncthreads_or(any_b != 0u) || a.traj ? n_steps : 0;
  // a quiet region whose bytes are all FireStates stores exactly what it loaded: both layer buffers
  // then hold the tile's canonical bytes at once (records: quiet streak 2 after one launch, so the
  // launch after a call's first one does not rerun every quiet tile)
  const bool canon_quiet = !DIMC && n_run == 0 && (a.list_mode || a.tflag_out) && !__syncthreads_or(noncanon != 0u);

  const DiagCounters dg{a.diag};
  const uint64_t gbase = static_cast<uint64_t>(a.row_off + R0) * W + C0;  // RNG index of region (0, 0)
  auto win3 = [&](const uint32_t* row, int j, int b) -> uint32_t {  // columns c-1, c, c+1 -> bits 0..2
    const uint32_t wj = row[j];
    uint32_t v = b > 0 ? wj >> (b - 1) : ((j > 0 ? row[j - 1] >> 31 : 0u) | (wj << 1));
    if (b == 31) v = (v & 3u) | ((j + 1 < wpr ? row[j + 1] & 1u : 0u) << 2);
    return v & 7u;
  };

  // output tile -> uint8 layer at `layer` (+ U/B/X counts when cnt3); layer rows outside
  // [row_lo, row_hi) skipped, rows shifted by dst_shift (peer layers)
  auto store_tile = [&](const uint32_t* Bs, uint8_t* __restrict__ layer, int* cnt3, int row_lo, int row_hi,
                        int dst_shift, const uint32_t* Bprev = nullptr, int* newly_out = nullptr) {
    for (WordIter it(twords, (tr1 - tr0) * twords); it.ok(); it.next()) {
      const int rr = tr0 + it.r, j = tj0 + it.j;
      const int lrow = R0 + rr;
      if (lrow < row_lo || lrow >= row_hi) continue;
      const uint32_t bb = Bs[ro(rr + 1) + j], xx = X[ro(rr) + j];
      const int nc = min(32, RW - 32 * j);
      if (cnt3) {
        cnt3[0] += nc - __popc(bb) - __popc(xx);
        cnt3[1] += __popc(bb);
        cnt3[2] += __popc(xx);
        // ignited in the last step: burning now, not burning before it (Burning never re-ignites)
        if (Bprev) *newly_out += __popc(bb & ~Bprev[ro(rr + 1) + j]);
      }
      uint8_t* dst = layer + static_cast<size_t>(lrow + dst_shift) * W + C0 + 32 * j;
      if (nc == 32 && vec) bits_to_bytes(bb, xx, dst);
      else
        for (int k = 0; k < nc; ++k) dst[k] = static_cast<uint8_t>(((bb >> k) & 1u) | (((xx >> k) & 1u) << 1));
    }
  };

  int cur = 0;
  int newly = 0;
  const bool has_sched = a.sched_len > 1, rec_traj = a.traj != nullptr;
#if EBL_PHASE_PROF
  // per warp (lane 0): dense-pass cycles, decide-pass cycles, passes, cells; CTA: step cycles
  long long pw_dense = 0, pw_dec = 0, pw_pass = 0, pw_cells = 0, pw_t0 = 0, p_step = 0, p_wait = 0;
  long long pw_loc = 0, pw_body = 0, pw_ts = 0, pw_lat = 0;
  __shared__ long long s_wd[4][7];
#endif
#if EBL_WARP_UNROLL2
#pragma unroll 2
#endif
  for (int t = 0; t < n_run; ++t) {
#if EBL_PHASE_PROF
    const long long st0 = clock64();
    pw_t0 = st0;
#endif
    const uint32_t* B = cur ? Bp1 : Bp0;
    uint32_t* Bn = cur ? Bp0 : Bp1;
#if EBL_WARP_MICRO
    int srow = 0;
    if (has_sched) {  // CTA-uniform: time-varying wind
      srow = sched_row(a, a.step + static_cast<uint64_t>(t));
      if (t > 0) {
        load_wind(srow);
        __syncthreads();
      }
    }
#else
    const int srow = a.sched_len > 1 ? sched_row(a, a.step + static_cast<uint64_t>(t)) : 0;
    if (t > 0 && a.sched_len > 1) {  // CTA-uniform: time-varying wind
      load_wind(srow);
      __syncthreads();
    }
#endif
    const uint64_t prefix = s_prefix[t & 127];
    [[maybe_unused]] const bool last = t == n_steps - 1;
    [[maybe_unused]] uint32_t rowb = 0u;  // (EXIT) a burning cell in this thread's rows at step start
    for (int rb = 0; rb < H; rb += kWpThreads) {
      // ---- dense pass over the lane's row ------------------------------------------------------
      const int r = rb + 4 * lane + warp;
      int cnt = 0;
      uint32_t cum = 0xffffffffu;  // (WPRC <= 4) exclusive per-word counts of the row, a byte each
      if (r < H) {
        const uint32_t* up = B + ro(r + 2);
        const uint32_t* mid = B + ro(r + 1);
        const uint32_t* dn = B + ro(r);
        uint32_t* bn = Bn + ro(r + 1);
        const uint32_t* xr = X + ro(r);
        uint32_t* ar = ACT + ro(r);
        uint32_t vl = 0u;
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
          const uint32_t any = ((vc << 1) | (vl >> 31)) | ((vc >> 1) | (vn << 31)) | uc | dc;
          bn[j] = mc;
          const uint32_t valid = j + 1 < wpr ? 0xffffffffu : last_mask;
          const uint32_t act = ((~(mc | xr[j]) & valid) & any) | mc;
          ar[j] = act;
          if constexpr (EXIT) rowb |= mc;
          if (WPRC != 0 && WPRC <= 4 && j + 1 < 4)
            cum = (cum & ~(0xffu << (8 * (j + 1)))) | (static_cast<uint32_t>(cnt + __popc(act)) << (8 * (j + 1)));
          cnt += __popc(act);
          vl = vc;
          vc = vn;
          uc = un;
          mc = mn;
          dc = dnn;
        }
      }
#if EBL_PHASE_PROF
      if (lane == 0) {
        const long long c = clock64();
        pw_dense += c - pw_t0;
        pw_t0 = c;
      }
#endif
      if (!__ballot_sync(0xffffffffu, cnt > 0)) continue;  // quiet rows of this warp
      __syncwarp();  // ACT / Bn rows of the warp visible to all its lanes
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int excl = incl - cnt;
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      // ---- this warp's active cells, 32 per pass ----------------------------------------------------
#if EBL_PHASE_PROF
      if (lane == 0) {
        pw_pass += (total + 31) / 32;
        pw_cells += total;
      }
#endif
      for (int p = 0; p < total; p += 32) {
#if EBL_PHASE_PROF
        __syncwarp();
        pw_ts = clock64();
#endif
        const int idx = p + lane;
        int L = 0;  // the last lane whose exclusive count is <= idx (counts are non-decreasing)
#pragma unroll
        for (int st = 16; st > 0; st >>= 1) {
          const int cand = L + st;
          const int v = __shfl_sync(0xffffffffu, excl, cand & 31);
          if (cand < 32 && v <= idx) L = cand;
        }
        int q = idx - __shfl_sync(0xffffffffu, excl, L);
        const uint32_t cumL = __shfl_sync(0xffffffffu, cum, L);
        if (idx >= total) continue;
        const int rr = rb + 4 * L + warp;
        const uint32_t* ar = ACT + ro(rr);
        int jj = 0;
        uint32_t wv;
        if (WPRC != 0 && WPRC <= 4) {  // the word from the packed exclusive counts: no search loop
          const uint32_t qq = static_cast<uint32_t>(q);
          jj = (qq >= ((cumL >> 8) & 0xffu)) + (qq >= ((cumL >> 16) & 0xffu)) + (qq >= (cumL >> 24));
          q -= jj ? static_cast<int>((cumL >> (8 * jj)) & 0xffu) : 0;
          wv = ar[jj];
        } else {
          wv = ar[0];
          for (;;) {  // the word holding the q-th active cell of row rr
            const int pc = __popc(wv);
            if (q < pc) break;
            q -= pc;
            wv = ar[++jj];
          }
        }
        int cc;
        if constexpr (kFast) cc = 32 * jj + nth_set_bit_lut(wv, q, kNthBitLut);
        else cc = 32 * jj + nth_set_bit(wv, q);
#if EBL_PHASE_PROF
        {
          const unsigned msk = __activemask();
          const int ccs = __shfl_sync(msk, cc, __ffs(msk) - 1);  // the warp's lanes have located
          __syncwarp(msk);
          if (lane == 0) pw_loc += clock64() - pw_ts + (ccs & 0);
          pw_ts = clock64();
        }
#endif
        const int gr = R0 + rr, gc = C0 + cc;  // layer coordinates
        if (kFast && use_tab) {
          // one code path for burning and candidate cells (no divergence inside the pass): the
          // record is requested first, the neighbour windows are branch-free (zero guard and
          // padding words), a burning cell takes the candidate arithmetic with an empty mask
          const float4* tp = reinterpret_cast<const float4*>(a.pot32t + static_cast<size_t>(env) * a.pot32t_stride) +
                             2 * (gr * W + gc);
          const float4 T0 = __ldg(tp), T1 = __ldg(tp + 1);
          const int j = cc >> 5, b = cc & 31;
          const uint32_t bit = 1u << b;
          const int wi = ro(rr + 1) + j;
          const uint64_t m = cell_bits53(prefix, gbase + static_cast<uint64_t>(rr) * W + cc, 0);
          auto win = [&](const uint32_t* row) -> uint32_t {  // columns c-1, c, c+1 -> bits 0..2
            const uint32_t lo = row[j - 1], md = row[j], hi = row[j + 1];
            return (b > 0 ? __funnelshift_r(md, hi, b - 1) : __funnelshift_r(lo, md, 31)) & 7u;
          };
          const uint32_t midw = win(B + ro(rr + 1)), dnw = win(B + ro(rr)), upw = win(B + ro(rr + 2));
          const bool burning = midw & 2u;
          const uint32_t nb = burning ? 0u
                                      : (midw & 1u) | (dnw << 1) | ((midw >> 2) << 4) | ((upw >> 2) << 5) |
                                            ((upw & 2u) << 5) | ((upw & 1u) << 7);
          const bool ig = ignite_pot_fast(a, env, srow, T0, T1, W, gr, gc, nb, m, dg);
          if (burning && m >= a.pc_thr) {  // burns out: u >= p_continue, integer form
            atomicAnd(Bn + wi, ~bit);
            atomicOr(X + ro(rr) + j, bit);
          }
          if (ig) atomicOr(Bn + wi, bit);
          continue;
        }
        // the candidate records are requested first (burning cells waste one), so their latency
        // overlaps the RNG rounds and the neighbour masks below
        CellRec rec{};
        if (use_tab) {  // the candidate's 8 terms of gamma * lambda (pot32t)
          const float4* tp = reinterpret_cast<const float4*>(a.pot32t + static_cast<size_t>(env) * a.pot32t_stride) +
                             2 * (gr * W + gc);
          rec.s0 = __ldg(tp);
          rec.s1 = __ldg(tp + 1);
#if EBL_PHASE_PROF
          if (lane == 0) {  // issue -> data ready of lane 0's record (the asm waits on the registers)
            long long c1;
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(c1) : "f"(rec.s0.x), "f"(rec.s1.w));
            pw_lat += c1 - pw_ts;
          }
#endif
        } else if (use_rec) {
          rec = load_rec(a.slope32 + static_cast<size_t>(env) * a.ter_stride * 8,
                         a.nfuel + static_cast<size_t>(env) * a.ter_stride, a.fuel + static_cast<size_t>(env) * a.ter_stride,
                         gr * W + gc);
        }
        // ---- decide (engine.cpp:12-26) ----
        const int j = cc >> 5, b = cc & 31;
        const uint32_t bit = 1u << b;
        const int wi = ro(rr + 1) + j;
        const uint64_t m = cell_bits53(prefix, gbase + static_cast<uint64_t>(rr) * W + cc, 0);
        const uint32_t midw = win3(B + ro(rr + 1), j, b);
        if (midw & 2u) {  // Burning: u < p_continue, integer form
          if (m >= a.pc_thr) {
            atomicAnd(Bn + wi, ~bit);
            atomicOr(X + ro(rr) + j, bit);
          }
        } else {  // Unburned with a burning neighbour
          const uint32_t dnw = win3(B + ro(rr), j, b), upw = win3(B + ro(rr + 2), j, b);
          const uint32_t nb = (midw & 1u) | (dnw << 1) | ((midw >> 2) << 4) | ((upw >> 2) << 5) |
                              ((upw & 2u) << 5) | ((upw & 1u) << 7);
          bool ig;
          if (use_tab)
            ig = ignite_pot(a, env, srow, rec.s0, rec.s1, W, gr, gc, nb, m, dg);
          else if (use_rec)
            ig = ignite_terrain_rec_pre(terrain_view(a, env, srow), rec, s_srckw, s_pal + 256, a.alpha_s_l2, W, gr, gc,
                                        nb, m, dg);
          else if constexpr (kTer)
            ig = ignite_terrain_tab(terrain_view(a, env, srow), a.slope32 + static_cast<size_t>(env) * a.ter_stride * 8,
                                    s_pal, s_kw, W, BH, gr, gc, nb, m, dg);
          else
            ig = ignite<MODE>(a, env, gr, gc, nb, m, dg, srow);
#if EBL_PHASE_PROF
          if (lane == 0) pw_body += clock64() - pw_ts + (ig & 0);
#endif
          if (ig) {
            atomicOr(Bn + wi, bit);
#if !EBL_WARP_MICRO
            newly += last && rr >= tr0 && rr < tr1 && cc >= tc0 && cc < tc1;  // counted in the tile only
#endif
          }
        }
      }
    }
    if (((t & 63) == 63) && t + 1 < n_steps) {  // refill the prefix ring with steps t+1 .. t+64
      for (int k = threadIdx.x; k < 64; k += blockDim.x)
        s_prefix[(t + 1 + k) & 127] = key_prefix(a.seed, stream, a.step + static_cast<uint64_t>(t + 1 + k));
    }
#if EBL_PHASE_PROF
    __syncwarp();
    if (lane == 0) {
      const long long c = clock64();
      pw_dec += c - pw_t0;
      pw_t0 = c;
    }
#endif
    if constexpr (EXIT) {
      // Bn / X complete: the next step reads them.  A step that started without a burning cell
      // changed nothing, and neither can any later one: the remaining steps are skipped (the
      // trajectory-recording form stores every step)
      if (!__syncthreads_or(rowb != 0u || rec_traj)) {
        cur ^= 1;
        break;
      }
    } else {
      __syncthreads();  // Bn / X complete: the next step reads them
    }
#if EBL_PHASE_PROF
    if (lane == 0) p_wait += clock64() - pw_t0;
    if (threadIdx.x == 0) p_step += clock64() - st0;
#endif
    cur ^= 1;
    if (rec_traj) {  // record (run_stochastic(record=true), engine.cpp:116): the tile after this step
      const uint32_t* Bs = cur ? Bp1 : Bp0;
      store_tile(Bs, a.traj + ((a.traj_t0 + t) * a.n_envs + env) * ncell, nullptr, 0, BH, 0);
    }
  }

#if EBL_PHASE_PROF
  if (a.prof) {
    if (lane == 0) {
      s_wd[warp][0] = pw_dense;
      s_wd[warp][1] = pw_dec;
      s_wd[warp][2] = pw_pass;
      s_wd[warp][3] = pw_wait_dummy(p_wait);
      s_wd[warp][4] = pw_loc;
      s_wd[warp][5] = pw_body;
      s_wd[warp][6] = pw_lat;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      long long mx[7] = {0, 0, 0, 0, 0, 0, 0}, passes = 0;
      for (int q = 0; q < 4; ++q) {
        for (int k = 0; k < 7; ++k) mx[k] = max(mx[k], s_wd[q][k]);
        passes += s_wd[q][2];
      }
      long long* o = a.prof + static_cast<size_t>(env) * 10;
      o[0] = mx[0];      // slowest warp: dense-pass cycles (sum over steps)
      o[1] = mx[1];      // slowest warp: decide cycles
      o[2] = pw_cells;   // warp 0's cells (for reference)
      o[3] = mx[6];      // max warp: lane 0's record load latency (issue -> data ready)
      o[4] = mx[2];      // max passes of a warp (sum over steps)
      o[5] = passes;     // passes of all warps
      o[6] = p_step;     // CTA step cycles (thread 0)
      o[7] = mx[3];      // max barrier wait
      o[8] = mx[4];      // max warp: locate cycles (pass start -> cell found)
      o[9] = mx[5];      // max warp: lane 0's decide body (cell found -> ignition decided)
    }
  }
#endif
  // ---- store + counts ----------------------------------------------------------------------------
  const uint32_t* Bs = cur ? Bp1 : Bp0;
  int c3[3] = {0, 0, 0};
#if EBL_WARP_MICRO
  store_tile(Bs, a.out + env * ncell, c3, a.store_lo, a.store_hi, 0, n_run > 0 ? (cur ? Bp0 : Bp1) : nullptr,
             &newly);
#else
  store_tile(Bs, a.out + env * ncell, c3, a.store_lo, a.store_hi, 0);
#endif
  if (a.out2) store_tile(Bs, a.out2 + env * ncell, nullptr, a.store_lo, a.store_hi, 0);
  for (int p = 0; p < a.n_peers; ++p)  // fused halo exchange: owned rows straight into the neighbour
    store_tile(Bs, a.peer_out[p], nullptr, a.peer_lo[p], a.peer_hi[p], a.peer_dst[p] - a.peer_lo[p]);
  int cu = c3[0], cb = c3[1], cx = c3[2];
  if (!a.counts && !a.tflag_out && !a.list_mode) return;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cu += __shfl_xor_sync(0xffffffffu, cu, o);
    cb += __shfl_xor_sync(0xffffffffu, cb, o);
    cx += __shfl_xor_sync(0xffffffffu, cx, o);
    newly += __shfl_xor_sync(0xffffffffu, newly, o);
  }
  if (lane == 0) {
    atomicAdd(&s_cnt[0], cu);
    atomicAdd(&s_cnt[1], cb);
    atomicAdd(&s_cnt[2], cx);
    atomicAdd(&s_newly, newly);
  }
  __syncthreads();
  if (a.counts) {  // (work-list runs: U/B/X summed from the records after the call, k_tile_counts)
    if (threadIdx.x < 3 && !a.list_mode) atomicAdd(a.counts + env * 4 + threadIdx.x, s_cnt[threadIdx.x]);
    if (threadIdx.x == 3) atomicAdd(a.counts + env * 4 + 3, s_newly);
  }
  if (tf_out && threadIdx.x == 0) {
    const int streak = n_run == 0 ? (canon_quiet ? 2 : min(streak0 + 1, 2)) : 0;  // output == input this launch
    tf_out[tile_id] = make_int4((s_cnt[1] > 0 ? 1 : 0) | (streak << 1), s_cnt[0], s_cnt[1], s_cnt[2]);
  }
  if (a.list_mode && threadIdx.x == 0) {
    // record in place, then the next launch's work list: a tile with a burning cell makes its 3x3
    // neighbourhood run (the light cone of one launch stays within the neighbours), a tile whose
    // buffers are not both canonical yet (streak < 2) makes itself run -- exactly the tiles the
    // grid form's skip rule would not skip (tiles outside the list keep a quiet record)
    const int streak = n_run == 0 ? (canon_quiet ? 2 : min(streak0 + 1, 2)) : 0;
    const bool burning = s_cnt[1] > 0;
    reinterpret_cast<int4*>(a.trec)[tile_id] = make_int4((burning ? 1 : 0) | (streak << 1), s_cnt[0], s_cnt[1], s_cnt[2]);
    auto enqueue = [&](int tx, int ty) {
      const size_t id = (static_cast<size_t>(env) * nty + ty) * ntx + tx;
      if (atomicExch(a.queued + id, a.list_stamp) != a.list_stamp) a.next_list[atomicAdd(a.next_count, 1)] = static_cast<int>(id);
    };
    // (row shards without record exchange: a tile holding halo rows a neighbour writes runs in
    // every launch)
    const bool exposed_t = !a.halo_marked && (r0 < a.keep_lo || r0 + g.tile_h > a.keep_hi);
    if (burning) {
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx)
          if (byi + dy >= 0 && byi + dy < nty && bxi + dx >= 0 && bxi + dx < ntx) enqueue(bxi + dx, byi + dy);
      // row shards: the records travel with the halo rows -- the neighbour's tiles whose regions
      // reach the rows stored into it run next launch (the light cone of a burning cell there);
      // a tile without a burning cell stores nothing that can change a neighbour's band
      for (int p = 0; p < a.n_peers; ++p) {
        if (!a.peer_queued[p]) continue;
        const int lo = max(r0, a.peer_lo[p]), hi = min(min(r0 + g.tile_h, BH), a.peer_hi[p]);
        if (lo >= hi) continue;
        const int qlo = lo + a.peer_dst[p] - a.peer_lo[p], qhi = hi + a.peer_dst[p] - a.peer_lo[p];
        const int th = a.peer_tile_h[p], tw = a.peer_tile_w[p], hr = a.peer_halo_r[p], hc = a.peer_halo_c[p];
        const int cl = c0, ch = min(c0 + g.tile_w, W);
        // tiles whose region [t*th - hr, (t+1)*th + hr) meets [qlo, qhi) (columns alike)
        const int ty0 = qlo - hr <= 0 ? 0 : (qlo - hr) / th, ty1 = min(a.peer_tiles_y[p] - 1, (qhi + hr + th - 1) / th - 1);
        const int tx0 = cl - hc <= 0 ? 0 : (cl - hc) / tw, tx1 = min(a.peer_tiles_x[p] - 1, (ch + hc + tw - 1) / tw - 1);
        for (int ty = ty0; ty <= ty1; ++ty)
          for (int tx = tx0; tx <= tx1; ++tx) {
            const int id = ty * a.peer_tiles_x[p] + tx;  // (shards hold one env)
            if (atomicExch_system(a.peer_queued[p] + id, a.peer_stamp[p]) != a.peer_stamp[p])
              a.peer_next_list[p][atomicAdd_system(a.peer_next_count[p], 1)] = id;
          }
      }
    } else if (streak < 2 || exposed_t) {
      enqueue(bxi, byi);
    }
  }
}

template <int MODE, int WPRC, int DIMC, bool EXIT = false>
__global__ void __launch_bounds__(kWpThreads, EBL_WARP_MINB) k_step_warp(StepArgs a, BlockGeom g) {
  if (DIMC == 0 && a.list_mode == 2) pdl_enter();  // work-list launches follow one another (PDL)
  if (DIMC == 0 && a.list_mode && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0) {
    *a.list_zero0 = 0;  // the next launch's append counter and cursor start at 0 (no memset launches)
    *a.list_zero1 = 0;
  }
  if (DIMC == 0 && a.list_mode == 2) {  // work list of this launch: persistent CTAs take tiles until it runs out
    __shared__ int s_item;
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.diag) atomicAdd(a.diag + 3, static_cast<unsigned long long>(a.tiles_total));
    for (;;) {
      __syncthreads();  // the previous region's shared state is consumed
      if (threadIdx.x == 0) s_item = atomicAdd(a.list_cursor, 1);
      __syncthreads();
      const int item = s_item;
      if (item >= *a.tile_count) break;
      const int tile = a.tile_list[item];
      const int bx = tile % a.tiles_x, rest = tile / a.tiles_x;
      warp_region<MODE, WPRC, DIMC>(a, g, rest / a.tiles_y, bx, rest % a.tiles_y, a.tiles_x, a.tiles_y);
    }
  } else {
    // (whole-env instantiations: one region per env, the tile coordinates are compile-time 0 / 1)
    warp_region<MODE, WPRC, DIMC, EXIT>(a, g, static_cast<int>(blockIdx.z), DIMC ? 0 : static_cast<int>(blockIdx.x),
                                        DIMC ? 0 : static_cast<int>(blockIdx.y), DIMC ? 1 : static_cast<int>(gridDim.x),
                                        DIMC ? 1 : static_cast<int>(gridDim.y));
  }
}

// Work-list launch of several row shards on one device: the persistent CTAs claim items of the
// concatenated lists (shard 0's cursor), item -> (shard, tile) by the list counts' prefix.  Each
// region runs with its shard's StepArgs, read in place from the kernel parameter block.
template <int MODE, int WPRC>
__global__ void __launch_bounds__(kWpThreads, EBL_WARP_MINB) k_step_warp_shards(const __grid_constant__ ShardsLaunch P) {
  pdl_enter();
  __shared__ int s_pref[kMaxShardLaunch + 1];
  __shared__ int s_item;
  if (blockIdx.x == 0 && threadIdx.x < P.n) {
    *P.sa[threadIdx.x].list_zero0 = 0;
    *P.sa[threadIdx.x].list_zero1 = 0;
    if (P.sa[threadIdx.x].diag && !P.all_tiles)  // (list_mode 1 regions count themselves)
      atomicAdd(P.sa[threadIdx.x].diag + 3, static_cast<unsigned long long>(P.sa[threadIdx.x].tiles_total));
  }
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int s = 0; s < P.n; ++s) {
      s_pref[s] = acc;
      acc += P.all_tiles ? P.sa[s].tiles_total : *P.sa[s].tile_count;
    }
    s_pref[P.n] = acc;
  }
  for (;;) {
    __syncthreads();  // the previous region's shared state is consumed (and s_pref written)
    if (threadIdx.x == 0) s_item = atomicAdd(P.sa[0].list_cursor, 1);
    __syncthreads();
    const int item = s_item;
    if (item >= s_pref[P.n]) break;
    int sh = 0;
    while (item >= s_pref[sh + 1]) ++sh;
    const StepArgs& a = P.sa[sh];
    const int tile = P.all_tiles ? item - s_pref[sh] : a.tile_list[item - s_pref[sh]];
    const int bx = tile % a.tiles_x, rest = tile / a.tiles_x;
    warp_region<MODE, WPRC, 0>(a, P.g[sh], rest / a.tiles_y, bx, rest % a.tiles_y, a.tiles_x, a.tiles_y);
  }
}

template <int MODE, int WPRC>
cudaError_t launch_wp_shards(const ShardsLaunch& P, size_t sm, cudaStream_t s) {
  const void* kern = reinterpret_cast<const void*>(k_step_warp_shards<MODE, WPRC>);
  cudaError_t e = smem_opt_in(kern, sm);
  if (e != cudaSuccess) return e;
  int wave = 0;
  e = resident_ctas(kern, kWpThreads, sm, &wave);
  if (e != cudaSuccess) return e;
  int tiles = 0;
  for (int i = 0; i < P.n; ++i) tiles += P.sa[i].tiles_total;
  return launch_pdl(k_step_warp_shards<MODE, WPRC>, dim3(std::max(1, std::min(tiles, wave))), dim3(kWpThreads), sm, s, P);
}

template <int MODE, int WPRC, int DIMC = 0, bool EXIT = false>
cudaError_t launch_wp(const StepArgs& a, const BlockGeom& g, size_t sm, cudaStream_t s) {
  const void* kern = reinterpret_cast<const void*>(k_step_warp<MODE, WPRC, DIMC, EXIT>);
  cudaError_t e = smem_opt_in(kern, sm);
  if (e != cudaSuccess) return e;
  if (a.list_mode == 2) {  // persistent: one wave of CTAs over the work list
    int wave = 0;
    e = resident_ctas(kern, kWpThreads, sm, &wave);
    if (e != cudaSuccess) return e;
    const int ctas = std::max(1, std::min(a.tiles_total, wave));
    return launch_pdl(k_step_warp<MODE, WPRC, DIMC, EXIT>, dim3(ctas), dim3(kWpThreads), sm, s, a, g);
  }
  const dim3 grid((a.w + g.tile_w - 1) / g.tile_w, (a.h + g.tile_h - 1) / g.tile_h, a.n_envs);
  k_step_warp<MODE, WPRC, DIMC, EXIT><<<grid, kWpThreads, sm, s>>>(a, g);
  return cudaGetLastError();
}

}  // namespace

// counts[env][0..2] += the U/B/X of every tile's record (work-list runs: tiles not in the last
// list kept their recorded counts; the listed tiles of the last launch add only counts[env][3]);
// blockIdx.y = env, blockIdx.x strides over its tiles
__global__ void k_tile_counts(const int4* __restrict__ trec, int tiles_per_env, int32_t* counts) {
  __shared__ int s[3];
  if (threadIdx.x < 3) s[threadIdx.x] = 0;
  __syncthreads();
  int u = 0, bb = 0, x = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < tiles_per_env; i += gridDim.x * blockDim.x) {
    const int4 r = trec[static_cast<size_t>(blockIdx.y) * tiles_per_env + i];
    u += r.y;
    bb += r.z;
    x += r.w;
  }
  atomicAdd(&s[0], u);
  atomicAdd(&s[1], bb);
  atomicAdd(&s[2], x);
  __syncthreads();
  if (threadIdx.x < 3) atomicAdd(counts + blockIdx.y * 4 + threadIdx.x, s[threadIdx.x]);
}

// First step of a work-list run without a grid launch: one warp per tile copies the tile's bytes into
// the other layer buffer, counts U/B/X, and writes its record {burning, quiet streak, U, B, X} --
// streak 2 when every byte is a FireState (both buffers then hold the tile's canonical bytes),
// else 0 (the tile must run once: its store maps the other bytes to Unburned) -- and enqueues the
// first launch's tiles: a burning tile's 3x3 neighbourhood, a non-canonical tile itself.  A tile
// no launch lists keeps these bytes, which is what stepping a region without fire produces.
__global__ void k_tile_init(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int h, int w, size_t ncell,
                            int tile_h, int tile_w, int ntx, int nty, int4* trec, int32_t* queued, int32_t stamp,
                            int32_t* next_list, int32_t* next_count, int count_lo, int count_hi) {
  // one warp per tile (kInitTiles tiles per CTA along x, no block barriers): the lanes stream the
  // tile's rows as 16-byte words, counts and flags by warp reductions
  const int lane = threadIdx.x & 31;
  const int tx = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), ty = blockIdx.y, env = blockIdx.z;
  if (tx >= ntx) return;
  const int r0 = ty * tile_h, c0 = tx * tile_w;
  const int rows = min(tile_h, h - r0), cols = min(tile_w, w - c0);
  int u = 0, bb = 0, x = 0, nc = 0, burn_any = 0;
  const uint8_t* src = in + env * ncell;
  uint8_t* dst = out + env * ncell;
  const bool vec = (w % 16) == 0 && (cols % 16) == 0;
  const int per_row = vec ? cols / 16 : cols;
#pragma unroll 4
  for (int i = lane; i < rows * per_row; i += 32) {
    const int r = r0 + i / per_row, k = i % per_row;
    const bool counted = r >= count_lo && r < count_hi;  // (row shards: the band rows only)
    if (vec) {
      const size_t o = static_cast<size_t>(r) * w + c0 + 16 * k;
      const uint4 q = *reinterpret_cast<const uint4*>(src + o);
      *reinterpret_cast<uint4*>(dst + o) = q;
      const uint32_t wd[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t v = wd[j];
        const uint32_t z = v & 0xFCFCFCFCu;
        const uint32_t small = ~((((z & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | z) >> 7) & 0x01010101u;
        const uint32_t b0 = v & 0x01010101u, b1 = (v >> 1) & 0x01010101u;
        const int n1 = __popc(b0 & ~b1 & small), n2 = __popc(b1 & ~b0 & small);
        if (counted) {
          bb += n1;
          x += n2;
          u += 4 - n1 - n2;  // (non-FireState bytes count as Unburned, as a step maps them)
        }
        burn_any |= n1;
        nc |= static_cast<int>((~small & 0x01010101u) | (b0 & b1));
      }
    } else {
      const size_t o = static_cast<size_t>(r) * w + c0 + k;
      const uint8_t v = src[o];
      dst[o] = v;
      if (counted) {
        bb += v == 1;
        x += v == 2;
        u += v != 1 && v != 2;
      }
      burn_any |= v == 1;
      nc |= v > 2;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    u += __shfl_xor_sync(0xffffffffu, u, o);
    bb += __shfl_xor_sync(0xffffffffu, bb, o);
    x += __shfl_xor_sync(0xffffffffu, x, o);
  }
  const bool burning = __any_sync(0xffffffffu, burn_any != 0);  // (a burning halo row counts for the lists)
  const bool canon = !__any_sync(0xffffffffu, nc != 0);
  if (lane != 0) return;
  const size_t id = (static_cast<size_t>(env) * nty + ty) * ntx + tx;
  trec[id] = make_int4((burning ? 1 : 0) | ((canon ? 2 : 0) << 1), u, bb, x);
  if (!next_list) return;  // grid-form records (carried across calls): no work list
  auto enqueue = [&](int qx, int qy) {
    const size_t q = (static_cast<size_t>(env) * nty + qy) * ntx + qx;
    if (atomicExch(queued + q, stamp) != stamp) next_list[atomicAdd(next_count, 1)] = static_cast<int>(q);
  };
  if (burning) {
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx)
        if (ty + dy >= 0 && ty + dy < nty && tx + dx >= 0 && tx + dx < ntx) enqueue(tx + dx, ty + dy);
  } else if (!canon) {
    enqueue(tx, ty);
  }
}

#ifndef EBL_INIT_TILES
#define EBL_INIT_TILES 4  // tiles (warps) per k_tile_init CTA
#endif
cudaError_t launch_tile_init(const uint8_t* in, uint8_t* out, int h, int w, int n_envs, int tile_h, int tile_w,
                             int32_t* trec, int32_t* queued, int32_t stamp, int32_t* next_list, int32_t* next_count,
                             int count_lo, int count_hi, cudaStream_t s) {
  const int ntx = (w + tile_w - 1) / tile_w, nty = (h + tile_h - 1) / tile_h;
  k_tile_init<<<dim3((ntx + EBL_INIT_TILES - 1) / EBL_INIT_TILES, nty, n_envs), 32 * EBL_INIT_TILES, 0, s>>>(
      in, out, h, w, static_cast<size_t>(h) * w, tile_h, tile_w, ntx, nty, reinterpret_cast<int4*>(trec), queued, stamp,
      next_list, next_count, count_lo, count_hi);
  return cudaGetLastError();
}

// Halo rows written into a row shard's layer between calls (ebl_batch_rows_device /
// ebl_batch_copy_rows): a burning cell sets the burning bit of its tile's carried record, so that
// tile and its 8 neighbours -- every tile whose region reaches the cell -- run next launch.
__global__ void k_mark_halo(const uint8_t* __restrict__ layer, int n_envs, size_t ncell, int w, int row0, int n_rows,
                            int4* tflags, int tile_h, int tile_w, int ntx, int nty) {
  const int chunks = (w + 15) / 16;
  const size_t total = static_cast<size_t>(n_envs) * n_rows * chunks;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int env = static_cast<int>(i / (static_cast<size_t>(n_rows) * chunks));
    const int rem = static_cast<int>(i - static_cast<size_t>(env) * n_rows * chunks);
    const int r = row0 + rem / chunks, c0 = 16 * (rem % chunks);
    const uint8_t* row = layer + env * ncell + static_cast<size_t>(r) * w;
    for (int c = c0; c < min(c0 + 16, w); ++c)
      if (row[c] == 1) {
        atomicOr(&tflags[(static_cast<size_t>(env) * nty + r / tile_h) * ntx + c / tile_w].x, 1);
        break;  // (a 16-byte chunk never straddles a tile column: tile_w is a multiple of 32)
      }
  }
}

cudaError_t launch_mark_halo(const uint8_t* layer, int n_envs, size_t ncell, int w, int row0, int n_rows,
                             int32_t* tflags, int tile_h, int tile_w, int ntx, int nty, cudaStream_t s) {
  if (n_rows <= 0) return cudaSuccess;
  const size_t total = static_cast<size_t>(n_envs) * n_rows * ((w + 15) / 16);
  const unsigned blocks = static_cast<unsigned>(std::min<size_t>((total + 255) / 256, 148 * 8));
  k_mark_halo<<<blocks, 256, 0, s>>>(layer, n_envs, ncell, w, row0, n_rows, reinterpret_cast<int4*>(tflags), tile_h,
                                     tile_w, ntx, nty);
  return cudaGetLastError();
}

cudaError_t launch_tile_counts(const int32_t* trec, int n_envs, int tiles_per_env, int32_t* counts, cudaStream_t s) {
  const int bx = std::max(1, std::min(64, (tiles_per_env + 255) / 256));
  k_tile_counts<<<dim3(bx, n_envs), 256, 0, s>>>(reinterpret_cast<const int4*>(trec), tiles_per_env, counts);
  return cudaGetLastError();
}

namespace {
struct LaunchKey {
  const void* f;
  int dev;
  size_t smem;
  int threads;
  bool operator==(const LaunchKey& o) const { return f == o.f && dev == o.dev && smem == o.smem && threads == o.threads; }
};
struct LaunchKeyHash {
  size_t operator()(const LaunchKey& k) const {
    return std::hash<const void*>()(k.f) ^ (static_cast<size_t>(k.dev) << 48) ^ (k.smem * 0x9E3779B97F4A7C15ull) ^
           static_cast<size_t>(k.threads);
  }
};
std::mutex g_launch_mu;
std::unordered_map<LaunchKey, int, LaunchKeyHash> g_smem_set;   // (f, dev) -> largest size opted in
std::unordered_map<LaunchKey, int, LaunchKeyHash> g_wave;       // (f, dev, smem, threads) -> CTAs per GPU
}  // namespace

cudaError_t smem_opt_in(const void* kernel, size_t smem) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_launch_mu);
  int& have = g_smem_set[LaunchKey{kernel, dev, 0, 0}];
  if (static_cast<size_t>(have) >= smem) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e == cudaSuccess) have = static_cast<int>(smem);
  return e;
}

cudaError_t resident_ctas(const void* kernel, int threads, size_t smem, int* ctas_per_gpu) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_launch_mu);
  const LaunchKey key{kernel, dev, smem, threads};
  auto it = g_wave.find(key);
  if (it == g_wave.end()) {
    int per_sm = 0, sms = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    it = g_wave.emplace(key, std::max(1, per_sm) * sms).first;
  }
  *ctas_per_gpu = it->second;
  return cudaSuccess;
}

size_t warp_smem_bytes(int h, int w) {
  const size_t S = plane_stride((w + 31) / 32);
  const size_t R = static_cast<size_t>(h) + 2;
  return 4 * (R * S + (R >> 2) + 1) * sizeof(uint32_t) + 16;  // B x2, X, ACT (ro() layout) + guard words
}

bool warp_fits(int h, int w) {
  return static_cast<size_t>(h) * w <= 65536 && warp_smem_bytes(h, w) <= kResMaxSmem;
}

// Any geometry plan_blocks produces with one env per CTA (whole env, or halo tiles).
cudaError_t launch_step_warp_shards(const ShardsLaunch& P, int mode, cudaStream_t s) {
  size_t sm = 0;
  bool whole_width = true;
  for (int i = 0; i < P.n; ++i) {
    const StepArgs& a = P.sa[i];
    const BlockGeom& g = P.g[i];
    const int rh = a.h < g.tile_h + 2 * g.halo_rows ? a.h : g.tile_h + 2 * g.halo_rows;
    const int rw = a.w < g.tile_w + 2 * g.halo_cols ? a.w : g.tile_w + 2 * g.halo_cols;
    sm = std::max(sm, warp_smem_bytes(rh, rw));
    whole_width = whole_width && g.tile_w >= a.w;
  }
  const int wpr = (P.sa[0].w + 31) / 32;
  const int frw = P.g[0].tile_w + 2 * P.g[0].halo_cols;
  bool fixed = mode == kStaticTerrain;
  for (int i = 0; i < P.n; ++i) fixed = fixed && P.g[i].fixed_region && P.g[i].tile_w + 2 * P.g[i].halo_cols == frw;
  if (fixed && frw == 320) return launch_wp_shards<kStaticTerrain, 10>(P, sm, s);
  if (fixed && frw == 192) return launch_wp_shards<kStaticTerrain, 6>(P, sm, s);
  if (fixed && frw == 128) return launch_wp_shards<kStaticTerrain, 4>(P, sm, s);
  if (mode == kStaticTables) {
    if (whole_width && wpr == 4) return launch_wp_shards<kStaticTables, 4>(P, sm, s);
    if (whole_width && wpr == 2) return launch_wp_shards<kStaticTables, 2>(P, sm, s);
    return launch_wp_shards<kStaticTables, 0>(P, sm, s);
  }
  if (whole_width && wpr == 4) return launch_wp_shards<kStaticTerrain, 4>(P, sm, s);
  if (whole_width && wpr == 2) return launch_wp_shards<kStaticTerrain, 2>(P, sm, s);
  return launch_wp_shards<kStaticTerrain, 0>(P, sm, s);
}

cudaError_t launch_step_warp(const StepArgs& a, int mode, const BlockGeom& g, cudaStream_t s) {
  const int rh = a.h < g.tile_h + 2 * g.halo_rows ? a.h : g.tile_h + 2 * g.halo_rows;
  const int rw = a.w < g.tile_w + 2 * g.halo_cols ? a.w : g.tile_w + 2 * g.halo_cols;
  const size_t sm = warp_smem_bytes(rh, rw);
  const bool whole_width = g.tile_w >= a.w, whole = whole_width && g.tile_h >= a.h;
  const int wpr = (a.w + 31) / 32;
  if (mode == kStaticTables) {
    if (whole_width && wpr == 4) return launch_wp<kStaticTables, 4>(a, g, sm, s);
    if (whole_width && wpr == 2) return launch_wp<kStaticTables, 2>(a, g, sm, s);
    return launch_wp<kStaticTables, 0>(a, g, sm, s);
  }
  // C1: the whole-env launch of ebl_step_batch leaves its step loop once the fire is out (EXIT)
  if (whole && a.h == 128 && a.w == 128)
    return a.early_exit ? launch_wp<kStaticTerrain, 4, 128, true>(a, g, sm, s) : launch_wp<kStaticTerrain, 4, 128>(a, g, sm, s);
  // fixed 128 / 192 / 320-column regions (64 / 128 / 256-column tiles with their halo): compile-time
  // words per row and the branch-free decide pass for every halo tile
  if (g.fixed_region && rw == 320) return launch_wp<kStaticTerrain, 10>(a, g, sm, s);
  if (g.fixed_region && rw == 192) return launch_wp<kStaticTerrain, 6>(a, g, sm, s);
  if (g.fixed_region && rw == 128) return launch_wp<kStaticTerrain, 4>(a, g, sm, s);
  if (whole && a.h == 64 && a.w == 64)
    return a.early_exit ? launch_wp<kStaticTerrain, 2, 64, true>(a, g, sm, s) : launch_wp<kStaticTerrain, 2, 64>(a, g, sm, s);
  if (whole_width && wpr == 4) return launch_wp<kStaticTerrain, 4>(a, g, sm, s);
  if (whole_width && wpr == 2) return launch_wp<kStaticTerrain, 2>(a, g, sm, s);
  return launch_wp<kStaticTerrain, 0>(a, g, sm, s);
}

}  // namespace ebl
