// Device-side core of the stochastic CA step: the reference's counter RNG
// (rng.hpp:28-58) reproduced bit-exactly, and the per-cell transition
// (engine.cpp:12-26 next_fire_cell) evaluated as
//   * an exact integer test for Burning cells (u < p_continue  <=>  (w>>11) < ceil(p_continue*2^53)),
//   * a skip for Unburned cells with no burning neighbour (lambda = 0 => p = 0 => u < p is false,
//     so the draw the reference takes there cannot change the outcome; the RNG is counter-based,
//     so not drawing is invisible to every other cell),
//   * an fp32 fast path with a relative guard band for Unburned front cells, falling back to
//     an fp64 evaluation in the reference's exact association (kernel.hpp:21-78,
//     engine.hpp:79-143) only when the draw lies inside the band.
#pragma once
#include <cstdint>

#include "ember_params.h"

namespace ebl {

// grid.hpp:74-83, (dx east, dy north), k = 0..7 : E NE N NW W SW S SE
__device__ __constant__ const int8_t kDx[8] = {1, 1, 0, -1, -1, -1, 0, 1};
__device__ __constant__ const int8_t kDy[8] = {0, 1, 1, 1, 0, -1, -1, -1};

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

// First three rounds of rng_word (seed -> stream -> step), constant per (env, step).
__device__ __forceinline__ uint64_t key_prefix(uint64_t seed, uint64_t stream, uint64_t step) {
  return mix64(mix64(mix64(0x243F6A8885A308D3ull ^ seed) ^ stream) ^ step);
}

// Remaining two rounds (cell, draw); >> 11 gives the 53-bit mantissa m, u = m * 2^-53.
__device__ __forceinline__ uint64_t cell_bits53(uint64_t prefix, uint64_t cell, uint64_t draw) {
  return mix64(mix64(prefix ^ cell) ^ draw) >> 11;
}

__device__ __forceinline__ double bits_to_uniform(uint64_t m) {
  return static_cast<double>(m) * 0x1.0p-53;  // exact
}

// rng_below (rng.hpp:54-58): truncating conversion of u*n, clamped.
__device__ __forceinline__ uint64_t below(uint64_t m, uint64_t n) {
  const double x = __dmul_rn(bits_to_uniform(m), static_cast<double>(n));
  const uint64_t v = __double2ull_rz(x);
  return v < n ? v : n - 1;
}

struct DiagCounters {
  unsigned long long* g;  // [0] fp64 fallbacks, [1] ambiguous draws
  __device__ __forceinline__ void fallback() const { atomicAdd(g + 0, 1ull); }
  __device__ __forceinline__ void ambiguous() const { atomicAdd(g + 1, 1ull); }
};

// |u - p| below this (absolute) is reported as "ambiguous": the device libm
// (exp/atan) may differ from glibc by an ulp there, so a flip vs the CPU is
// possible only for these draws.
constexpr double kAmbiguousBand = 1e-12;

// ---- general form: SpreadTables<double> resident in HBM --------------------------
// lambda fold in k order, skipping zero weights, then p = 1 - exp(-(gamma*lambda))
// (engine.hpp:130-143, engine.cpp:21-25), all fp64 with explicit round-to-nearest ops.
__device__ __forceinline__ bool ignite_tables(const double* __restrict__ pot,
                                              const double* __restrict__ gamma, int w, int r,
                                              int c, uint32_t nb, uint64_t m,
                                              const DiagCounters& dg) {
  double lam = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (nb & (1u << k)) {
      const int u = (r - kDy[k]) * w + (c - kDx[k]);
      lam = __dadd_rn(lam, __ldg(pot + static_cast<size_t>(u) * 8 + k));
    }
  }
  const double p = __dsub_rn(1.0, exp(-__dmul_rn(__ldg(gamma + r * w + c), lam)));
  const double u = bits_to_uniform(m);
  if (fabs(u - p) < kAmbiguousBand) dg.ambiguous();
  return u < p;
}

// ---- terrain form: uint8 fuel class + fp32 elevation -------------------------------
struct TerrainView {
  const uint8_t* __restrict__ fuel;  // env base applied
  const float* __restrict__ elev;
  const float* pal_src32;   // [256] (p_base*(1+veg))*(1+den)   (kernel.hpp:39-40)
  const float* pal_gam32;   // [256] (alpha_gamma*(1+veg))*(1+den) (kernel.hpp:75-76)
  const double* pal_src64;
  const double* pal_gam64;
  const float* kw32;        // [8] kappa_wind of this env (kernel.hpp:21-26)
  const double* kw64;
  float alpha_s32;
  double alpha_s;
  float inv_dist32[2];      // 1/cellsize, 1/(cellsize*sqrt2)
  double dist64[2];         // cellsize*1.0, cellsize*sqrt2 (geodata.cpp:222-223)
  int force64;              // parameters outside the fp32 guard's validity range
};

// fp64 re-evaluation in the reference's exact association:
//   S   = atan((z(v) - z(u)) / dist)                 geodata.cpp:222-224
//   pot = (source(u) * kappa_wind(k)) * exp(alpha_s*S)  engine.hpp:91,106-107
//   p   = 1 - exp(-(gamma(v) * lambda))               engine.cpp:24
static __device__ __noinline__ double terrain_p64(const TerrainView& t, int w, int r, int c, uint32_t nb) {
  const int v = r * w + c;
  const double zv = static_cast<double>(t.elev[v]);
  double lam = 0.0;
  for (int k = 0; k < 8; ++k) {
    if (nb & (1u << k)) {
      const int u = (r - kDy[k]) * w + (c - kDx[k]);
      const double dz = __dsub_rn(zv, static_cast<double>(t.elev[u]));
      // DEM nodata (NaN) on either end: slope 0 (geodata.cpp:214,220)
      const double s = dz == dz ? atan(__ddiv_rn(dz, t.dist64[k & 1])) : 0.0;
      const double ks = exp(__dmul_rn(t.alpha_s, s));
      const double pot = __dmul_rn(__dmul_rn(t.pal_src64[t.fuel[u]], t.kw64[k]), ks);
      lam = __dadd_rn(lam, pot);
    }
  }
  return __dsub_rn(1.0, exp(-__dmul_rn(t.pal_gam64[t.fuel[v]], lam)));
}

// fp32 fast path: lambda and p within ~1e-6 relative of fp64 for |alpha_s| <= 50.
__device__ __forceinline__ float terrain_lambda32(const TerrainView& t, int w, int r, int c,
                                                  uint32_t nb) {
  const float zv = t.elev[r * w + c];
  float lam = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (nb & (1u << k)) {
      const int u = (r - kDy[k]) * w + (c - kDx[k]);
      const float dz = zv - t.elev[u];
      const float s = dz == dz ? atanf(dz * t.inv_dist32[k & 1]) : 0.f;  // nodata: slope 0
      // ex2.approx: relative error ~1e-7 for |alpha_s * s| <= 80 (force64 beyond), far inside the guard
      lam += t.pal_src32[t.fuel[u]] * t.kw32[k] * __expf(t.alpha_s32 * s);
    }
  }
  return lam;
}

// terrain_lambda32 over the fp32 slope table (launch_slope_table: slope_from_dem of the layers,
// built once with them like the reference's SlopeField): the candidate's 8 slopes are one 32-byte
// record, the 8 sources' fuel classes are loaded unconditionally (indices clamped into the h x w
// layer) -- one memory round trip, no atan -- and the directions without a burning source are
// selected away.  Same per-direction fp32 expression as terrain_lambda32.  pal_src: the palette's
// fp32 source values (shared memory).
__device__ __forceinline__ float terrain_lambda32_tab(const TerrainView& t, const float* __restrict__ slope32,
                                                      const float* pal_src, const float* kw, int w, int h,
                                                      int r, int c, uint32_t nb, uint8_t* fuel_v) {
  const int rs = r > 0 ? r - 1 : 0, rn = r + 1 < h ? r + 1 : h - 1;
  const int cw = c > 0 ? c - 1 : 0, ce = c + 1 < w ? c + 1 : w - 1;
  // u_k = (r - dy_k, c - dx_k), k = E NE N NW W SW S SE (kDx/kDy)
  const int ur[8] = {r, rs, rs, rs, r, rn, rn, rn};
  const int uc[8] = {cw, cw, c, ce, ce, ce, c, cw};
  const int v = r * w + c;
  const float4 s0 = __ldg(reinterpret_cast<const float4*>(slope32) + 2 * v);
  const float4 s1 = __ldg(reinterpret_cast<const float4*>(slope32) + 2 * v + 1);
  const float s[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
  *fuel_v = __ldg(t.fuel + v);
  uint8_t f[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) f[k] = __ldg(t.fuel + ur[k] * w + uc[k]);
  float lam = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float contrib = pal_src[f[k]] * kw[k] * __expf(t.alpha_s32 * s[k]);
    lam += (nb >> k) & 1u ? contrib : 0.f;
  }
  return lam;
}

__device__ __forceinline__ float ex2_approx(float x) {  // 2^x, rel. error ~2^-22 (MUFU.EX2)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// The leanest fp32 lambda: the candidate's slope record, its sources' class record, and a
// shared-memory table srckw[class * 8 + k] = src32(class) * kappa_wind32(k) of the wind in force;
// kappa_slope = 2^(alpha_s log2e * S).  Within ~3e-7 relative of terrain_lambda32 (guard 1e-4).
__device__ __forceinline__ float terrain_lambda32_rec(const float* __restrict__ slope32, const uint2* __restrict__ nfuel,
                                                      const float* srckw, float alpha_l2, int v, uint32_t nb) {
  const float4 s0 = __ldg(reinterpret_cast<const float4*>(slope32) + 2 * v);
  const float4 s1 = __ldg(reinterpret_cast<const float4*>(slope32) + 2 * v + 1);
  const uint2 nf = __ldg(nfuel + v);
  const float s[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
  float lam = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t f = ((k < 4 ? nf.x : nf.y) >> (8 * (k & 3))) & 0xffu;
    const float contrib = srckw[f * 8 + k] * ex2_approx(alpha_l2 * s[k]);
    lam += (nb >> k) & 1u ? contrib : 0.f;
  }
  return lam;
}

constexpr double kGuardRel = 1e-4;

__device__ __forceinline__ bool ignite_terrain(const TerrainView& t, int w, int r, int c,
                                               uint32_t nb, uint64_t m, const DiagCounters& dg) {
  const double u = bits_to_uniform(m);
  if (!t.force64) {
    const float lam = terrain_lambda32(t, w, r, c, nb);
    const float x = t.pal_gam32[t.fuel[r * w + c]] * lam;
    if (x == 0.f) return false;  // gamma or lambda exactly 0: p = 1 - exp(-0) = 0, u < 0 is false
    const double p32 = static_cast<double>(-expm1f(-x));
    // tiny p: the reference's 1 - exp(-x) is quantised to multiples of 2^-53 there; decide in fp64
    if (p32 > 1e-12) {
      if (u < p32 * (1.0 - kGuardRel)) return true;
      if (u >= p32 * (1.0 + kGuardRel)) return false;
    }
  }
  dg.fallback();
  const double p = terrain_p64(t, w, r, c, nb);
  if (fabs(u - p) < kAmbiguousBand) dg.ambiguous();
  return u < p;
}

// ignite_terrain with the slope-table fp32 lambda (blocked kernel); pal32s = [src 256][gam 256] in
// shared memory.  Same decisions as ignite_terrain (same fp32 values to rounding, same guard band,
// same fp64 path).
__device__ __forceinline__ bool ignite_terrain_tab(const TerrainView& t, const float* slope32, const float* pal32s,
                                                   const float* kw, int w, int h, int r, int c, uint32_t nb,
                                                   uint64_t m, const DiagCounters& dg) {
  const double u = bits_to_uniform(m);
  if (!t.force64) {
    uint8_t fv;
    const float lam = terrain_lambda32_tab(t, slope32, pal32s, kw, w, h, r, c, nb, &fv);
    const float x = pal32s[256 + fv] * lam;
    if (x == 0.f) return false;  // gamma or lambda exactly 0: p = 1 - exp(-0) = 0, u < 0 is false
    const double p32 = static_cast<double>(-expm1f(-x));
    if (p32 > 1e-12) {
      if (u < p32 * (1.0 - kGuardRel)) return true;
      if (u >= p32 * (1.0 + kGuardRel)) return false;
    }
  }
  dg.fallback();
  const double p = terrain_p64(t, w, r, c, nb);
  if (fabs(u - p) < kAmbiguousBand) dg.ambiguous();
  return u < p;
}

// p = 1 - e^-x in fp32 for the record form: a 4-term Taylor series below x = 0.03 (relative error
// < 1e-8), 1 - 2^(-x log2e) with MUFU.EX2 above (< 6e-6: the 2^-22 error of ex2 on e^-x, divided by
// p >= 0.03); within the 1e-5 bar and far inside the decision guard (kGuardRel = 1e-4).
__device__ __forceinline__ float p_ignite32(float x) {
  if (x < 0.03f) return x * (1.f - x * (0.5f - x * (1.f / 6.f - x * (1.f / 24.f))));
  return 1.f - ex2_approx(-x * 1.44269504088896341f);
}

// The same decision with the candidate's records already loaded (loads hoisted by the caller).
struct CellRec {
  float4 s0, s1;
  uint2 nf;
  uint32_t fv;
};
__device__ __forceinline__ CellRec load_rec(const float* __restrict__ slope32, const uint2* __restrict__ nfuel,
                                            const uint8_t* __restrict__ fuel, int v) {
  CellRec c;
  c.s0 = __ldg(reinterpret_cast<const float4*>(slope32) + 2 * v);
  c.s1 = __ldg(reinterpret_cast<const float4*>(slope32) + 2 * v + 1);
  c.nf = __ldg(nfuel + v);
  c.fv = __ldg(fuel + v);
  return c;
}
__device__ __forceinline__ bool ignite_terrain_rec_pre(const TerrainView& t, const CellRec& rc, const float* srckw,
                                                       const float* pal_gam, float alpha_l2, int w, int r, int c,
                                                       uint32_t nb, uint64_t m, const DiagCounters& dg) {
  if (!t.force64) {
    const float s[8] = {rc.s0.x, rc.s0.y, rc.s0.z, rc.s0.w, rc.s1.x, rc.s1.y, rc.s1.z, rc.s1.w};
    float lam = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t f = ((k < 4 ? rc.nf.x : rc.nf.y) >> (8 * (k & 3))) & 0xffu;
      const float contrib = srckw[f * 8 + k] * ex2_approx(alpha_l2 * s[k]);
      lam += (nb >> k) & 1u ? contrib : 0.f;
    }
    const float x = pal_gam[rc.fv] * lam;
    if (x == 0.f) return false;  // gamma or lambda exactly 0: p = 1 - exp(-0) = 0, u < 0 is false
    const float p32 = p_ignite32(x);
    if (p32 > 1e-12f) {
      // u < p (1 -+ guard)  <=>  m < p (1 -+ guard) 2^53: the thresholds in fp32 (relative rounding
      // 6e-8, inside the 1e-4 guard) and the 53-bit draw compared as an integer
      const uint64_t lo = static_cast<uint64_t>(p32 * static_cast<float>((1.0 - kGuardRel) * 0x1p53));
      const uint64_t hi = static_cast<uint64_t>(p32 * static_cast<float>((1.0 + kGuardRel) * 0x1p53));
      if (m < lo) return true;
      if (m >= hi) return false;
    }
  }
  dg.fallback();
  const double u = bits_to_uniform(m);
  const double p = terrain_p64(t, w, r, c, nb);
  if (fabs(u - p) < kAmbiguousBand) dg.ambiguous();
  return u < p;
}

// The same decision from the candidate's pot32t row (T0, T1: its 8 source terms gamma(v) * pot32,
// built by k_pot32t): x = gamma(v) lambda(v) is the k-ordered sum of the burning sources' terms --
// no exponentials, class lookups or fuel load per candidate.
__device__ __forceinline__ bool ignite_terrain_pot_pre(const TerrainView& t, float4 T0, float4 T1, int w, int r, int c,
                                                       uint32_t nb, uint64_t m, const DiagCounters& dg) {
  if (!t.force64) {
    const float T[8] = {T0.x, T0.y, T0.z, T0.w, T1.x, T1.y, T1.z, T1.w};
    float x = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) x += (nb >> k) & 1u ? T[k] : 0.f;
    if (x == 0.f) return false;  // gamma or lambda exactly 0: p = 0, u < 0 is false
    const float p32 = p_ignite32(x);
    if (p32 > 1e-12f) {
      const uint64_t lo = static_cast<uint64_t>(p32 * static_cast<float>((1.0 - kGuardRel) * 0x1p53));
      const uint64_t hi = static_cast<uint64_t>(p32 * static_cast<float>((1.0 + kGuardRel) * 0x1p53));
      if (m < lo) return true;
      if (m >= hi) return false;
    }
  }
  dg.fallback();
  const double u = bits_to_uniform(m);
  const double p = terrain_p64(t, w, r, c, nb);
  if (fabs(u - p) < kAmbiguousBand) dg.ambiguous();
  return u < p;
}

// ignite_terrain over terrain_lambda32_rec (blocked / tanker kernels when the palette has <= 32
// classes); pal_gam: the palette's fp32 gamma values (shared memory).
__device__ __forceinline__ bool ignite_terrain_rec(const TerrainView& t, const float* slope32, const uint2* nfuel,
                                                   const float* srckw, const float* pal_gam, float alpha_l2, int w,
                                                   int r, int c, uint32_t nb, uint64_t m, const DiagCounters& dg) {
  const double u = bits_to_uniform(m);
  if (!t.force64) {
    const int v = r * w + c;
    const float lam = terrain_lambda32_rec(slope32, nfuel, srckw, alpha_l2, v, nb);
    const float x = pal_gam[__ldg(t.fuel + v)] * lam;
    if (x == 0.f) return false;  // gamma or lambda exactly 0: p = 1 - exp(-0) = 0, u < 0 is false
    const double p32 = static_cast<double>(-expm1f(-x));
    if (p32 > 1e-12) {
      if (u < p32 * (1.0 - kGuardRel)) return true;
      if (u >= p32 * (1.0 + kGuardRel)) return false;
    }
  }
  dg.fallback();
  const double p = terrain_p64(t, w, r, c, nb);
  if (fabs(u - p) < kAmbiguousBand) dg.ambiguous();
  return u < p;
}

// Row of a wind schedule in force at absolute step `step` (WindSchedule::at_step clamps to the
// last entry, engine.cpp:81-86); 0 without a schedule.
__device__ __forceinline__ int sched_row(const StepArgs& a, uint64_t step) {
  return a.sched_len > 1 ? static_cast<int>(step < static_cast<uint64_t>(a.sched_len - 1) ? step : a.sched_len - 1)
                         : 0;
}

__device__ __forceinline__ TerrainView terrain_view(const StepArgs& a, int env, int srow = 0) {
  TerrainView t;
  const size_t base = static_cast<size_t>(env) * a.ter_stride;
  t.fuel = a.fuel + base;
  t.elev = a.elev + base;
  t.pal_src32 = a.pal32;
  t.pal_gam32 = a.pal32 + 256;
  t.pal_src64 = a.pal64;
  t.pal_gam64 = a.pal64 + 256;
  t.kw32 = a.kw32 + static_cast<size_t>(srow) * a.kw_sched_stride + env * a.kw_stride;
  t.kw64 = a.kw64 + static_cast<size_t>(srow) * a.kw_sched_stride + env * a.kw_stride;
  t.alpha_s32 = a.alpha_s32;
  t.alpha_s = a.alpha_s;
  t.inv_dist32[0] = a.inv_dist32[0];
  t.inv_dist32[1] = a.inv_dist32[1];
  t.dist64[0] = a.dist64[0];
  t.dist64[1] = a.dist64[1];
  t.force64 = a.force64;
  return t;
}

// ignite_terrain_pot_pre with the terrain view built only on the fp64 fallback path (the common
// fp32 decision needs none of its pointers).
__device__ __forceinline__ bool ignite_pot(const StepArgs& a, int env, int srow, float4 T0, float4 T1, int w, int r,
                                           int c, uint32_t nb, uint64_t m, const DiagCounters& dg) {
  if (!a.force64) {
    const float T[8] = {T0.x, T0.y, T0.z, T0.w, T1.x, T1.y, T1.z, T1.w};
    float x = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) x += (nb >> k) & 1u ? T[k] : 0.f;
    if (x == 0.f) return false;  // gamma or lambda exactly 0: p = 0, u < 0 is false
    const float p32 = p_ignite32(x);
    if (p32 > 1e-12f) {
      const uint64_t lo = static_cast<uint64_t>(p32 * static_cast<float>((1.0 - kGuardRel) * 0x1p53));
      const uint64_t hi = static_cast<uint64_t>(p32 * static_cast<float>((1.0 + kGuardRel) * 0x1p53));
      if (m < lo) return true;
      if (m >= hi) return false;
    }
  }
  const TerrainView t = terrain_view(a, env, srow);
  dg.fallback();
  const double u = bits_to_uniform(m);
  const double p = terrain_p64(t, w, r, c, nb);
  if (fabs(u - p) < kAmbiguousBand) dg.ambiguous();
  return u < p;
}

// ignite_pot with a shallower fp32 chain: the masked terms summed as a tree and p = 1 - e^-x
// without a branch (both forms evaluated, selected).  Same decision: the fp32 x only has to lie
// well inside the 1e-4 guard band (any order of 8 positive terms: within 4e-7 relative); every
// draw in the band is decided by the fp64 re-evaluation in the reference's association.  nb = 0
// (a burning cell routed through the same code path) returns false without touching the guard.
__device__ __forceinline__ bool ignite_pot_fast(const StepArgs& a, int env, int srow, float4 T0, float4 T1, int w,
                                                int r, int c, uint32_t nb, uint64_t m, const DiagCounters& dg) {
  if (!a.force64) {
    const float t0 = (nb & 1u) ? T0.x : 0.f, t1 = (nb & 2u) ? T0.y : 0.f, t2 = (nb & 4u) ? T0.z : 0.f;
    const float t3 = (nb & 8u) ? T0.w : 0.f, t4 = (nb & 16u) ? T1.x : 0.f, t5 = (nb & 32u) ? T1.y : 0.f;
    const float t6 = (nb & 64u) ? T1.z : 0.f, t7 = (nb & 128u) ? T1.w : 0.f;
    const float x = ((t0 + t1) + (t2 + t3)) + ((t4 + t5) + (t6 + t7));
    if (x == 0.f) return false;  // gamma or lambda exactly 0 (or no burning source): p = 0
    const float poly = x * (1.f - x * (0.5f - x * (1.f / 6.f - x * (1.f / 24.f))));
    const float p32 = x < 0.03f ? poly : 1.f - ex2_approx(-x * 1.44269504088896341f);
    if (p32 > 1e-12f) {
      const uint64_t lo = static_cast<uint64_t>(p32 * static_cast<float>((1.0 - kGuardRel) * 0x1p53));
      const uint64_t hi = static_cast<uint64_t>(p32 * static_cast<float>((1.0 + kGuardRel) * 0x1p53));
      if (m < lo) return true;
      if (m >= hi) return false;
    }
  } else if (nb == 0u) {
    return false;
  }
  const TerrainView t = terrain_view(a, env, srow);
  dg.fallback();
  const double u = bits_to_uniform(m);
  const double p = terrain_p64(t, w, r, c, nb);
  if (fabs(u - p) < kAmbiguousBand) dg.ambiguous();
  return u < p;
}

// Decision for an Unburned cell with burning-neighbour mask nb != 0.
// `srow` selects the wind-schedule entry in force (sched_row).
template <int MODE>
__device__ __forceinline__ bool ignite(const StepArgs& a, int env, int r, int c, uint32_t nb,
                                       uint64_t m, const DiagCounters& dg, int srow = 0) {
  if constexpr (MODE == kStaticTables) {
    const size_t base = static_cast<size_t>(env) * a.tab_stride;
    return ignite_tables(a.pot + static_cast<size_t>(srow) * a.pot_sched_stride + base * 8,
                         a.gamma + base, a.w, r, c, nb, m, dg);
  } else {
    return ignite_terrain(terrain_view(a, env, srow), a.w, r, c, nb, m, dg);
  }
}

}  // namespace ebl
