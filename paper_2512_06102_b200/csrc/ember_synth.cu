// Environment construction on the device:
//   * the C1 synthetic terrain generator (ember_host.cpp synth_terrain), bit-identical to the
//     host version: value noise summed in fp64 with explicit round-to-nearest ops (no FMA
//     contraction, as the host's -ffp-contract=off), exact min/max, an exact 4096-bin
//     histogram and the same integer quantile thresholds;
//   * seeded ignitions (ember_host.cpp synth_ignitions / FireSuppressionEnv::reset,
//     rl_env.cpp:125-145): one thread per env replays the redraw loop;
//   * fuel_from_landcover / grid_from_rasters (geodata.cpp:324-369): landcover codes mapped to
//     palette indices by binary search over the FuelTable's sorted codes, nodata (landcover
//     sentinel or DEM NaN) to the inert class.
// Layout: [env][row][col], row 0 = south, fuel uint8 palette index, elevation fp32.
#include <cstdint>

#include "ember_device.cuh"
#include "ember_kernels.h"

namespace ebl {

namespace {

constexpr int kSynthThreads = 256;
constexpr int kBins = 4096;          // ember_host.cpp synth_one
constexpr int kClasses = 11;
constexpr uint64_t kDrawSynthesis = 3;  // rng.hpp:25
constexpr uint64_t kDrawEnvSetup = 1;   // rng.hpp:23
constexpr int kMaxOctaves = 6;

__device__ __forceinline__ double lattice(uint64_t prefix, uint64_t i) {
  return bits_to_uniform(cell_bits53(prefix, i, kDrawSynthesis));
}

__device__ __forceinline__ double smooth(int rel, int L) {
  double f = __ddiv_rn(__dadd_rn(static_cast<double>(rel), 0.5), static_cast<double>(L));
  return __dmul_rn(__dmul_rn(f, f), __dsub_rn(3.0, __dmul_rn(2.0, f)));
}

// Octave-summed value noise at (r, c); pre[o] = key_prefix(seed, stream, layer + o).
__device__ double value_noise_at(const uint64_t* pre, int octaves, int base, int r, int c, int w) {
  double acc = 0.0, amp = 1.0;
  for (int o = 0; o < octaves; ++o) {
    const int L = max(1, base >> o);
    const int gw = w / L + 2;
    const int gy = r / L, gx = c / L;
    const double fy = smooth(r - gy * L, L), fx = smooth(c - gx * L, L);
    const uint64_t i0 = static_cast<uint64_t>(gy) * gw + gx, i1 = i0 + gw;
    const double a0 = lattice(pre[o], i0), a1 = lattice(pre[o], i0 + 1);
    const double b0 = lattice(pre[o], i1), b1 = lattice(pre[o], i1 + 1);
    const double top = __dadd_rn(a0, __dmul_rn(__dsub_rn(a1, a0), fx));
    const double bot = __dadd_rn(b0, __dmul_rn(__dsub_rn(b1, b0), fx));
    acc = __dadd_rn(acc, __dmul_rn(amp, __dadd_rn(top, __dmul_rn(__dsub_rn(bot, top), fy))));
    amp *= 0.5;
  }
  return acc;
}

// Noise values are sums of non-negative terms, so their IEEE bit patterns order like the values.
__device__ __forceinline__ void block_minmax(double v, bool valid, unsigned long long* g_lo,
                                             unsigned long long* g_hi) {
  __shared__ unsigned long long s_lo, s_hi;
  if (threadIdx.x == 0) {
    s_lo = ~0ull;
    s_hi = 0ull;
  }
  __syncthreads();
  unsigned long long lo = valid ? static_cast<unsigned long long>(__double_as_longlong(v)) : ~0ull;
  unsigned long long hi = valid ? lo : 0ull;
  for (int off = 16; off; off >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, off));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, off));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&s_lo, lo);
    atomicMax(&s_hi, hi);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicMin(g_lo, s_lo);
    atomicMax(g_hi, s_hi);
  }
}

__device__ __forceinline__ void load_prefixes(uint64_t* s_pre, const SynthArgs& a, int env,
                                              uint64_t layer, int octaves) {
  if (threadIdx.x < octaves)
    s_pre[threadIdx.x] = key_prefix(a.seed, a.env_id0 + static_cast<uint64_t>(env), layer + threadIdx.x);
  __syncthreads();
}

// pass 0: per-env min slots to all-ones, max slots and histogram to zero
__global__ void __launch_bounds__(kSynthThreads) k_synth_init(SynthArgs a) {
  const int env = blockIdx.x;
  if (threadIdx.x < 4) a.mm[env * 4 + threadIdx.x] = (threadIdx.x & 1) ? 0ull : ~0ull;
  for (int b = threadIdx.x; b < kBins; b += kSynthThreads) a.hist[static_cast<size_t>(env) * kBins + b] = 0;
}

// pass 1: landcover noise (layer 1000, 4 octaves) -> scratch, per-env min/max
__global__ void __launch_bounds__(kSynthThreads) k_synth_landcover(SynthArgs a) {
  __shared__ uint64_t s_pre[kMaxOctaves];
  const int env = blockIdx.y;
  load_prefixes(s_pre, a, env, 1000, 4);
  const size_t n = static_cast<size_t>(a.h) * a.w;
  const size_t i = static_cast<size_t>(blockIdx.x) * kSynthThreads + threadIdx.x;
  double v = 0.0;
  if (i < n) {
    v = value_noise_at(s_pre, 4, a.lc_base, static_cast<int>(i / a.w), static_cast<int>(i % a.w), a.w);
    a.scratch[static_cast<size_t>(env) * n + i] = v;
  }
  block_minmax(v, i < n, a.mm + env * 4 + 0, a.mm + env * 4 + 1);
}

__device__ __forceinline__ int bin_of(double x, double lo, double scale) {
  return min(kBins - 1, __double2int_rz(__dmul_rn(__dsub_rn(x, lo), scale)));
}

__device__ __forceinline__ double bits_double(unsigned long long b) {
  return __longlong_as_double(static_cast<long long>(b));
}

// pass 2: exact per-env histogram of the landcover bins (shared-memory counts, flushed once per CTA)
constexpr int kHistCellsPerThread = 16;
__global__ void __launch_bounds__(kSynthThreads) k_synth_hist(SynthArgs a) {
  __shared__ unsigned int s_hist[kBins];
  const int env = blockIdx.y;
  for (int b = threadIdx.x; b < kBins; b += kSynthThreads) s_hist[b] = 0;
  __syncthreads();
  const size_t n = static_cast<size_t>(a.h) * a.w;
  const double lo = bits_double(a.mm[env * 4 + 0]), hi = bits_double(a.mm[env * 4 + 1]);
  const double scale = hi > lo ? __ddiv_rn(static_cast<double>(kBins), __dsub_rn(hi, lo)) : 0.0;
  const double* v = a.scratch + static_cast<size_t>(env) * n;
  const size_t i0 = static_cast<size_t>(blockIdx.x) * kSynthThreads * kHistCellsPerThread;
  for (int j = 0; j < kHistCellsPerThread; ++j) {
    const size_t i = i0 + static_cast<size_t>(j) * kSynthThreads + threadIdx.x;
    if (i < n) atomicAdd(&s_hist[bin_of(v[i], lo, scale)], 1u);
  }
  __syncthreads();
  unsigned int* g = a.hist + static_cast<size_t>(env) * kBins;
  for (int b = threadIdx.x; b < kBins; b += kSynthThreads)
    if (s_hist[b]) atomicAdd(&g[b], s_hist[b]);
}

// pass 3: the ten equal-count thresholds per env (serial integer scan, one thread per env)
__global__ void k_synth_thresholds(SynthArgs a) {
  const int env = blockIdx.x * blockDim.x + threadIdx.x;
  if (env >= a.n_envs) return;
  const uint64_t n = static_cast<uint64_t>(a.h) * a.w;
  const unsigned int* hist = a.hist + static_cast<size_t>(env) * kBins;
  int* thr = a.thr + env * (kClasses - 1);
  uint64_t cum = 0;
  int j = 0;
  for (int b = 0; b < kBins && j < kClasses - 1; ++b) {
    cum += hist[b];
    while (j < kClasses - 1 && cum * kClasses >= static_cast<uint64_t>(j + 1) * n) thr[j++] = b + 1;
  }
  while (j < kClasses - 1) thr[j++] = kBins;
}

// pass 4: classify landcover -> fuel class; elevation noise (layer 2000, 6 octaves) -> scratch
__global__ void __launch_bounds__(kSynthThreads) k_synth_classify(SynthArgs a) {
  __shared__ uint64_t s_pre[kMaxOctaves];
  __shared__ int s_thr[kClasses - 1];
  const int env = blockIdx.y;
  if (threadIdx.x < kClasses - 1) s_thr[threadIdx.x] = a.thr[env * (kClasses - 1) + threadIdx.x];
  load_prefixes(s_pre, a, env, 2000, 6);
  const size_t n = static_cast<size_t>(a.h) * a.w;
  const size_t i = static_cast<size_t>(blockIdx.x) * kSynthThreads + threadIdx.x;
  double v = 0.0;
  if (i < n) {
    const double lo = bits_double(a.mm[env * 4 + 0]), hi = bits_double(a.mm[env * 4 + 1]);
    const double scale = hi > lo ? __ddiv_rn(static_cast<double>(kBins), __dsub_rn(hi, lo)) : 0.0;
    const size_t gi = static_cast<size_t>(env) * n + i;
    const int b = bin_of(a.scratch[gi], lo, scale);
    int k = 0;
    while (k < kClasses - 1 && b >= s_thr[k]) ++k;
    a.fuel[gi] = static_cast<uint8_t>(k);
    v = value_noise_at(s_pre, 6, a.el_base, static_cast<int>(i / a.w), static_cast<int>(i % a.w), a.w);
    a.scratch[gi] = v;
  }
  block_minmax(v, i < n, a.mm + env * 4 + 2, a.mm + env * 4 + 3);
}

// pass 5: elevation = float((v - lo) * (elev_max / (hi - lo)))
__global__ void __launch_bounds__(kSynthThreads) k_synth_elevation(SynthArgs a) {
  const int env = blockIdx.y;
  const size_t n = static_cast<size_t>(a.h) * a.w;
  const size_t i = static_cast<size_t>(blockIdx.x) * kSynthThreads + threadIdx.x;
  if (i >= n) return;
  const double lo = bits_double(a.mm[env * 4 + 2]), hi = bits_double(a.mm[env * 4 + 3]);
  const double es = hi > lo ? __ddiv_rn(a.elev_max, __dsub_rn(hi, lo)) : 0.0;
  const size_t gi = static_cast<size_t>(env) * n + i;
  a.elev[gi] = __double2float_rn(__dmul_rn(__dsub_rn(a.scratch[gi], lo), es));
}

// Seeded ignitions: rng_below(key{seed, 0, env_id0 + e}, counter++, kDrawEnvSetup, H*W), redrawn on
// an already-burning or unburnable cell, at most 64*H*W draws (ember_host.cpp synth_ignitions).
__global__ void k_synth_ignitions(IgniteArgs a) {
  const int env = blockIdx.x * blockDim.x + threadIdx.x;
  if (env >= a.n_envs) return;
  const uint64_t n = static_cast<uint64_t>(a.h) * a.w;
  uint8_t* st = a.states + static_cast<size_t>(env) * n;
  const uint8_t* fc = a.fuel + static_cast<size_t>(env) * a.fuel_stride;
  const uint64_t pre = key_prefix(a.seed, a.env_id0 + static_cast<uint64_t>(env), 0);
  uint64_t counter = 0;
  int placed = 0;
  while (placed < a.count && counter < 64 * n) {
    const uint64_t cell = below(cell_bits53(pre, counter++, kDrawEnvSetup), n);
    if (st[cell] == 1 || !(a.burnable[fc[cell]] > 0.0)) continue;
    st[cell] = 1;
    ++placed;
  }
  a.placed[env] = placed;
}

// Landcover code -> palette index: the FuelTable's codes sorted ascending occupy indices
// 0..n_codes-1, the fallback (if any) n_codes, the inert nodata class the next index.
__global__ void __launch_bounds__(kSynthThreads) k_landcover_map(LandcoverArgs a) {
  __shared__ int32_t s_codes[256];
  for (int k = threadIdx.x; k < a.n_codes; k += kSynthThreads) s_codes[k] = a.codes[k];
  __syncthreads();
  const size_t i = static_cast<size_t>(blockIdx.x) * kSynthThreads + threadIdx.x;
  if (i >= a.n) return;
  const int32_t code = a.landcover[i];
  const bool nodata = (a.has_nodata && code == a.nodata_code) ||
                      (a.elev != nullptr && isnan(a.elev[i]));
  int k;
  if (nodata) {
    k = a.nodata_index;
  } else {
    int lo = 0, hi = a.n_codes;  // first index with s_codes[idx] >= code
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (s_codes[mid] < code) lo = mid + 1; else hi = mid;
    }
    if (lo < a.n_codes && s_codes[lo] == code) {
      k = lo;
    } else if (a.fallback_index >= 0) {
      k = a.fallback_index;
    } else {
      // FuelTable::lookup throws naming the code (geodata.cpp:248-253): report the first cell
      atomicMin(a.missing, static_cast<unsigned long long>(i));
      k = 0;
    }
  }
  a.fuel[i] = static_cast<uint8_t>(k);
}

// Also the fuel classes of each cell's 8 sources (one 8-byte record), so a candidate's lambda needs
// one slope record + one source-class record.
// slope_from_dem (geodata.cpp:209-229) in the fp32 fast-path form: S[cell][k] = atan((z(v) - z(u_k)) /
// dist_k) for target v and source u_k = v - d_k, the same fp32 expression terrain_lambda32 evaluates
// on the fly (so the tabulated and the on-the-fly lambda are bit-identical).  Sources outside the
// layer and DEM nodata (NaN) on either end give 0.
__global__ void __launch_bounds__(kSynthThreads) k_slope_table(const float* __restrict__ elev,
                                                                const uint8_t* __restrict__ fuel, size_t n_cells,
                                                                int h, int w, float inv_d0, float inv_d1,
                                                                float4* __restrict__ out, uint2* __restrict__ nf) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_cells) return;
  const size_t layer = static_cast<size_t>(h) * w;
  const size_t g = i / layer;
  const int v = static_cast<int>(i - g * layer);
  const int r = v / w, c = v - r * w;
  const float* z = elev + g * layer;
  const float zv = z[v];
  const uint8_t* f = fuel + g * layer;
  float s[8];
  uint32_t nf0 = 0u, nf1 = 0u;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int ur = r - kDy[k], uc = c - kDx[k];
    float sk = 0.f;
    uint32_t fk = 0u;  // outside the layer: class 0 (never weighted: no burning source there)
    if (ur >= 0 && ur < h && uc >= 0 && uc < w) {
      const float dz = zv - z[ur * w + uc];
      sk = dz == dz ? atanf(dz * (k & 1 ? inv_d1 : inv_d0)) : 0.f;
      fk = f[ur * w + uc];
    }
    s[k] = sk;
    if (k < 4) nf0 |= fk << (8 * k);
    else nf1 |= fk << (8 * (k - 4));
  }
  out[2 * i] = make_float4(s[0], s[1], s[2], s[3]);
  out[2 * i + 1] = make_float4(s[4], s[5], s[6], s[7]);
  nf[i] = make_uint2(nf0, nf1);
}

// pot32t[env][v][k] = gamma32(v) (src32(class of u_k) kappa_wind32(k) 2^(alpha_s log2e S(v, k))):
// the fp32 term of source u_k = v - d_k in x = gamma(v) lambda(v) -- the product the record form
// evaluates per candidate (terrain_lambda32_rec), scaled by the target's gamma -- built once per
// (terrain, wind, config).
__global__ void __launch_bounds__(kSynthThreads) k_pot32t(const float4* __restrict__ slope32, const uint2* __restrict__ nfuel,
                                                        const uint8_t* __restrict__ fuel, const float* __restrict__ pal32,
                                                        const float* __restrict__ kw32, int n_envs, size_t ncell,
                                                        size_t ter_stride, int kw_stride, float alpha_l2,
                                                        float4* __restrict__ out) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= ncell * n_envs) return;
  const size_t env = i / ncell, v = i - env * ncell;
  const size_t g = env * ter_stride + v;
  const float4 s0 = slope32[2 * g], s1 = slope32[2 * g + 1];
  const uint2 nf = nfuel[g];
  const float s[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
  const float* kw = kw32 + env * kw_stride;
  const float gam = pal32[256 + fuel[g]];  // the target's gamma32 (0 for non-burnable targets)
  float o[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t f = ((k < 4 ? nf.x : nf.y) >> (8 * (k & 3))) & 0xffu;
    const float srckw = pal32[f] * kw[k];
    o[k] = gam * (srckw * ex2_approx(alpha_l2 * s[k]));
  }
  out[2 * i] = make_float4(o[0], o[1], o[2], o[3]);
  out[2 * i + 1] = make_float4(o[4], o[5], o[6], o[7]);
}

// Snapshot text (serialize_snapshot, snapshot.cpp:55-70) of n layers: one CTA per layer writes
// its header, the H lines of W characters from {U, B, X} (northmost row first; other byte values
// '?', as state_char), and its optional agent line, at the layer's offset of the concatenation.
// meta holds the host-formatted header and agent strings; off[i] = {text offset, meta offset,
// header length, agent length}.
__global__ void k_snapshot_text(const uint8_t* __restrict__ layers, int h, int w, const char* __restrict__ meta,
                                const unsigned long long* __restrict__ off, char* __restrict__ out) {
  const int i = blockIdx.x;
  const unsigned long long o = off[4 * i], mo = off[4 * i + 1], hl = off[4 * i + 2], al = off[4 * i + 3];
  char* t = out + o;
  for (unsigned long long k = threadIdx.x; k < hl; k += blockDim.x) t[k] = meta[mo + k];
  t += hl;
  const uint8_t* L = layers + static_cast<size_t>(i) * h * w;
  const int line = w + 1;
  const size_t body = static_cast<size_t>(h) * line;
  for (size_t k = threadIdx.x; k < body; k += blockDim.x) {
    const int ln = static_cast<int>(k / line), col = static_cast<int>(k - static_cast<size_t>(ln) * line);
    char ch = '\n';
    if (col < w) {
      const uint8_t v = L[static_cast<size_t>(h - 1 - ln) * w + col];
      ch = v == 0 ? 'U' : v == 1 ? 'B' : v == 2 ? 'X' : '?';
    }
    t[k] = ch;
  }
  t += body;
  for (unsigned long long k = threadIdx.x; k < al; k += blockDim.x) t[k] = meta[mo + hl + k];
}

inline unsigned grid_x(size_t n) { return static_cast<unsigned>((n + kSynthThreads - 1) / kSynthThreads); }

}  // namespace

cudaError_t launch_synth_terrain(const SynthArgs& a, cudaStream_t s) {
  const size_t n = static_cast<size_t>(a.h) * a.w;
  const dim3 grid(grid_x(n), a.n_envs);
  k_synth_init<<<a.n_envs, kSynthThreads, 0, s>>>(a);
  k_synth_landcover<<<grid, kSynthThreads, 0, s>>>(a);
  const size_t per_cta = static_cast<size_t>(kSynthThreads) * kHistCellsPerThread;
  k_synth_hist<<<dim3(static_cast<unsigned>((n + per_cta - 1) / per_cta), a.n_envs), kSynthThreads, 0, s>>>(a);
  k_synth_thresholds<<<(a.n_envs + 127) / 128, 128, 0, s>>>(a);
  k_synth_classify<<<grid, kSynthThreads, 0, s>>>(a);
  k_synth_elevation<<<grid, kSynthThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_synth_ignitions(const IgniteArgs& a, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(a.states, 0, static_cast<size_t>(a.n_envs) * a.h * a.w, s);
  if (e != cudaSuccess) return e;
  k_synth_ignitions<<<(a.n_envs + 63) / 64, 64, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_slope_table(const float* elev, const uint8_t* fuel, size_t n_grids, int h, int w, float inv_d0,
                               float inv_d1, float* out, uint2* nfuel, cudaStream_t s) {
  const size_t n = n_grids * h * w;
  k_slope_table<<<grid_x(n), kSynthThreads, 0, s>>>(elev, fuel, n, h, w, inv_d0, inv_d1, reinterpret_cast<float4*>(out),
                                                    nfuel);
  return cudaGetLastError();
}

cudaError_t launch_pot32t(const float* slope32, const uint2* nfuel, const uint8_t* fuel, const float* pal32,
                          const float* kw32, int n_envs, size_t ncell, size_t ter_stride, int kw_stride, float alpha_l2,
                          float* out, cudaStream_t s) {
  const size_t n = ncell * n_envs;
  k_pot32t<<<grid_x(n), kSynthThreads, 0, s>>>(reinterpret_cast<const float4*>(slope32), nfuel, fuel, pal32, kw32, n_envs,
                                               ncell, ter_stride, kw_stride, alpha_l2, reinterpret_cast<float4*>(out));
  return cudaGetLastError();
}

cudaError_t launch_snapshot_text(const uint8_t* layers, int n, int h, int w, const char* meta,
                                 const unsigned long long* off, char* out, cudaStream_t s) {
  if (n > 0) k_snapshot_text<<<n, kSynthThreads, 0, s>>>(layers, h, w, meta, off, out);
  return cudaGetLastError();
}

cudaError_t launch_landcover_map(const LandcoverArgs& a, cudaStream_t s) {
  k_landcover_map<<<grid_x(a.n), kSynthThreads, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace ebl
