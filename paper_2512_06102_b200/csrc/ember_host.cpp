// Host-side fp64 math and input generators; see ember_host.h.
#include "ember_host.h"

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <vector>

namespace ebl {

namespace {
constexpr double kTwoPi = 2.0 * 3.14159265358979323846;
constexpr int kDx[8] = {1, 1, 0, -1, -1, -1, 0, 1};
constexpr int kDy[8] = {0, 1, 1, 1, 0, -1, -1, -1};
constexpr uint64_t kDrawSynthesis = 3;  // rng.hpp:25
constexpr uint64_t kDrawEnvSetup = 1;   // rng.hpp:23

inline uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}
}  // namespace

uint64_t rng_word(uint64_t seed, uint64_t step, uint64_t stream, uint64_t cell, uint64_t draw) {
  return mix64(mix64(mix64(mix64(mix64(0x243F6A8885A308D3ull ^ seed) ^ stream) ^ step) ^ cell) ^ draw);
}

double rng_uniform(uint64_t seed, uint64_t step, uint64_t stream, uint64_t cell, uint64_t draw) {
  return static_cast<double>(rng_word(seed, step, stream, cell, draw) >> 11) * 0x1.0p-53;
}

uint64_t rng_below(uint64_t seed, uint64_t step, uint64_t stream, uint64_t cell, uint64_t draw,
                   uint64_t n) {
  const auto v = static_cast<uint64_t>(rng_uniform(seed, step, stream, cell, draw) * static_cast<double>(n));
  return v < n ? v : n - 1;
}

double wrap_angle(double a) {
  double w = std::fmod(a, kTwoPi);
  if (w < 0.0) w += kTwoPi;
  return w;
}

double offset_angle(int k) {
  return wrap_angle(std::atan2(static_cast<double>(kDy[k]), static_cast<double>(kDx[k])));
}

double clamp_fuel(double v) { return std::clamp(v, -1.0, 1.0); }

void kappa_wind8(double speed, double direction, const Cfg6& c, double kw[8]) {
  const double dir = wrap_angle(direction);
  for (int k = 0; k < 8; ++k) {
    const double align = std::cos(offset_angle(k) - dir) - 1.0;
    kw[k] = std::exp(c.alpha_w1 * speed) * std::exp((c.alpha_w2 * speed) * align);
  }
}

void build_tables(size_t n, const double* speed, const double* dir, const double* veg,
                  const double* den, const double* slope8, const Cfg6& c, double* pot,
                  double* gamma) {
#pragma omp parallel for schedule(static) if (n > 16384)
  for (long long ii = 0; ii < static_cast<long long>(n); ++ii) {
    const size_t i = static_cast<size_t>(ii);
    const double v = clamp_fuel(veg[i]), d = clamp_fuel(den[i]);
    const double source = (c.p_base * (1.0 + v)) * (1.0 + d);
    gamma[i] = (c.alpha_gamma * (1.0 + v)) * (1.0 + d);
    double kw[8];
    kappa_wind8(speed[i], dir[i], c, kw);
    for (int k = 0; k < 8; ++k) {
      const double sf = std::exp(c.alpha_s * slope8[i * 8 + k]);
      pot[i * 8 + k] = (source * kw[k]) * sf;
    }
  }
}

void build_det_factors(size_t n, const double* speed, const double* dir, const double* veg,
                       const double* den, const double* slope8, const Cfg6& c, double* F,
                       double* pb, double* V, double* Va, double* S) {
#pragma omp parallel for schedule(static) if (n > 16384)
  for (long long ii = 0; ii < static_cast<long long>(n); ++ii) {
    const size_t i = static_cast<size_t>(ii);
    const double v = clamp_fuel(veg[i]), d = clamp_fuel(den[i]);
    F[i] = (1.0 + v) * (1.0 + d);
    V[i] = speed[i];
    double kw[8];
    kappa_wind8(speed[i], dir[i], c, kw);
    const double wd = wrap_angle(dir[i]);
    for (int k = 0; k < 8; ++k) {
      const double s = slope8[i * 8 + k];
      pb[i * 8 + k] = (F[i] * kw[k]) * std::exp(c.alpha_s * s);  // dpot/dp_base
      Va[i * 8 + k] = speed[i] * (std::cos(offset_angle(k) - wd) - 1.0);
      S[i * 8 + k] = s;
    }
  }
}

void build_terrain_tables(int n_tables, int h, int w, const uint8_t* fuel, const float* elev,
                          size_t grid_stride, const double* class_veg, const double* class_den,
                          double cellsize, const double* wind_speed, const double* wind_dir,
                          int wind_stride, const Cfg6& c, double* pot, double* gamma) {
  const size_t n = static_cast<size_t>(h) * w;
  const double dist[2] = {cellsize * 1.0, cellsize * 1.41421356237309504880};  // geodata.cpp:222-223
#pragma omp parallel for schedule(dynamic, 1)
  for (int t = 0; t < n_tables; ++t) {
    const uint8_t* f = fuel + t * grid_stride;
    const float* z = elev + t * grid_stride;
    double kw[8];
    kappa_wind8(wind_speed[t * wind_stride], wind_dir[t * wind_stride], c, kw);
    double* P = pot + t * n * 8;
    double* G = gamma + t * n;
    for (int r = 0; r < h; ++r)
      for (int col = 0; col < w; ++col) {
        const size_t i = static_cast<size_t>(r) * w + col;
        const double v = clamp_fuel(class_veg[f[i]]), d = clamp_fuel(class_den[f[i]]);
        const double source = (c.p_base * (1.0 + v)) * (1.0 + d);  // engine.hpp:88
        G[i] = (c.alpha_gamma * (1.0 + v)) * (1.0 + d);           // engine.hpp:89
        for (int k = 0; k < 8; ++k) {
          const int nr = r + kDy[k], nc = col + kDx[k];
          double s = 0.0;  // slope_from_dem: 0 toward out-of-bounds neighbours
          if (nr >= 0 && nr < h && nc >= 0 && nc < w) {
            const double dz = static_cast<double>(z[static_cast<size_t>(nr) * w + nc]) - static_cast<double>(z[i]);
            if (dz == dz) s = std::atan(dz / dist[k & 1]);  // NaN = DEM nodata: slope 0 (geodata.cpp:214,220)
          }
          P[i * 8 + k] = (source * kw[k]) * std::exp(c.alpha_s * s);  // engine.hpp:91,106-107
        }
      }
  }
}

void build_terrain_slopes64(int n_grids, int h, int w, const float* elev, size_t grid_stride, double cellsize,
                            double* S) {
  const size_t n = static_cast<size_t>(h) * w;
  const double dist[2] = {cellsize * 1.0, cellsize * 1.41421356237309504880};  // geodata.cpp:222-223
#pragma omp parallel for schedule(dynamic, 1)
  for (int g = 0; g < n_grids; ++g) {
    const float* z = elev + g * grid_stride;
    double* out = S + g * n * 8;
    for (int r = 0; r < h; ++r)
      for (int col = 0; col < w; ++col) {
        const size_t i = static_cast<size_t>(r) * w + col;
        for (int k = 0; k < 8; ++k) {
          const int nr = r + kDy[k], nc = col + kDx[k];
          double s = 0.0;  // exactly the expression of build_terrain_tables
          if (nr >= 0 && nr < h && nc >= 0 && nc < w) {
            const double dz = static_cast<double>(z[static_cast<size_t>(nr) * w + nc]) - static_cast<double>(z[i]);
            if (dz == dz) s = std::atan(dz / dist[k & 1]);
          }
          out[i * 8 + k] = s;
        }
      }
  }
}

uint64_t continue_threshold(double pc) {
  if (!(pc > 0.0)) return 0;  // also NaN: u < NaN is false
  if (pc >= 1.0) return 1ull << 53;
  return static_cast<uint64_t>(std::ceil(pc * 0x1.0p53));
}

// ---- synthetic inputs ---------------------------------------------------------------
namespace {

// Octave-summed 2-D value noise on a lattice of period base>>o, smoothstep-bilinear,
// lattice values rng_uniform(seed, layer+o, stream, lattice index, kDrawSynthesis).
void value_noise(uint64_t seed, uint64_t layer, uint64_t stream, int h, int w, int octaves,
                 int base, bool par, std::vector<double>& out) {
  out.assign(static_cast<size_t>(h) * w, 0.0);
  double amp = 1.0;
  for (int o = 0; o < octaves; ++o) {
    const int L = std::max(1, base >> o);
    const int gh = h / L + 2, gw = w / L + 2;
    std::vector<double> lat(static_cast<size_t>(gh) * gw);
    for (size_t i = 0; i < lat.size(); ++i)
      lat[i] = rng_uniform(seed, layer + static_cast<uint64_t>(o), stream, i, kDrawSynthesis);
#pragma omp parallel for schedule(static) if (par)
    for (int r = 0; r < h; ++r) {
      const int gy = r / L;
      double fy = (r - gy * L + 0.5) / L;
      fy = fy * fy * (3.0 - 2.0 * fy);
      for (int c = 0; c < w; ++c) {
        const int gx = c / L;
        double fx = (c - gx * L + 0.5) / L;
        fx = fx * fx * (3.0 - 2.0 * fx);
        const double* l0 = &lat[static_cast<size_t>(gy) * gw + gx];
        const double* l1 = l0 + gw;
        const double top = l0[0] + (l0[1] - l0[0]) * fx;
        const double bot = l1[0] + (l1[1] - l1[0]) * fx;
        out[static_cast<size_t>(r) * w + c] += amp * (top + (bot - top) * fy);
      }
    }
    amp *= 0.5;
  }
}

void synth_one(uint64_t seed, uint64_t stream, int h, int w, double elev_max, bool par,
               uint8_t* cls, float* elev) {
  const size_t n = static_cast<size_t>(h) * w;
  std::vector<double> v;
  // landcover: 4 octaves, period min(64, max(4, min(h,w)/4)); 11 equal-count classes
  const int lc_base = std::min(64, std::max(4, std::min(h, w) / 4));
  value_noise(seed, 1000, stream, h, w, 4, lc_base, par, v);
  double lo = v[0], hi = v[0];
  for (double x : v) lo = std::min(lo, x), hi = std::max(hi, x);
  constexpr int kBins = 4096;
  std::vector<uint64_t> hist(kBins, 0);
  const double scale = hi > lo ? kBins / (hi - lo) : 0.0;
  auto bin_of = [&](double x) { return std::min(kBins - 1, static_cast<int>((x - lo) * scale)); };
  for (double x : v) hist[bin_of(x)]++;
  int thr[10];
  {
    uint64_t cum = 0;
    int j = 0;
    for (int b = 0; b < kBins && j < 10; ++b) {
      cum += hist[b];
      while (j < 10 && cum * 11 >= static_cast<uint64_t>(j + 1) * n) thr[j++] = b + 1;
    }
    while (j < 10) thr[j++] = kBins;
  }
#pragma omp parallel for schedule(static) if (par)
  for (long long i = 0; i < static_cast<long long>(n); ++i) {
    const int b = bin_of(v[i]);
    int k = 0;
    while (k < 10 && b >= thr[k]) ++k;
    cls[i] = static_cast<uint8_t>(k);
  }
  // elevation: 6-octave fractal noise, period min(128, max(8, min(h,w)/2)), scaled to [0, elev_max]
  const int el_base = std::min(128, std::max(8, std::min(h, w) / 2));
  value_noise(seed, 2000, stream, h, w, 6, el_base, par, v);
  lo = v[0], hi = v[0];
  for (double x : v) lo = std::min(lo, x), hi = std::max(hi, x);
  const double es = hi > lo ? elev_max / (hi - lo) : 0.0;
#pragma omp parallel for schedule(static) if (par)
  for (long long i = 0; i < static_cast<long long>(n); ++i) elev[i] = static_cast<float>((v[i] - lo) * es);
}

}  // namespace

void synth_terrain(uint64_t seed, uint32_t env_id0, int n_envs, int h, int w, double elev_max,
                   double wind_max, uint8_t* fuel_class, float* elevation, double* wind_speed,
                   double* wind_direction) {
  const size_t n = static_cast<size_t>(h) * w;
  const bool inner = n_envs < 4;
#pragma omp parallel for schedule(dynamic, 1) if (!inner)
  for (int e = 0; e < n_envs; ++e) {
    const uint64_t stream = env_id0 + static_cast<uint64_t>(e);
    synth_one(seed, stream, h, w, elev_max, inner, fuel_class + e * n, elevation + e * n);
    if (wind_speed) wind_speed[e] = wind_max * rng_uniform(seed, 3000, stream, 0, kDrawSynthesis);
    if (wind_direction) wind_direction[e] = kTwoPi * rng_uniform(seed, 3000, stream, 1, kDrawSynthesis);
  }
}

// default_worldcover_table (geodata.cpp:305-319) as a dense palette in code order.
void worldcover_palette(int32_t* codes, double* veg, double* den) {
  static const int32_t c[11] = {10, 20, 30, 40, 50, 60, 70, 80, 90, 95, 100};
  static const double v[11] = {0.4, 0.25, 0.15, 0.0, -0.8, -0.7, -1.0, -1.0, -0.4, -0.2, -0.3};
  static const double d[11] = {0.3, 0.1, -0.1, -0.2, -0.8, -0.6, -1.0, -1.0, -0.3, -0.1, -0.4};
  for (int i = 0; i < 11; ++i) {
    if (codes) codes[i] = c[i];
    if (veg) veg[i] = v[i];
    if (den) den[i] = d[i];
  }
}

int synth_ignitions(uint64_t seed, uint32_t env_id0, int n_envs, int h, int w,
                    const uint8_t* fuel_class, const double* class_veg, const double* class_den,
                    int count, uint8_t* states) {
  const uint64_t n = static_cast<uint64_t>(h) * w;
  int total = 0;
#pragma omp parallel for schedule(static) reduction(+ : total) if (n_envs > 64)
  for (int e = 0; e < n_envs; ++e) {
    uint8_t* st = states + e * n;
    const uint8_t* fc = fuel_class + e * n;
    std::fill(st, st + n, uint8_t{0});
    const uint64_t stream = env_id0 + static_cast<uint64_t>(e);
    uint64_t counter = 0;
    int placed = 0;
    while (placed < count && counter < 64 * n) {
      const uint64_t cell = rng_below(seed, 0, stream, counter++, kDrawEnvSetup, n);
      const uint8_t k = fc[cell];
      const bool burnable = (1.0 + clamp_fuel(class_veg[k])) * (1.0 + clamp_fuel(class_den[k])) > 0.0;
      if (st[cell] == 1 || !burnable) continue;
      st[cell] = 1;
      ++placed;
    }
    total += placed;
  }
  return total;
}

}  // namespace ebl
