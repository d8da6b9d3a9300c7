/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's hot path.
 * See ember_oracle.h for the contract and what pins it.  Compiled with
 * -ffp-contract=off like the reference (proj/CMakeLists.txt:16) so every
 * double expression rounds exactly as the reference's does; the association
 * of each product below is the reference's (kernel.hpp:9-10 "fixed on
 * purpose"). */
#include "ember_oracle.h"

#include <math.h>
#include <stdio.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define TWO_PI (2.0 * 3.14159265358979323846)
#define SQRT2 1.41421356237309504880

/* grid.hpp:74-83 — (dx east, dy north) */
static const int kDx[8] = {1, 1, 0, -1, -1, -1, 0, 1};
static const int kDy[8] = {0, 1, 1, 1, 0, -1, -1, -1};

enum { DRAW_FIRE = 0, DRAW_SETUP = 1, DRAW_POLICY = 2 }; /* rng.hpp:22-25 */

/* ---------------------------------------------------------------- rng.hpp:28-58 */
static uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

uint64_t ebo_rng_word(uint64_t seed, uint64_t step, uint64_t stream, uint64_t cell, uint64_t draw) {
  /* hash order seed -> stream -> step -> cell -> draw (rng.hpp:40-44) */
  uint64_t h = mix64(0x243F6A8885A308D3ull ^ seed);
  h = mix64(h ^ stream);
  h = mix64(h ^ step);
  h = mix64(h ^ cell);
  return mix64(h ^ draw);
}

double ebo_rng_uniform(uint64_t seed, uint64_t step, uint64_t stream, uint64_t cell, uint64_t draw) {
  return (double)(ebo_rng_word(seed, step, stream, cell, draw) >> 11) * 0x1.0p-53;
}

uint64_t ebo_rng_below(uint64_t seed, uint64_t step, uint64_t stream, uint64_t cell, uint64_t draw,
                       uint64_t n) {
  const uint64_t v = (uint64_t)(ebo_rng_uniform(seed, step, stream, cell, draw) * (double)n);
  return v < n ? v : n - 1;
}

/* ---------------------------------------------------------------- grid.cpp:35-47 */
double ebo_wrap_angle(double a) {
  double w = fmod(a, TWO_PI);
  if (w < 0.0) w += TWO_PI;
  return w;
}

double ebo_offset_angle(int k) { return ebo_wrap_angle(atan2((double)kDy[k], (double)kDx[k])); }

static double clamp1(double v) { return v < -1.0 ? -1.0 : (v > 1.0 ? 1.0 : v); }

static ebo_grid* grid_alloc(int h, int w) {
  ebo_grid* g = (ebo_grid*)calloc(1, sizeof(ebo_grid));
  const size_t n = (size_t)h * w;
  g->h = h;
  g->w = w;
  g->speed = (double*)malloc(n * sizeof(double));
  g->dir = (double*)malloc(n * sizeof(double));
  g->veg = (double*)malloc(n * sizeof(double));
  g->den = (double*)malloc(n * sizeof(double));
  g->slope8 = (double*)calloc(n * 8, sizeof(double));
  return g;
}

ebo_grid* ebo_grid_layers(int h, int w, const double* speed, const double* dir, const double* veg,
                          const double* den, const double* slope8) {
  ebo_grid* g = grid_alloc(h, w);
  const size_t n = (size_t)h * w;
  for (size_t i = 0; i < n; ++i) {
    g->speed[i] = speed[i];
    g->dir[i] = ebo_wrap_angle(dir[i]); /* WindField ctor, grid.cpp:57-60 */
    g->veg[i] = clamp1(veg[i]);         /* FuelField ctor, grid.cpp:75-76 */
    g->den[i] = clamp1(den[i]);
  }
  memcpy(g->slope8, slope8, n * 8 * sizeof(double));
  return g;
}

/* slope_from_dem (geodata.cpp:209-229) on model-order fp32 elevation widened
 * exactly to double; a NaN elevation marks a DEM nodata cell. */
ebo_grid* ebo_grid_terrain(int h, int w, const double* veg, const double* den, const float* elev,
                           double cellsize, double speed, double dir) {
  ebo_grid* g = grid_alloc(h, w);
  const double wd = ebo_wrap_angle(dir);
  for (int r = 0; r < h; ++r)
    for (int c = 0; c < w; ++c) {
      const size_t i = (size_t)r * w + c;
      g->speed[i] = speed;
      g->dir[i] = wd;
      g->veg[i] = clamp1(veg[i]);
      g->den[i] = clamp1(den[i]);
      for (int k = 0; k < 8; ++k) {
        const int nr = r + kDy[k], nc = c + kDx[k];
        if (nr < 0 || nr >= h || nc < 0 || nc >= w) continue;
        const double dist = cellsize * ((kDx[k] != 0 && kDy[k] != 0) ? SQRT2 : 1.0);
        if (isnan(elev[i]) || isnan(elev[(size_t)nr * w + nc])) continue; /* nodata: slope 0 (:214,220) */
        g->slope8[i * 8 + k] = atan(((double)elev[(size_t)nr * w + nc] - (double)elev[i]) / dist);
      }
    }
  return g;
}

void ebo_grid_free(ebo_grid* g) {
  if (!g) return;
  free(g->speed);
  free(g->dir);
  free(g->veg);
  free(g->den);
  free(g->slope8);
  free(g);
}

/* ---------------------------------------------------------------- kernel.hpp:21-78 */
static double kappa_wind(double speed, double direction, int k, const double* cfg) {
  const double align = cos(ebo_offset_angle(k) - direction) - 1.0;
  return exp(cfg[1] * speed) * exp((cfg[2] * speed) * align);
}

static double kappa_slope(double s, const double* cfg) { return exp(cfg[3] * s); }

static double source_of(const ebo_grid* g, size_t i, const double* cfg) {
  return (cfg[0] * (1.0 + g->veg[i])) * (1.0 + g->den[i]);
}

static double gamma_of(const ebo_grid* g, size_t i, const double* cfg) {
  return (cfg[4] * (1.0 + g->veg[i])) * (1.0 + g->den[i]);
}

/* potential(u, d) (kernel.hpp:37-45) */
static double potential(const ebo_grid* g, size_t u, int k, const double* cfg) {
  const double src = source_of(g, u, cfg);
  const double wind = kappa_wind(g->speed[u], g->dir[u], k, cfg);
  const double slope = kappa_slope(g->slope8[u * 8 + k], cfg);
  return (src * wind) * slope;
}

/* SpreadTables (engine.hpp:79-110): same products, so bitwise equal to potential(). */
void ebo_tables(const ebo_grid* g, const double* cfg, double* pot, double* gamma) {
  const size_t n = (size_t)g->h * g->w;
#pragma omp parallel for schedule(static) if (n > 65536)
  for (long long ii = 0; ii < (long long)n; ++ii) {
    const size_t i = (size_t)ii;
    const double src = source_of(g, i, cfg);
    gamma[i] = gamma_of(g, i, cfg);
    for (int k = 0; k < 8; ++k) {
      const double sf = kappa_slope(g->slope8[i * 8 + k], cfg);
      const double kw = kappa_wind(g->speed[i], g->dir[i], k, cfg);
      pot[i * 8 + k] = (src * kw) * sf;
    }
  }
}

/* arrival_intensity: fixed k order, skip OOB, skip zero weight (kernel.hpp:53-67) */
void ebo_intensity(const ebo_grid* g, const double* cfg, const uint8_t* fire, double* lambda,
                   double* p) {
  const int h = g->h, w = g->w;
  for (int r = 0; r < h; ++r)
    for (int c = 0; c < w; ++c) {
      double l = 0.0;
      for (int k = 0; k < 8; ++k) {
        const int ur = r - kDy[k], uc = c - kDx[k];
        if (ur < 0 || ur >= h || uc < 0 || uc >= w) continue;
        const size_t u = (size_t)ur * w + uc;
        if (fire[u] != 1) continue;
        l += 1.0 * potential(g, u, k, cfg);
      }
      const size_t v = (size_t)r * w + c;
      lambda[v] = l;
      p[v] = 1.0 - exp(-(gamma_of(g, v, cfg) * l)); /* kernel.hpp:71-78 */
    }
}

/* ---------------------------------------------------------------- engine.cpp:12-38 */
static uint8_t next_cell(int h, int w, const double* pot, const double* gamma, double pc,
                         uint64_t seed, uint64_t step, uint64_t stream, const uint8_t* in, int r,
                         int c) {
  const size_t i = (size_t)r * w + c;
  const uint8_t s = in[i];
  if (s == 2) return 2;
  const double u = ebo_rng_uniform(seed, step, stream, (uint64_t)i, DRAW_FIRE);
  if (s == 1) return u < pc ? 1 : 2;
  double l = 0.0;
  for (int k = 0; k < 8; ++k) {
    const int ur = r - kDy[k], uc = c - kDx[k];
    if (ur < 0 || ur >= h || uc < 0 || uc >= w) continue;
    const size_t uu = (size_t)ur * w + uc;
    if (in[uu] != 1) continue;
    l += 1.0 * pot[uu * 8 + k];
  }
  const double p = 1.0 - exp(-(gamma[i] * l));
  return u < p ? 1 : 0;
}

void ebo_step_tables(int h, int w, const double* pot, const double* gamma, double p_continue,
                     uint64_t seed, uint64_t step, uint64_t stream, const uint8_t* in, uint8_t* out) {
  for (int r = 0; r < h; ++r)
    for (int c = 0; c < w; ++c)
      out[(size_t)r * w + c] = next_cell(h, w, pot, gamma, p_continue, seed, step, stream, in, r, c);
}

void ebo_run(const ebo_grid* g, const double* cfg, uint64_t seed, uint64_t step0, uint64_t stream,
             int steps, uint8_t* state) {
  const size_t n = (size_t)g->h * g->w;
  double* pot = (double*)malloc(n * 8 * sizeof(double));
  double* gam = (double*)malloc(n * sizeof(double));
  uint8_t* tmp = (uint8_t*)malloc(n);
  ebo_tables(g, cfg, pot, gam);
  for (int t = 0; t < steps; ++t) {
    ebo_step_tables(g->h, g->w, pot, gam, cfg[5], seed, step0 + (uint64_t)t, stream, state, tmp);
    memcpy(state, tmp, n);
  }
  free(pot);
  free(gam);
  free(tmp);
}

double ebo_run_envs(ebo_grid* const* grids, int n_envs, const double* cfg, uint64_t seed,
                    const uint64_t* streams, int steps, uint8_t* states, int threads) {
  const size_t n = (size_t)grids[0]->h * grids[0]->w;
  if (threads > 0) omp_set_num_threads(threads);
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
#pragma omp parallel for schedule(dynamic, 1)
  for (int e = 0; e < n_envs; ++e) ebo_run(grids[e], cfg, seed, 0, streams[e], steps, states + e * n);
  clock_gettime(CLOCK_MONOTONIC, &t1);
  return (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
}

void ebo_counts(const uint8_t* fire, int n, int32_t* counts) {
  counts[0] = counts[1] = counts[2] = 0;
  for (int i = 0; i < n; ++i) counts[fire[i] > 2 ? 2 : fire[i]]++;
}

/* ---------------------------------------------------------------- rl_env.cpp */
int ebo_env_obs_size(const ebo_env_cfg* c) {
  const int side = 2 * c->window_radius + 1;
  return 3 * side * side + 3;
}

static int count_state(const uint8_t* f, int n, uint8_t v) {
  int k = 0;
  for (int i = 0; i < n; ++i) k += f[i] == v;
  return k;
}

/* reset (rl_env.cpp:125-145) */
void ebo_env_reset(const ebo_env_cfg* c, uint64_t seed, uint64_t stream, ebo_env_state* s,
                   uint8_t* fire) {
  const uint64_t n = (uint64_t)c->height * c->width;
  memset(fire, 0, n);
  uint64_t counter = 0;
  for (int placed = 0; placed < c->ignition_count;) {
    const uint64_t cell = ebo_rng_below(seed, 0, stream, counter++, DRAW_SETUP, n);
    if (fire[cell] == 1) continue;
    fire[cell] = 1;
    ++placed;
  }
  const uint64_t a = ebo_rng_below(seed, 0, stream, counter++, DRAW_SETUP, n);
  s->agent_row = (int)(a / (uint64_t)c->width);
  s->agent_col = (int)(a % (uint64_t)c->width);
  s->water = c->water_capacity;
  s->step = 0;
  s->seed = seed;
  s->stream = stream;
  s->done = count_state(fire, (int)n, 1) == 0;
}

/* observe (rl_env.cpp:147-170) */
void ebo_env_observe(const ebo_env_cfg* c, const ebo_env_state* s, const uint8_t* fire,
                     double* obs) {
  const int r = c->window_radius;
  memset(obs, 0, sizeof(double) * (size_t)ebo_env_obs_size(c));
  size_t at = 0;
  for (int dy = r; dy >= -r; --dy)
    for (int dx = -r; dx <= r; ++dx) {
      const int row = s->agent_row + dy, col = s->agent_col + dx;
      if (row >= 0 && row < c->height && col >= 0 && col < c->width)
        obs[at + fire[row * c->width + col]] = 1.0;
      at += 3;
    }
  obs[at++] = (double)s->water / c->water_capacity;
  obs[at++] = c->height > 1 ? (double)s->agent_row / (c->height - 1) : 0.0;
  obs[at++] = c->width > 1 ? (double)s->agent_col / (c->width - 1) : 0.0;
}

/* step (rl_env.cpp:172-210) on the flat terrain of the config (rl_env.cpp:99-105) */
int ebo_env_step(const ebo_env_cfg* c, const ebo_env_state* s, const uint8_t* fire, int action,
                 ebo_env_state* so, uint8_t* fo, double* reward, double* obs) {
  if (s->done) return -1;
  if (action < 0 || action >= 10) return -2;
  const int h = c->height, w = c->width, n = h * w;
  *so = *s;
  uint8_t* cur = (uint8_t*)malloc((size_t)n);
  memcpy(cur, fire, (size_t)n);
  const int move = action / 2, open = action % 2;
  switch (move) {
    case 0: so->agent_row = so->agent_row + 1 < h - 1 ? so->agent_row + 1 : h - 1; break;
    case 1: so->agent_row = so->agent_row - 1 > 0 ? so->agent_row - 1 : 0; break;
    case 2: so->agent_col = so->agent_col + 1 < w - 1 ? so->agent_col + 1 : w - 1; break;
    case 3: so->agent_col = so->agent_col - 1 > 0 ? so->agent_col - 1 : 0; break;
    default: break;
  }
  if (open && so->water > 0) {
    const int a = so->agent_row * w + so->agent_col;
    const int on_fire = cur[a] == 1;
    if (on_fire) cur[a] = 2;
    if (on_fire || c->waste_water) so->water -= 1;
  }
  /* flat terrain tables */
  double* pot = (double*)malloc(sizeof(double) * 8 * (size_t)n);
  double* gam = (double*)malloc(sizeof(double) * (size_t)n);
  double* zero8 = (double*)calloc((size_t)n * 8, sizeof(double));
  double *sp = (double*)malloc(sizeof(double) * n), *dr = (double*)malloc(sizeof(double) * n);
  double *vg = (double*)malloc(sizeof(double) * n), *dn = (double*)malloc(sizeof(double) * n);
  for (int i = 0; i < n; ++i) {
    sp[i] = c->wind_speed;
    dr[i] = c->wind_direction;
    vg[i] = c->fuel_veg;
    dn[i] = c->fuel_den;
  }
  ebo_grid* g = ebo_grid_layers(h, w, sp, dr, vg, dn, zero8);
  ebo_tables(g, c->spread, pot, gam);
  ebo_step_tables(h, w, pot, gam, c->spread[5], s->seed, (uint64_t)s->step, s->stream, cur, fo);
  so->step = s->step + 1;
  const int burning = count_state(fo, n, 1);
  double rw = -c->burn_penalty * burning;
  if (burning == 0 && count_state(fo, n, 0) != n) rw += 10.0; /* kTerminalBonus */
  so->done = burning == 0 || so->step >= c->max_episode_steps;
  *reward = rw;
  if (obs) ebo_env_observe(c, so, fo, obs);
  ebo_grid_free(g);
  free(pot), free(gam), free(zero8), free(sp), free(dr), free(vg), free(dn), free(cur);
  return 0;
}

/* random_policy (rl_env.cpp:237-239) */
int ebo_random_policy(uint64_t seed, uint64_t step, uint64_t stream) {
  return (int)ebo_rng_below(seed, step, stream, 0, DRAW_POLICY, 10);
}

/* ---------------------------------------------------------------- tanker (C2) */
static uint64_t tanker_stream(uint32_t env_id, uint32_t episode) {
  return ((uint64_t)episode << 32) | env_id;
}

static int burnable(const ebo_grid* g, size_t i) {
  return (1.0 + g->veg[i]) * (1.0 + g->den[i]) > 0.0;
}

void ebo_tanker_reset(const ebo_grid* g, const ebo_tanker_cfg* tc, uint64_t seed, uint32_t env_id,
                      uint32_t episode, ebo_tanker_state* s, uint8_t* fire, uint8_t* wet) {
  const uint64_t n = (uint64_t)g->h * g->w;
  const uint64_t stream = tanker_stream(env_id, episode);
  memset(fire, 0, n);
  memset(wet, 0, n);
  uint64_t counter = 0;
  const uint64_t max_draws = 64 * n;
  for (int placed = 0; placed < tc->ignitions && counter < max_draws;) {
    const uint64_t cell = ebo_rng_below(seed, 0, stream, counter++, DRAW_SETUP, n);
    if (fire[cell] == 1 || !burnable(g, cell)) continue;
    fire[cell] = 1;
    ++placed;
  }
  s->step = 0;
  s->episode = episode;
  s->done = count_state(fire, (int)n, 1) == 0;
}

int ebo_tanker_policy(uint64_t seed, uint32_t env_id, const ebo_tanker_state* s, int n_cells) {
  return (int)ebo_rng_below(seed, (uint64_t)s->step, tanker_stream(env_id, s->episode), 0,
                            DRAW_POLICY, (uint64_t)n_cells);
}

void ebo_tanker_step(const ebo_grid* g, const double* pot, const double* gamma, double p_continue,
                     const ebo_tanker_cfg* tc, uint64_t seed, uint32_t env_id, int action,
                     ebo_tanker_state* s, uint8_t* fire, uint8_t* wet, float* reward,
                     uint8_t* done) {
  const int h = g->h, w = g->w, n = h * w;
  const int ar = action / w, ac = action % w;
  /* 1) drop: extinguish (Burning -> Burned) and wet (Unburned stays, never ignites) a 3x3 patch */
  for (int dr = -1; dr <= 1; ++dr)
    for (int dc = -1; dc <= 1; ++dc) {
      const int r = ar + dr, c = ac + dc;
      if (r < 0 || r >= h || c < 0 || c >= w) continue;
      const int i = r * w + c;
      if (fire[i] == 1) fire[i] = 2;
      else if (fire[i] == 0) wet[i] = 1;
    }
  /* 2) fire step with key {seed, step, stream}; wet cells are not ignitable */
  const uint64_t stream = tanker_stream(env_id, s->episode);
  uint8_t* nx = (uint8_t*)malloc((size_t)n);
  int newly = 0;
  for (int r = 0; r < h; ++r)
    for (int c = 0; c < w; ++c) {
      const int i = r * w + c;
      if (fire[i] == 0 && wet[i]) {
        nx[i] = 0;
        continue;
      }
      nx[i] = next_cell(h, w, pot, gamma, p_continue, seed, (uint64_t)s->step, stream, fire, r, c);
      newly += fire[i] == 0 && nx[i] == 1;
    }
  memcpy(fire, nx, (size_t)n);
  free(nx);
  s->step += 1;
  const int burning = count_state(fire, n, 1);
  *reward = -(float)newly;
  s->done = burning == 0 || s->step >= tc->max_steps;
  *done = (uint8_t)s->done;
  if (s->done && tc->autoreset) ebo_tanker_reset(g, tc, seed, env_id, s->episode + 1, s, fire, wet);
}

/* ---------------------------------------------------------------- engine.hpp:147-175 */
void ebo_det_step_tables(int h, int w, const double* pot, const double* gamma, double pc,
                         const double* un, const double* burn, const double* bd, double* un_o,
                         double* burn_o, double* bd_o) {
  for (int r = 0; r < h; ++r)
    for (int c = 0; c < w; ++c) {
      const size_t i = (size_t)r * w + c;
      double l = 0.0;
      for (int k = 0; k < 8; ++k) {
        const int ur = r - kDy[k], uc = c - kDx[k];
        if (ur < 0 || ur >= h || uc < 0 || uc >= w) continue;
        const size_t u = (size_t)ur * w + uc;
        const double wgt = burn[u];
        if (wgt == 0.0) continue;
        l += wgt * pot[u * 8 + k];
      }
      const double p_ig = 1.0 - exp(-(gamma[i] * l));
      const double newly = un[i] * p_ig;
      const double continuing = burn[i] * pc;
      const double burned_now = burn[i] * (1.0 - pc);
      burn_o[i] = newly + continuing;
      un_o[i] = un[i] - newly;
      bd_o[i] = bd[i] + burned_now;
    }
}

/* ---------------------------------------------------------------- dual.hpp:21-200 (N = 6)
 * Forward-mode dual numbers with the reference's exact per-operation formulas, used to
 * restate run_deterministic<Dual<6>> + loss (engine.hpp:147-245, calibrate.hpp:86-146):
 * the C4 gradient oracle. */
typedef struct { double v, g[6]; } dual6;

static dual6 d_const(double x) { dual6 r; r.v = x; for (int i = 0; i < 6; ++i) r.g[i] = 0.0; return r; }
static dual6 d_add(dual6 a, dual6 b) { a.v += b.v; for (int i = 0; i < 6; ++i) a.g[i] += b.g[i]; return a; }
static dual6 d_sub(dual6 a, dual6 b) { a.v -= b.v; for (int i = 0; i < 6; ++i) a.g[i] -= b.g[i]; return a; }
static dual6 d_mul(dual6 a, dual6 b) {  /* operator*= (dual.hpp:57-61): grads first, then value */
  for (int i = 0; i < 6; ++i) a.g[i] = a.g[i] * b.v + a.v * b.g[i];
  a.v *= b.v;
  return a;
}
static dual6 d_muls(dual6 a, double b) { a.v *= b; for (int i = 0; i < 6; ++i) a.g[i] *= b; return a; }
static dual6 d_divs(dual6 a, double b) { a.v /= b; for (int i = 0; i < 6; ++i) a.g[i] /= b; return a; }
static dual6 d_neg(dual6 a) { a.v = -a.v; for (int i = 0; i < 6; ++i) a.g[i] = -a.g[i]; return a; }
static dual6 d_rsub(double a, dual6 b) {  /* double - Dual (dual.hpp:101-106) */
  dual6 r; r.v = a - b.v; for (int i = 0; i < 6; ++i) r.g[i] = -b.g[i]; return r;
}
static dual6 d_subs(dual6 a, double b) { a.v -= b; return a; }
static dual6 d_exp(dual6 a) {
  dual6 r; r.v = exp(a.v); for (int i = 0; i < 6; ++i) r.g[i] = r.v * a.g[i]; return r;
}
static dual6 d_log(dual6 a) {
  dual6 r; r.v = log(a.v); for (int i = 0; i < 6; ++i) r.g[i] = a.g[i] / a.v; return r;
}

/* Loss + d loss / d theta after `steps` deterministic steps from a discrete layer;
 * theta = the six SimConfig fields lifted as parameters 0..5 (ParamIndex order,
 * calibrate.hpp:21-28).  loss = bce_w * BCE + mse_w * MSE(avgpool) (calibrate.hpp:120-146). */
/* run_deterministic<Dual<6>> from a continuous initial state (lift_state: constant duals) with
 * config P[0..5], then loss; returns the Dual loss. */
static dual6 det_loss_dual(const ebo_grid* g, const dual6* P, int steps, const double* un0,
                           const double* bu0, const double* bd0, const double* mask, double bce_w,
                           double mse_w, int pool);

void ebo_det_loss_grad(const ebo_grid* g, const double* cfg, int steps, const uint8_t* fire0,
                       const double* mask, double bce_w, double mse_w, int pool, double* loss_out,
                       double* grad6) {
  const size_t n = (size_t)g->h * g->w;
  dual6 P[6];
  for (int i = 0; i < 6; ++i) { P[i] = d_const(cfg[i]); P[i].g[i] = 1.0; }
  double* s0 = (double*)malloc(3 * n * sizeof(double));
  for (size_t i = 0; i < n; ++i) {  /* state_from_fire (engine.cpp:42-52) */
    s0[i] = fire0[i] == 0 ? 1.0 : 0.0;
    s0[n + i] = fire0[i] == 1 ? 1.0 : 0.0;
    s0[2 * n + i] = fire0[i] == 2 ? 1.0 : 0.0;
  }
  const dual6 l = det_loss_dual(g, P, steps, s0, s0 + n, s0 + 2 * n, mask, bce_w, mse_w, pool);
  *loss_out = l.v;
  for (int i = 0; i < 6; ++i) grad6[i] = l.g[i];
  free(s0);
}

static dual6 det_loss_dual(const ebo_grid* g, const dual6* P, int steps, const double* un0,
                           const double* bu0, const double* bd0, const double* mask, double bce_w,
                           double mse_w, int pool) {
  const int h = g->h, w = g->w;
  const size_t n = (size_t)h * w;
  /* SpreadTables<Dual<6>> (engine.hpp:79-110) */
  dual6* pot = (dual6*)malloc(n * 8 * sizeof(dual6));
  dual6* gam = (dual6*)malloc(n * sizeof(dual6));
  for (size_t i = 0; i < n; ++i) {
    const dual6 source = d_muls(d_muls(P[0], 1.0 + g->veg[i]), 1.0 + g->den[i]);
    gam[i] = d_muls(d_muls(P[4], 1.0 + g->veg[i]), 1.0 + g->den[i]);
    for (int k = 0; k < 8; ++k) {
      const dual6 sf = d_exp(d_muls(P[3], g->slope8[i * 8 + k]));
      const double align = cos(ebo_offset_angle(k) - g->dir[i]) - 1.0;
      const dual6 kw = d_mul(d_exp(d_muls(P[1], g->speed[i])),
                             d_exp(d_muls(d_muls(P[2], g->speed[i]), align)));
      pot[i * 8 + k] = d_mul(d_mul(source, kw), sf);
    }
  }
  dual6 *un = (dual6*)malloc(n * sizeof(dual6)), *bu = (dual6*)malloc(n * sizeof(dual6)),
        *bd = (dual6*)malloc(n * sizeof(dual6));
  dual6 *un2 = (dual6*)malloc(n * sizeof(dual6)), *bu2 = (dual6*)malloc(n * sizeof(dual6)),
        *bd2 = (dual6*)malloc(n * sizeof(dual6));
  for (size_t i = 0; i < n; ++i) {  /* lift_state (engine.hpp:46-57) */
    un[i] = d_const(un0[i]);
    bu[i] = d_const(bu0[i]);
    bd[i] = d_const(bd0[i]);
  }
  for (int t = 0; t < steps; ++t) {
    for (int r = 0; r < h; ++r)
      for (int c = 0; c < w; ++c) {
        const size_t i = (size_t)r * w + c;
        dual6 lam = d_const(0.0);
        for (int k = 0; k < 8; ++k) {
          const int ur = r - kDy[k], uc = c - kDx[k];
          if (ur < 0 || ur >= h || uc < 0 || uc >= w) continue;
          const size_t u = (size_t)ur * w + uc;
          if (bu[u].v == 0.0) continue;
          lam = d_add(lam, d_mul(bu[u], pot[u * 8 + k]));
        }
        const dual6 p_ig = d_rsub(1.0, d_exp(d_neg(d_mul(gam[i], lam))));
        const dual6 newly = d_mul(un[i], p_ig);
        const dual6 continuing = d_mul(bu[i], P[5]);
        const dual6 burned_now = d_mul(bu[i], d_rsub(1.0, P[5]));
        bu2[i] = d_add(newly, continuing);
        un2[i] = d_sub(un[i], newly);
        bd2[i] = d_add(bd[i], burned_now);
      }
    dual6* tmp;
    tmp = un; un = un2; un2 = tmp;
    tmp = bu; bu = bu2; bu2 = tmp;
    tmp = bd; bd = bd2; bd2 = tmp;
  }
  /* pred = p_burn + p_bd (calibrate.hpp:86-91) */
  dual6* pred = un2;
  for (size_t i = 0; i < n; ++i) pred[i] = d_add(bu[i], bd[i]);
  const double eps = 1e-6;  /* LossConfig::bce_epsilon */
  dual6 bce = d_const(0.0);
  for (size_t i = 0; i < n; ++i) {
    dual6 p = pred[i];
    p = p.v >= eps ? p : d_const(eps);                /* max(pred, eps): ties keep pred */
    p = p.v <= 1.0 - eps ? p : d_const(1.0 - eps);    /* min(., 1-eps) */
    const double m = mask[i];
    bce = d_add(bce, d_neg(d_add(d_muls(d_log(p), m), d_muls(d_log(d_rsub(1.0, p)), 1.0 - m))));
  }
  bce = d_divs(bce, (double)n);
  /* avgpool (calibrate.hpp:95-115) of pred and mask, then MSE */
  const int oh = (h + pool - 1) / pool, ow = (w + pool - 1) / pool;
  dual6 mse = d_const(0.0);
  for (int pr = 0; pr < oh; ++pr)
    for (int pc = 0; pc < ow; ++pc) {
      dual6 s = d_const(0.0);
      double sm = 0.0;
      int count = 0;
      for (int r = pr * pool; r < (pr + 1) * pool && r < h; ++r)
        for (int c = pc * pool; c < (pc + 1) * pool && c < w; ++c) {
          s = d_add(s, pred[(size_t)r * w + c]);
          sm += mask[(size_t)r * w + c];
          ++count;
        }
      const dual6 pp = d_divs(s, (double)count);
      const double pm = sm / (double)count;
      const dual6 d = d_subs(pp, pm);
      mse = d_add(mse, d_mul(d, d));
    }
  mse = d_divs(mse, (double)(oh * ow));
  const dual6 l = d_add(d_muls(bce, bce_w), d_muls(mse, mse_w));
  free(pot), free(gam), free(un), free(bu), free(bd), free(un2), free(bu2), free(bd2);
  return l;
}

/* ---------------------------------------------------------------- calibrate.cpp / .hpp */
static dual6 d_addl(double a, dual6 b) { b.v += a; return b; } /* double + Dual (dual.hpp:90) */
static dual6 d_div(dual6 a, dual6 b) {                          /* operator/= (dual.hpp:62-68) */
  for (int i = 0; i < 6; ++i) a.g[i] = (a.g[i] * b.v - a.v * b.g[i]) / (b.v * b.v);
  a.v /= b.v;
  return a;
}
static dual6 softplus6(dual6 x) { /* calibrate.hpp:44-49 */
  if (x.v > 0.0) return d_add(x, d_log(d_addl(1.0, d_exp(d_neg(x)))));
  return d_log(d_addl(1.0, d_exp(x)));
}
static dual6 logistic6(dual6 x) { /* calibrate.hpp:51-57 */
  if (x.v >= 0.0) return d_div(d_const(1.0), d_addl(1.0, d_exp(d_neg(x))));
  const dual6 e = d_exp(x);
  return d_div(e, d_addl(1.0, e));
}

/* calibrate (calibrate.cpp:104-167) with ThetaTransform (calibrate.hpp:59-68, calibrate.cpp:35-55)
 * and adam_step (calibrate.cpp:84-102); returns 0, -1 on a non-finite loss or gradient
 * (NumericalError), -2 on an init_theta outside the transform's domain (invalid_argument). */
int ebo_calibrate(const ebo_grid* g, const double* un0, const double* bu0, const double* bd0,
                  const double* mask, int horizon, double bce_w, double mse_w, int pool,
                  int iterations, const double* init_theta, const int* optimize, double lr,
                  double* loss_hist, double* theta_hist, double* best_theta, double* best_loss) {
  double u[6];
  for (int i = 0; i < 6; ++i) u[i] = init_theta[i];
  const int pos[2] = {0, 4};
  for (int j = 0; j < 2; ++j) { /* inverse_softplus */
    const double y = init_theta[pos[j]];
    if (!(y > 0.0)) return -2;
    u[pos[j]] = y > 20.0 ? y : log(expm1(y));
  }
  {
    const double p = init_theta[5]; /* logit */
    if (!(p > 0.0 && p < 1.0)) return -2;
    u[5] = log(p / (1.0 - p));
  }
  double m[6] = {0}, v[6] = {0};
  int t_adam = 0;
  const double beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
  *best_loss = INFINITY;
  for (int iter = 0; iter <= iterations; ++iter) {
    dual6 ud[6], th[6];
    for (int i = 0; i < 6; ++i) {
      ud[i] = d_const(u[i]);
      if (optimize[i]) ud[i].g[i] = 1.0;
    }
    th[0] = softplus6(ud[0]);
    th[1] = ud[1];
    th[2] = ud[2];
    th[3] = ud[3];
    th[4] = softplus6(ud[4]);
    th[5] = logistic6(ud[5]);
    const dual6 l = det_loss_dual(g, th, horizon, un0, bu0, bd0, mask, bce_w, mse_w, pool);
    if (!isfinite(l.v)) return -1;
    loss_hist[iter] = l.v;
    for (int i = 0; i < 6; ++i) theta_hist[iter * 6 + i] = th[i].v;
    if (l.v < *best_loss) {
      *best_loss = l.v;
      for (int i = 0; i < 6; ++i) best_theta[i] = th[i].v;
    }
    if (iter == iterations) break;
    for (int i = 0; i < 6; ++i)
      if (!isfinite(l.g[i])) return -1;
    t_adam += 1;
    const double bc1 = 1.0 - pow(beta1, t_adam), bc2 = 1.0 - pow(beta2, t_adam);
    for (int i = 0; i < 6; ++i) {
      m[i] = beta1 * m[i] + (1.0 - beta1) * l.g[i];
      v[i] = beta2 * v[i] + (1.0 - beta2) * l.g[i] * l.g[i];
      const double m_hat = m[i] / bc1, v_hat = v[i] / bc2;
      u[i] = u[i] - lr * m_hat / (sqrt(v_hat) + eps);
    }
  }
  return 0;
}

/* Deterministic forward from a discrete layer, double (run_deterministic<double>). */
void ebo_det_run(const ebo_grid* g, const double* cfg, int steps, double* un, double* burn,
                 double* bd) {
  const int h = g->h, w = g->w;
  const size_t n = (size_t)h * w;
  double* pot = (double*)malloc(n * 8 * sizeof(double));
  double* gam = (double*)malloc(n * sizeof(double));
  double *a = (double*)malloc(n * sizeof(double)), *b = (double*)malloc(n * sizeof(double)),
         *c = (double*)malloc(n * sizeof(double));
  ebo_tables(g, cfg, pot, gam);
  for (int t = 0; t < steps; ++t) {
    ebo_det_step_tables(h, w, pot, gam, cfg[5], un, burn, bd, a, b, c);
    memcpy(un, a, n * sizeof(double));
    memcpy(burn, b, n * sizeof(double));
    memcpy(bd, c, n * sizeof(double));
  }
  free(pot), free(gam), free(a), free(b), free(c);
}

/* ---- snapshot.cpp:55-70 serialize_snapshot ------------------------------------------------- */
long ebo_snapshot_text(int h, int w, const uint8_t* fire, uint64_t step, int ar, int ac, int water, char* out,
                       long cap) {
  char hdr[96], ag[96];
  const int hl = snprintf(hdr, sizeof hdr, "emberline-snapshot v1 %d %d %llu\n", h, w, (unsigned long long)step);
  const int al = ar >= 0 ? snprintf(ag, sizeof ag, "agent %d %d %d\n", ar, ac, water) : 0;
  const long total = hl + (long)h * (w + 1) + al;
  long o = 0;
#define EBO_PUT(ch) do { if (out && o < cap) out[o] = (ch); ++o; } while (0)
  for (int k = 0; k < hl; ++k) EBO_PUT(hdr[k]);
  for (int row = h - 1; row >= 0; --row) { /* state_char, snapshot.cpp:14-21 */
    for (int col = 0; col < w; ++col) {
      const uint8_t v = fire[(size_t)row * w + col];
      EBO_PUT(v == 0 ? 'U' : v == 1 ? 'B' : v == 2 ? 'X' : '?');
    }
    EBO_PUT('\n');
  }
  for (int k = 0; k < al; ++k) EBO_PUT(ag[k]);
#undef EBO_PUT
  return total;
}

/* ---------------------------------------------------------------- synthetic C1 inputs
 * The benchmark's own input generator (not a reference function), restated
 * here so the CPU arms of bench.py build their inputs without the product library.  Pinned
 * bit-for-bit against ebl_synth_terrain / ebl_synth_ignitions by tests/test_oracle_pin.py.
 * Lattice values and wind are keyed by the reference RNG (rng.hpp:38-58) with draw domain
 * kDrawSynthesis = 3; ignitions by kDrawEnvSetup = 1 (rng.hpp:22-25).  The palette is
 * default_worldcover_table (geodata.cpp:305-319). */
enum { DRAW_SYNTH = 3 };

static void noise2d(uint64_t seed, uint64_t layer, uint64_t stream, int h, int w, int octaves,
                    int period, double* out) {
  memset(out, 0, sizeof(double) * (size_t)h * w);
  double amp = 1.0;
  for (int o = 0; o < octaves; ++o) {
    int L = period >> o;
    if (L < 1) L = 1;
    const int gh = h / L + 2, gw = w / L + 2;
    double* lat = (double*)malloc(sizeof(double) * (size_t)gh * gw);
    for (size_t i = 0; i < (size_t)gh * gw; ++i)
      lat[i] = ebo_rng_uniform(seed, layer + (uint64_t)o, stream, i, DRAW_SYNTH);
    for (int r = 0; r < h; ++r) {
      const int gy = r / L;
      double ty = (r - gy * L + 0.5) / L;
      ty = ty * ty * (3.0 - 2.0 * ty); /* smoothstep */
      for (int c = 0; c < w; ++c) {
        const int gx = c / L;
        double tx = (c - gx * L + 0.5) / L;
        tx = tx * tx * (3.0 - 2.0 * tx);
        const double* a = lat + (size_t)gy * gw + gx;
        const double* b = a + gw;
        const double s0 = a[0] + (a[1] - a[0]) * tx;
        const double s1 = b[0] + (b[1] - b[0]) * tx;
        out[(size_t)r * w + c] += amp * (s0 + (s1 - s0) * ty);
      }
    }
    free(lat);
    amp *= 0.5;
  }
}

static void minmax(const double* v, size_t n, double* lo, double* hi) {
  *lo = *hi = v[0];
  for (size_t i = 0; i < n; ++i) {
    if (v[i] < *lo) *lo = v[i];
    if (v[i] > *hi) *hi = v[i];
  }
}

#define SYNTH_BINS 4096
static int imin(int a, int b) { return a < b ? a : b; }
static int imax(int a, int b) { return a > b ? a : b; }

static void synth_env(uint64_t seed, uint64_t stream, int h, int w, double elev_max, uint8_t* cls,
                      float* elev, double* scratch) {
  const size_t n = (size_t)h * w;
  double lo, hi;
  /* landcover: 4 octaves, period clamp(min(h,w)/4, 4, 64), 11 equal-count classes by a
   * 4096-bin histogram of the noise */
  noise2d(seed, 1000, stream, h, w, 4, imin(64, imax(4, imin(h, w) / 4)), scratch);
  minmax(scratch, n, &lo, &hi);
  const double scale = hi > lo ? SYNTH_BINS / (hi - lo) : 0.0;
  static __thread uint64_t hist[SYNTH_BINS];
  memset(hist, 0, sizeof hist);
  for (size_t i = 0; i < n; ++i) hist[imin(SYNTH_BINS - 1, (int)((scratch[i] - lo) * scale))]++;
  int cut[10], j = 0;
  uint64_t acc = 0;
  for (int b = 0; b < SYNTH_BINS && j < 10; ++b) {
    acc += hist[b];
    while (j < 10 && acc * 11 >= (uint64_t)(j + 1) * n) cut[j++] = b + 1;
  }
  while (j < 10) cut[j++] = SYNTH_BINS;
  for (size_t i = 0; i < n; ++i) {
    const int b = imin(SYNTH_BINS - 1, (int)((scratch[i] - lo) * scale));
    int k = 0;
    while (k < 10 && b >= cut[k]) ++k;
    cls[i] = (uint8_t)k;
  }
  /* elevation: 6 octaves, period clamp(min(h,w)/2, 8, 128), affinely mapped to [0, elev_max] */
  noise2d(seed, 2000, stream, h, w, 6, imin(128, imax(8, imin(h, w) / 2)), scratch);
  minmax(scratch, n, &lo, &hi);
  const double es = hi > lo ? elev_max / (hi - lo) : 0.0;
  for (size_t i = 0; i < n; ++i) elev[i] = (float)((scratch[i] - lo) * es);
}

void ebo_synth_terrain(uint64_t seed, uint32_t env_id0, int n_envs, int h, int w, double elev_max,
                       double wind_max, uint8_t* fuel_class, float* elevation, double* wind_speed,
                       double* wind_direction) {
  const size_t n = (size_t)h * w;
#pragma omp parallel
  {
    double* scratch = (double*)malloc(sizeof(double) * n);
#pragma omp for schedule(dynamic, 1)
    for (int e = 0; e < n_envs; ++e) {
      const uint64_t stream = (uint64_t)env_id0 + (uint64_t)e;
      synth_env(seed, stream, h, w, elev_max, fuel_class + e * n, elevation + e * n, scratch);
      if (wind_speed) wind_speed[e] = wind_max * ebo_rng_uniform(seed, 3000, stream, 0, DRAW_SYNTH);
      if (wind_direction) wind_direction[e] = TWO_PI * ebo_rng_uniform(seed, 3000, stream, 1, DRAW_SYNTH);
    }
    free(scratch);
  }
}

void ebo_worldcover_palette(int32_t* codes, double* veg, double* den) {
  /* default_worldcover_table (geodata.cpp:305-319), dense in code order */
  static const int32_t kc[11] = {10, 20, 30, 40, 50, 60, 70, 80, 90, 95, 100};
  static const double kv[11] = {0.4, 0.25, 0.15, 0.0, -0.8, -0.7, -1.0, -1.0, -0.4, -0.2, -0.3};
  static const double kd[11] = {0.3, 0.1, -0.1, -0.2, -0.8, -0.6, -1.0, -1.0, -0.3, -0.1, -0.4};
  for (int i = 0; i < 11; ++i) {
    if (codes) codes[i] = kc[i];
    if (veg) veg[i] = kv[i];
    if (den) den[i] = kd[i];
  }
}

int ebo_synth_ignitions(uint64_t seed, uint32_t env_id0, int n_envs, int h, int w,
                        const uint8_t* fuel_class, const double* class_veg, const double* class_den,
                        int count, uint8_t* states) {
  const uint64_t n = (uint64_t)h * w;
  int total = 0;
#pragma omp parallel for schedule(static) reduction(+ : total)
  for (int e = 0; e < n_envs; ++e) {
    uint8_t* st = states + e * n;
    const uint8_t* fc = fuel_class + e * n;
    memset(st, 0, n);
    const uint64_t stream = (uint64_t)env_id0 + (uint64_t)e;
    int placed = 0;
    /* uniform cells until `count` distinct burnable ones ((1+veg)(1+den) > 0, veg/den clamped
     * as FuelField does, grid.cpp:75-76); at most 64 n draws */
    for (uint64_t k = 0; placed < count && k < 64 * n; ++k) {
      const uint64_t cell = ebo_rng_below(seed, 0, stream, k, DRAW_SETUP, n);
      const double v = clamp1(class_veg[fc[cell]]), d = clamp1(class_den[fc[cell]]);
      if (st[cell] == 1 || !((1.0 + v) * (1.0 + d) > 0.0)) continue;
      st[cell] = 1;
      ++placed;
    }
    total += placed;
  }
  return total;
}

/* ---------------------------------------------------------------- CPU-baseline harnesses
 * C2: the tanker step (ebo_tanker_step) over n envs, OpenMP over envs, random device policy
 * (ebo_tanker_policy), auto-reset.  Tables per env are built before the clock starts (the
 * reference's FireSuppressionEnv likewise holds its tables for the whole episode).  Env e has id
 * env_ids[e] (null: env_id0 + e).  Returns the wall seconds of `steps` steps of every env;
 * optional outputs: *reward_sum (all envs), per env the final fire / wet layers [n][h*w], the
 * reward sum and the number of finished episodes. */
double ebo_tanker_run_envs(ebo_grid* const* grids, int n_envs, const double* cfg,
                           const ebo_tanker_cfg* tc, uint64_t seed, uint32_t env_id0,
                           const uint32_t* env_ids, int steps, int threads, double* reward_sum,
                           uint8_t* fire_out, uint8_t* wet_out, double* env_reward, int32_t* env_episodes) {
  if (threads > 0) omp_set_num_threads(threads);
  const size_t n = (size_t)grids[0]->h * grids[0]->w;
  double** pots = (double**)malloc(sizeof(double*) * n_envs);
  double** gams = (double**)malloc(sizeof(double*) * n_envs);
  uint8_t* fire = fire_out ? fire_out : (uint8_t*)malloc(n * n_envs);
  uint8_t* wet = wet_out ? wet_out : (uint8_t*)malloc(n * n_envs);
  ebo_tanker_state* st = (ebo_tanker_state*)malloc(sizeof(ebo_tanker_state) * n_envs);
#pragma omp parallel for schedule(dynamic, 4)
  for (int e = 0; e < n_envs; ++e) {
    const uint32_t id = env_ids ? env_ids[e] : env_id0 + (uint32_t)e;
    pots[e] = (double*)malloc(sizeof(double) * n * 8);
    gams[e] = (double*)malloc(sizeof(double) * n);
    ebo_tables(grids[e], cfg, pots[e], gams[e]);
    ebo_tanker_reset(grids[e], tc, seed, id, 0, st + e, fire + e * n, wet + e * n);
  }
  double total = 0.0;
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : total)
  for (int e = 0; e < n_envs; ++e) {
    const uint32_t id = env_ids ? env_ids[e] : env_id0 + (uint32_t)e;
    double mine = 0.0;
    int32_t eps = 0;
    for (int t = 0; t < steps; ++t) {
      float rw;
      uint8_t dn;
      const int a = ebo_tanker_policy(seed, id, st + e, (int)n);
      ebo_tanker_step(grids[e], pots[e], gams[e], cfg[5], tc, seed, id, a, st + e, fire + e * n,
                      wet + e * n, &rw, &dn);
      mine += rw;
      eps += dn;
    }
    if (env_reward) env_reward[e] = mine;
    if (env_episodes) env_episodes[e] = eps;
    total += mine;
  }
  clock_gettime(CLOCK_MONOTONIC, &t1);
  for (int e = 0; e < n_envs; ++e) {
    free(pots[e]);
    free(gams[e]);
  }
  free(pots);
  free(gams);
  if (!fire_out) free(fire);
  if (!wet_out) free(wet);
  free(st);
  if (reward_sum) *reward_sum = total;
  return (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
}
