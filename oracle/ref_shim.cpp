// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI shim over the UNMODIFIED reference sources under /root/reference/proj.
// oracle/Makefile compiles those sources together with this file into
// oracle/_ref/libebl_ref.so with -Demberline=ebl_ref, so the reference's
// own code (engine.cpp, geodata.cpp, rl_env.cpp, calibrate.cpp, kernel.hpp,
// reference.hpp, dual.hpp) is what answers every call below.  The shim only
// marshals flat arrays into the reference's types and back; it contains no
// simulation logic of its own.  Consumers: tests/ (parity + pinning of
// oracle/ember_oracle.c), tests/golden/make_golden.py, and bench.py's
// `--impl reference` / cpu_baseline leg.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include <omp.h>

#include "emberline/calibrate.hpp"
#include "emberline/engine.hpp"
#include "emberline/geodata.hpp"
#include "emberline/kernel.hpp"
#include "emberline/reference.hpp"
#include "emberline/rl_env.hpp"
#include "emberline/rng.hpp"
#include "emberline/snapshot.hpp"

namespace R = ::emberline;  // expands to ::ebl_ref under -Demberline=ebl_ref

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  return -1;
}

R::SimConfig cfg_of(const double* c) {
  R::SimConfig cfg;
  cfg.p_base = c[0];
  cfg.alpha_w1 = c[1];
  cfg.alpha_w2 = c[2];
  cfg.alpha_s = c[3];
  cfg.alpha_gamma = c[4];
  cfg.p_continue = c[5];
  return cfg;
}

R::FireLayer layer_of(int h, int w, const std::uint8_t* s) {
  R::FireLayer f(h, w);
  for (int i = 0; i < h * w; ++i) f[i] = static_cast<R::FireState>(s[i]);
  return f;
}

void unlayer(const R::FireLayer& f, std::uint8_t* out) {
  for (int i = 0; i < f.size(); ++i) out[i] = static_cast<std::uint8_t>(f[i]);
}

R::Grid<double> grid_of(int h, int w, const double* v) {
  R::Grid<double> g(h, w);
  for (int i = 0; i < h * w; ++i) g[i] = v[i];
  return g;
}

// Model-order values -> Raster; NaN cells become NODATA (has_nodata, sentinel, flag), as
// parse_ascii_grid marks them (geodata.hpp:19-35).
R::Raster raster_of(int h, int w, const double* v, double cellsize) {
  R::Grid<double> z(h, w);
  bool any = false;
  for (int i = 0; i < h * w; ++i) {
    z[i] = v[i];
    any = any || std::isnan(v[i]);
  }
  R::Raster r = R::raster_from_model(z, cellsize);
  if (any) {
    r.has_nodata = true;
    for (int mr = 0; mr < h; ++mr)
      for (int c = 0; c < w; ++c)
        if (std::isnan(z(mr, c))) {
          r.values(h - 1 - mr, c) = r.nodata;
          r.nodata_flag(h - 1 - mr, c) = 1;
        }
  }
  return r;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- rng.hpp ---------------------------------------------------------------
std::uint64_t ref_rng_word(std::uint64_t seed, std::uint64_t step, std::uint64_t stream,
                           std::uint64_t cell, std::uint64_t draw) {
  return R::rng_word(R::RngKey{seed, step, stream}, cell, draw);
}
double ref_rng_uniform(std::uint64_t seed, std::uint64_t step, std::uint64_t stream,
                       std::uint64_t cell, std::uint64_t draw) {
  return R::rng_uniform(R::RngKey{seed, step, stream}, cell, draw);
}
std::uint64_t ref_rng_below(std::uint64_t seed, std::uint64_t step, std::uint64_t stream,
                            std::uint64_t cell, std::uint64_t draw, std::uint64_t n) {
  return R::rng_below(R::RngKey{seed, step, stream}, cell, draw, n);
}

// ---- grid construction -----------------------------------------------------
// General layers: per-cell wind speed/direction, veg/den, 8 slopes per cell.
void* ref_grid_layers(int h, int w, const double* speed, const double* dir, const double* veg,
                      const double* den, const double* slope8) {
  try {
    R::SlopeField slope(h, w);
    for (int i = 0; i < h * w; ++i)
      for (int k = 0; k < 8; ++k) slope.set_toward(i / w, i % w, k, slope8[i * 8 + k]);
    return new R::GridState(R::FireLayer(h, w), R::WindField(grid_of(h, w, speed), grid_of(h, w, dir)),
                            R::FuelField(grid_of(h, w, veg), grid_of(h, w, den)), slope);
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

// Terrain: per-cell veg/den, fp32 elevation (widened exactly) -> slope_from_dem
// at `cellsize`, spatially uniform wind.  This is how C1-C4 inputs reach the oracle.
void* ref_grid_terrain(int h, int w, const double* veg, const double* den, const float* elev,
                       double cellsize, double speed, double dir) {
  try {
    std::vector<double> z(static_cast<size_t>(h) * w);
    for (int i = 0; i < h * w; ++i) z[i] = static_cast<double>(elev[i]);
    const R::SlopeField slope = R::slope_from_dem(raster_of(h, w, z.data(), cellsize));
    return new R::GridState(R::FireLayer(h, w), R::WindField::uniform(h, w, speed, dir),
                            R::FuelField(grid_of(h, w, veg), grid_of(h, w, den)), slope);
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

// grid_from_rasters (geodata.cpp:351-369): DEM (fp32 widened, NaN = nodata) + landcover codes
// (NaN = nodata) through a FuelTable {codes -> (veg, den)} with an optional fallback.
// Returns null with ref_last_error() on FileError / invalid_argument.
void* ref_grid_from_rasters(int h, int w, const float* elev, const double* landcover, int n_codes,
                            const int* codes, const double* veg, const double* den, int has_fallback,
                            double fb_veg, double fb_den, double cellsize, double speed, double dir) {
  try {
    std::vector<double> z(static_cast<size_t>(h) * w);
    for (int i = 0; i < h * w; ++i) z[i] = static_cast<double>(elev[i]);
    R::FuelTable table;
    for (int k = 0; k < n_codes; ++k) table.set(codes[k], R::FuelTable::Entry{veg[k], den[k]});
    if (has_fallback) table.set_fallback(R::FuelTable::Entry{fb_veg, fb_den});
    return new R::GridState(R::grid_from_rasters(raster_of(h, w, z.data(), cellsize),
                                                 raster_of(h, w, landcover, cellsize), table, speed, dir));
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

// Per-cell FuelField of a GridState (model order).
int ref_grid_fuel(const void* gp, double* veg, double* den) {
  const auto& g = *static_cast<const R::GridState*>(gp);
  const int w = g.width();
  for (int i = 0; i < g.height() * w; ++i) {
    veg[i] = g.fuel().veg(i / w, i % w);
    den[i] = g.fuel().den(i / w, i % w);
  }
  return 0;
}

void ref_grid_free(void* g) { delete static_cast<R::GridState*>(g); }

int ref_grid_slope(const void* gp, double* out8) {
  const auto& g = *static_cast<const R::GridState*>(gp);
  const int w = g.width();
  for (int i = 0; i < g.height() * w; ++i)
    for (int k = 0; k < 8; ++k) out8[i * 8 + k] = g.slope().toward(i / w, i % w, k);
  return 0;
}

// SpreadTables<double> contents: pot[cell*8+k], gamma[cell].
int ref_tables(const void* gp, const double* c, double* pot, double* gamma) {
  const auto& g = *static_cast<const R::GridState*>(gp);
  const R::SpreadTables<double> t(g, cfg_of(c));
  for (int i = 0; i < g.height() * g.width(); ++i) {
    gamma[i] = t.gamma(i);
    for (int k = 0; k < 8; ++k) pot[i * 8 + k] = t.pot(i, k);
  }
  return 0;
}

// kernel.hpp arrival_intensity + ignition_probability per cell, weights = burning.
int ref_intensity(const void* gp, const double* c, const std::uint8_t* fire, double* lambda,
                  double* p) {
  const auto& g = *static_cast<const R::GridState*>(gp);
  const R::SimConfig cfg = cfg_of(c);
  const int h = g.height(), w = g.width();
  auto weight = [&](int r, int cc) { return fire[r * w + cc] == 1 ? 1.0 : 0.0; };
  for (int r = 0; r < h; ++r)
    for (int cc = 0; cc < w; ++cc) {
      const R::CellIndex v{r, cc};
      const double l = R::arrival_intensity(v, weight, g, cfg);
      lambda[r * w + cc] = l;
      p[r * w + cc] = R::ignition_probability(v, l, g, cfg);
    }
  return 0;
}

// ---- stochastic engine -----------------------------------------------------
// run_stochastic(initial, grid, cfg, RngKey{seed, step0, stream}, steps, exec)
int ref_run_stochastic(const void* gp, const double* c, std::uint64_t seed, std::uint64_t step0,
                       std::uint64_t stream, int steps, int parallel, const std::uint8_t* in,
                       std::uint8_t* out) {
  try {
    const auto& g = *static_cast<const R::GridState*>(gp);
    const R::StochasticRun run =
        R::run_stochastic(layer_of(g.height(), g.width(), in), g, cfg_of(c),
                          R::RngKey{seed, step0, stream}, steps, false, nullptr,
                          parallel ? R::Exec::parallel : R::Exec::serial);
    unlayer(run.final_state, out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Straight-line serial reference.hpp step.
int ref_reference_step(const void* gp, const double* c, std::uint64_t seed, std::uint64_t step,
                       std::uint64_t stream, const std::uint8_t* in, std::uint8_t* out) {
  const auto& g = *static_cast<const R::GridState*>(gp);
  unlayer(R::reference_step_stochastic(layer_of(g.height(), g.width(), in), g, cfg_of(c),
                                       R::RngKey{seed, step, stream}),
          out);
  return 0;
}

// Lockstep StochasticBatch over one shared grid: make_stochastic_batch + step_batch.
int ref_step_batch(const void* gp, const double* c, std::uint64_t seed, std::uint64_t first_stream,
                   int count, int steps, const std::uint8_t* initial, std::uint8_t* out) {
  try {
    const auto& g = *static_cast<const R::GridState*>(gp);
    const R::SimConfig cfg = cfg_of(c);
    R::StochasticBatch b =
        R::make_stochastic_batch(layer_of(g.height(), g.width(), initial), count, seed, first_stream);
    const R::SpreadTables<double> t(g, cfg);
    for (int s = 0; s < steps; ++s) R::step_batch(b, t, cfg);
    const int n = g.height() * g.width();
    for (int m = 0; m < count; ++m) unlayer(b.members[m].fire, out + static_cast<std::size_t>(m) * n);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Per-env grids, OpenMP over envs, run_stochastic(Exec::serial) per env (the
// SURVEY §8(d) CPU-baseline harness for C1).  grids[e], streams[e]; states in/out
// [n_envs][h*w].  Returns wall seconds of the run (tables built inside, as the
// reference's run_stochastic does).
double ref_run_envs(void* const* grids, int n_envs, const double* c, std::uint64_t seed,
                    const std::uint64_t* streams, int steps, std::uint8_t* states, int threads) {
  const auto* g0 = static_cast<const R::GridState*>(grids[0]);
  const std::size_t n = static_cast<std::size_t>(g0->height()) * g0->width();
  const R::SimConfig cfg = cfg_of(c);
  if (threads > 0) omp_set_num_threads(threads);
  const auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel for schedule(dynamic, 1)
  for (int e = 0; e < n_envs; ++e) {
    const auto& g = *static_cast<const R::GridState*>(grids[e]);
    const R::StochasticRun run = R::run_stochastic(layer_of(g.height(), g.width(), states + e * n), g,
                                                   cfg, R::RngKey{seed, 0, streams[e]}, steps, false,
                                                   nullptr, R::Exec::serial);
    unlayer(run.final_state, states + e * n);
  }
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int ref_max_threads() { return omp_get_max_threads(); }

// C4 CPU-baseline harness: run_deterministic<Dual<6>> + loss per env, OpenMP
// over envs, the body of ref_loss_grad (calibrate.cpp:144-146 per env).  fire0s/masks
// [n_envs][h*w]; losses [n_envs], grads [n_envs][6].  Returns wall seconds (-1 on error).
int ref_loss_grad(const void* gp, const double* c, int steps, const std::uint8_t* fire0,
                  const double* mask, double bce_w, double mse_w, int pool, double* loss_out,
                  double* grad6);
double ref_loss_grad_envs(void* const* grids, int n_envs, const double* c, int steps,
                          const std::uint8_t* fire0s, const double* masks, double bce_w, double mse_w,
                          int pool, double* losses, double* grads, int threads) {
  const auto* g0 = static_cast<const R::GridState*>(grids[0]);
  const std::size_t n = static_cast<std::size_t>(g0->height()) * g0->width();
  if (threads > 0) omp_set_num_threads(threads);
  int bad = 0;
  const auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : bad)
  for (int e = 0; e < n_envs; ++e)
    bad += ref_loss_grad(grids[e], c, steps, fire0s + e * n, masks + e * n, bce_w, mse_w, pool, losses + e,
                         grads + 6 * e) != 0;
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return bad ? -1.0 : s;
}



// ---- fuel table (geodata.cpp default_worldcover_table) -----------------------
int ref_worldcover(int code, double* veg, double* den) {
  try {
    const auto e = R::default_worldcover_table().lookup(code);
    *veg = e.veg;
    *den = e.den;
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

// ---- RL environment (rl_env.hpp) --------------------------------------------
struct RefEnvCfg {
  int height, width, window_radius, water_capacity;
  double burn_penalty;
  int max_episode_steps, ignition_count, waste_water;
  double wind_speed, wind_direction, fuel_veg, fuel_den;
  double spread[6];
};

struct RefEnvState {  // flat EnvState; fire layer passed separately
  int agent_row, agent_col, water, step;
  std::uint64_t seed, stream;
  int done;
};

static R::EnvConfig env_cfg_of(const RefEnvCfg& c) {
  R::EnvConfig e;
  e.height = c.height;
  e.width = c.width;
  e.window_radius = c.window_radius;
  e.water_capacity = c.water_capacity;
  e.burn_penalty = c.burn_penalty;
  e.max_episode_steps = c.max_episode_steps;
  e.ignition_count = c.ignition_count;
  e.waste_water = c.waste_water != 0;
  e.wind_speed = c.wind_speed;
  e.wind_direction = c.wind_direction;
  e.fuel_veg = c.fuel_veg;
  e.fuel_den = c.fuel_den;
  e.spread = cfg_of(c.spread);
  return e;
}

int ref_env_preset(int which, RefEnvCfg* out) {
  const R::EnvConfig e = which == 0 ? R::default_preset() : R::smoke10_preset();
  out->height = e.height;
  out->width = e.width;
  out->window_radius = e.window_radius;
  out->water_capacity = e.water_capacity;
  out->burn_penalty = e.burn_penalty;
  out->max_episode_steps = e.max_episode_steps;
  out->ignition_count = e.ignition_count;
  out->waste_water = e.waste_water ? 1 : 0;
  out->wind_speed = e.wind_speed;
  out->wind_direction = e.wind_direction;
  out->fuel_veg = e.fuel_veg;
  out->fuel_den = e.fuel_den;
  const double s[6] = {e.spread.p_base, e.spread.alpha_w1, e.spread.alpha_w2,
                       e.spread.alpha_s, e.spread.alpha_gamma, e.spread.p_continue};
  std::memcpy(out->spread, s, sizeof s);
  return 0;
}

static R::EnvState state_of(const R::EnvConfig& c, const RefEnvState& s, const std::uint8_t* fire) {
  R::EnvState st;
  st.fire = layer_of(c.height, c.width, fire);
  st.agent = R::CellIndex{s.agent_row, s.agent_col};
  st.water = s.water;
  st.step = s.step;
  st.seed = s.seed;
  st.stream = s.stream;
  st.done = s.done != 0;
  return st;
}

static void flat_of(const R::EnvState& st, RefEnvState* s, std::uint8_t* fire) {
  s->agent_row = st.agent.row;
  s->agent_col = st.agent.col;
  s->water = st.water;
  s->step = st.step;
  s->seed = st.seed;
  s->stream = st.stream;
  s->done = st.done ? 1 : 0;
  unlayer(st.fire, fire);
}

int ref_env_reset(const RefEnvCfg* c, std::uint64_t seed, std::uint64_t stream, RefEnvState* s,
                  std::uint8_t* fire) {
  try {
    const R::FireSuppressionEnv env(env_cfg_of(*c));
    flat_of(env.reset(seed, stream), s, fire);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// One FireSuppressionEnv::step; returns the reward, writes next state + observation.
int ref_env_step(const RefEnvCfg* c, const RefEnvState* s, const std::uint8_t* fire, int action,
                 RefEnvState* s_out, std::uint8_t* fire_out, double* reward, double* obs) {
  try {
    const R::EnvConfig ec = env_cfg_of(*c);
    const R::FireSuppressionEnv env(ec);
    const R::StepResult r = env.step(state_of(ec, *s, fire), R::action_from_index(action));
    flat_of(r.state, s_out, fire_out);
    *reward = r.reward;
    if (obs) std::memcpy(obs, r.observation.values.data(), r.observation.values.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_env_observe(const RefEnvCfg* c, const RefEnvState* s, const std::uint8_t* fire, double* obs) {
  const R::EnvConfig ec = env_cfg_of(*c);
  const R::FireSuppressionEnv env(ec);
  const R::Observation o = env.observe(state_of(ec, *s, fire));
  std::memcpy(obs, o.values.data(), o.values.size() * sizeof(double));
  return static_cast<int>(o.values.size());
}

int ref_random_policy(std::uint64_t seed, std::uint64_t step, std::uint64_t stream) {
  return R::action_index(R::random_policy(R::RngKey{seed, step, stream}));
}

// ---- deterministic mode + calibration loss ------------------------------------
int ref_run_deterministic(const void* gp, const double* c, int steps, double* p_un, double* p_burn,
                          double* p_bd) {
  const auto& g = *static_cast<const R::GridState*>(gp);
  const int h = g.height(), w = g.width();
  R::ContinuousState s{grid_of(h, w, p_un), grid_of(h, w, p_burn), grid_of(h, w, p_bd)};
  const auto run = R::run_deterministic(s, g, cfg_of(c), steps);
  for (int i = 0; i < h * w; ++i) {
    p_un[i] = run.final_state.p_un[i];
    p_burn[i] = run.final_state.p_burn[i];
    p_bd[i] = run.final_state.p_bd[i];
  }
  return 0;
}

// Loss (LossConfig{bce_w, mse_w, pool}) after `steps` deterministic steps from a
// discrete initial layer, and d loss / d theta for the six SimConfig fields via
// forward-mode Dual<6> (the pattern of tests/test_calibrate.cpp:276-298).
int ref_loss_grad(const void* gp, const double* c, int steps, const std::uint8_t* fire0,
                  const double* mask, double bce_w, double mse_w, int pool, double* loss_out,
                  double* grad6) {
  try {
    const auto& g = *static_cast<const R::GridState*>(gp);
    const int h = g.height(), w = g.width();
    using D = R::Dual<6>;
    R::BasicSimConfig<D> dc;
    dc.p_base = R::lift_parameter<6>(0, c[0]);
    dc.alpha_w1 = R::lift_parameter<6>(1, c[1]);
    dc.alpha_w2 = R::lift_parameter<6>(2, c[2]);
    dc.alpha_s = R::lift_parameter<6>(3, c[3]);
    dc.alpha_gamma = R::lift_parameter<6>(4, c[4]);
    dc.p_continue = R::lift_parameter<6>(5, c[5]);
    const auto init = R::lift_state<6>(R::state_from_fire(layer_of(h, w, fire0)));
    const auto run = R::run_deterministic(init, g, dc, steps);
    R::CalibrationTarget tgt{grid_of(h, w, mask), steps};
    R::LossConfig lc;
    lc.bce_weight = bce_w;
    lc.mse_weight = mse_w;
    lc.pool_size = pool;
    const D l = R::loss(R::burn_probability_map(run.final_state), tgt, lc);
    *loss_out = l.value;
    for (int i = 0; i < 6; ++i) grad6[i] = l.grad[i];
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// calibrate(grid, initial, target, lc, opts) (calibrate.cpp:104-167).  Returns 0, or -1 with
// ref_last_error() set (invalid_argument / NumericalError).
int ref_calibrate(const void* gp, const double* un0, const double* bu0, const double* bd0,
                  const double* mask, int horizon, double bce_w, double mse_w, int pool,
                  int iterations, const double* init_theta, const int* optimize, double lr,
                  double* loss_hist, double* theta_hist, double* best_theta, double* best_loss) {
  try {
    const auto& g = *static_cast<const R::GridState*>(gp);
    const int h = g.height(), w = g.width();
    R::ContinuousState init{grid_of(h, w, un0), grid_of(h, w, bu0), grid_of(h, w, bd0)};
    R::CalibrationTarget tgt{grid_of(h, w, mask), horizon};
    R::LossConfig lc;
    lc.bce_weight = bce_w;
    lc.mse_weight = mse_w;
    lc.pool_size = pool;
    R::CalibrationOptions opts;
    opts.iterations = iterations;
    for (int i = 0; i < 6; ++i) {
      opts.init_theta[i] = init_theta[i];
      opts.optimize[i] = optimize[i] != 0;
    }
    opts.lr = lr;
    opts.exec = R::Exec::serial;
    const R::CalibrationResult res = R::calibrate(g, init, tgt, lc, opts);
    for (int i = 0; i <= iterations; ++i) {
      loss_hist[i] = res.loss_history[i];
      for (int k = 0; k < 6; ++k) theta_hist[i * 6 + k] = res.theta_history[i][k];
    }
    for (int k = 0; k < 6; ++k) best_theta[k] = res.best_theta[k];
    *best_loss = res.best_loss;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---- snapshot.hpp ----------------------------------------------------------
// serialize_snapshot of one layer (agent row < 0: none); returns the text length, writes at most
// cap bytes.
long ref_serialize_snapshot(int h, int w, const std::uint8_t* fire, std::uint64_t step, int ar, int ac, int water,
                            char* out, long cap) {
  try {
    R::Snapshot snap;
    snap.fire = R::FireLayer(h, w);
    for (int r = 0; r < h; ++r)
      for (int c = 0; c < w; ++c) snap.fire(r, c) = static_cast<R::FireState>(fire[r * w + c]);
    snap.step = step;
    if (ar >= 0) snap.agent = R::AgentMark{R::CellIndex{ar, ac}, water};
    const std::string t = R::serialize_snapshot(snap);
    if (out) std::memcpy(out, t.data(), std::min<long>(cap, static_cast<long>(t.size())));
    return static_cast<long>(t.size());
  } catch (const std::exception& e) {
    fail(e);
    return -1;
  }
}
// parse_snapshot: 0 ok (dims, step, layer up to cap bytes, agent), -1 with ref_last_error().
int ref_parse_snapshot(const char* text, long len, int* h, int* w, std::uint64_t* step, std::uint8_t* layer, long cap,
                       int* agent3, int* has_agent) {
  try {
    const R::Snapshot snap = R::parse_snapshot(std::string(text, static_cast<size_t>(len)));
    *h = snap.fire.height();
    *w = snap.fire.width();
    *step = snap.step;
    for (int r = 0; r < *h; ++r)
      for (int c = 0; c < *w; ++c)
        if (r * *w + c < cap) layer[r * *w + c] = static_cast<std::uint8_t>(snap.fire(r, c));
    *has_agent = snap.agent.has_value() ? 1 : 0;
    if (snap.agent) {
      agent3[0] = snap.agent->cell.row;
      agent3[1] = snap.agent->cell.col;
      agent3[2] = snap.agent->water;
    }
    return 0;
  } catch (const std::exception& e) {
    fail(e);
    return -1;
  }
}

// C2 reference CPU baseline: FireSuppressionEnv (rl_env.cpp:125-210) over n envs with OpenMP
// over envs (the parallel form of run_batch_episodes, rl_env.cpp:263-285), random_policy
// actions, an env that finishes is reset with the next stream (first_stream + k * n_envs).
// `steps` env-steps per env; returns wall seconds, *env_steps and *reward_sum.
double ref_env_batch(const RefEnvCfg* c, int n_envs, std::uint64_t seed, std::uint64_t first_stream,
                     int steps, int threads, long long* env_steps, double* reward_sum) {
  const R::EnvConfig ec = env_cfg_of(*c);
  const R::FireSuppressionEnv env(ec);
  if (threads > 0) omp_set_num_threads(threads);
  long long cnt = 0;
  double total = 0.0;
  const auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : cnt, total)
  for (int e = 0; e < n_envs; ++e) {
    std::uint64_t stream = first_stream + static_cast<std::uint64_t>(e);
    R::EnvState st = env.reset(seed, stream);
    for (int t = 0; t < steps; ++t) {
      if (st.done) {
        stream += static_cast<std::uint64_t>(n_envs);
        st = env.reset(seed, stream);
      }
      const R::Action a = R::random_policy(R::RngKey{seed, static_cast<std::uint64_t>(st.step), stream});
      R::StepResult r = env.step(st, a);
      total += r.reward;
      st = std::move(r.state);
      ++cnt;
    }
  }
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (env_steps) *env_steps = cnt;
  if (reward_sum) *reward_sum = total;
  return s;
}

}  // extern "C"
