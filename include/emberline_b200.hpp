// emberline_b200.hpp — C++ drop-in for the reference's stochastic engine and RL env
// (namespace emberline, signatures of proj/include/emberline/{grid,rng,engine,rl_env}.hpp),
// implemented over the C-ABI of include/ember_b200.h: every step runs on the B200.
//
// Switching: replace `#include "emberline/engine.hpp"` / `"emberline/rl_env.hpp"` with
// `#include "emberline_b200.hpp"` and link libemberline_b200.so.
// Semantics are the reference's bit for bit (tests/cpp/test_dropin.cpp runs the same
// checks against both).  Exceptions are the reference's: std::invalid_argument,
// std::logic_error, std::out_of_range.  There is no CPU path: constructing device state
// without a CUDA device throws std::runtime_error.
//
// Scope: the stochastic path of engine.hpp (step_stochastic, run_stochastic,
// StochasticBatch/step_batch, fire_fraction_stats), the deterministic path
// (state_from_fire, DeterministicBatch/step_batch, loss_and_gradient), rl_env.hpp's
// FireSuppressionEnv reset/observe/step, and the device-resident DeviceBatch the
// throughput path uses.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "ember_b200.h"

namespace emberline {

// ---- grid.hpp -------------------------------------------------------------------------
template <class T>
class Grid {
 public:
  Grid() = default;
  Grid(int height, int width, T fill = T{}) {
    if (height < 1 || width < 1) throw std::invalid_argument("Grid: dimensions must be at least 1x1");
    h_ = height;
    w_ = width;
    v_.assign(static_cast<std::size_t>(h_) * w_, fill);
  }
  int height() const { return h_; }
  int width() const { return w_; }
  int size() const { return h_ * w_; }
  bool in_bounds(int r, int c) const { return r >= 0 && r < h_ && c >= 0 && c < w_; }
  int index(int r, int c) const { return r * w_ + c; }
  T& operator()(int r, int c) { return v_[index(r, c)]; }
  const T& operator()(int r, int c) const { return v_[index(r, c)]; }
  T& operator[](int i) { return v_[i]; }
  const T& operator[](int i) const { return v_[i]; }
  std::vector<T>& data() { return v_; }
  const std::vector<T>& data() const { return v_; }
  bool operator==(const Grid&) const = default;

 private:
  int h_ = 0, w_ = 0;
  std::vector<T> v_;
};

struct CellIndex {
  int row = 0, col = 0;
  bool operator==(const CellIndex&) const = default;
};

struct NeighborOffset {
  int dx = 0, dy = 0;
  bool operator==(const NeighborOffset&) const = default;
};

inline constexpr std::array<NeighborOffset, 8> kNeighborOffsets = {
    {{1, 0}, {1, 1}, {0, 1}, {-1, 1}, {-1, 0}, {-1, -1}, {0, -1}, {1, -1}}};

int offset_index(NeighborOffset d);
double offset_angle(NeighborOffset d);
double wrap_angle(double a);

enum class FireState : std::uint8_t { Unburned = 0, Burning = 1, Burned = 2 };
using FireLayer = Grid<FireState>;

class WindField {
 public:
  WindField(Grid<double> speed, Grid<double> direction);
  static WindField uniform(int h, int w, double speed, double direction);
  int height() const { return speed_.height(); }
  int width() const { return speed_.width(); }
  double speed(int r, int c) const { return speed_(r, c); }
  double direction(int r, int c) const { return dir_(r, c); }
  const Grid<double>& speed_layer() const { return speed_; }
  const Grid<double>& direction_layer() const { return dir_; }

 private:
  Grid<double> speed_, dir_;
};

class FuelField {
 public:
  FuelField(Grid<double> veg, Grid<double> den);
  static FuelField uniform(int h, int w, double veg, double den);
  int height() const { return veg_.height(); }
  int width() const { return veg_.width(); }
  double veg(int r, int c) const { return veg_(r, c); }
  double den(int r, int c) const { return den_(r, c); }
  const Grid<double>& veg_layer() const { return veg_; }
  const Grid<double>& den_layer() const { return den_; }

 private:
  Grid<double> veg_, den_;
};

class SlopeField {
 public:
  SlopeField() = default;
  SlopeField(int height, int width);
  int height() const { return h_; }
  int width() const { return w_; }
  double toward(int r, int c, int k) const { return s_[static_cast<std::size_t>(r * w_ + c) * 8 + k]; }
  void set_toward(int r, int c, int k, double slope);
  const std::vector<double>& values() const { return s_; }

 private:
  int h_ = 0, w_ = 0;
  std::vector<double> s_;
};

template <class S>
struct BasicSimConfig {
  S p_base{0.12};
  S alpha_w1{0.2};
  S alpha_w2{0.4};
  S alpha_s{1.0};
  S alpha_gamma{1.0};
  S p_continue{0.6};
  int max_steps = 200;
};
using SimConfig = BasicSimConfig<double>;

void validate_config(const SimConfig& cfg);

class GridState {
 public:
  GridState(FireLayer fire, WindField wind, FuelField fuel, SlopeField slope);
  int height() const { return fire_.height(); }
  int width() const { return fire_.width(); }
  const FireLayer& fire() const { return fire_; }
  const WindField& wind() const { return wind_; }
  const FuelField& fuel() const { return fuel_; }
  const SlopeField& slope() const { return slope_; }
  GridState with_wind(WindField wind) const;

 private:
  FireLayer fire_;
  WindField wind_;
  FuelField fuel_;
  SlopeField slope_;
};

inline GridState new_grid(FireLayer f, WindField w, FuelField u, SlopeField s) {
  return GridState(std::move(f), std::move(w), std::move(u), std::move(s));
}

// ---- rng.hpp ---------------------------------------------------------------------------
struct RngKey {
  std::uint64_t seed = 0, step = 0, stream = 0;
};
inline constexpr std::uint64_t kDrawFireEvent = 0, kDrawEnvSetup = 1, kDrawPolicy = 2,
                               kDrawSynthesis = 3;
std::uint64_t rng_word(const RngKey& key, std::uint64_t cell, std::uint64_t draw);
double rng_uniform(const RngKey& key, std::uint64_t cell, std::uint64_t draw);
std::uint64_t rng_below(const RngKey& key, std::uint64_t cell, std::uint64_t draw, std::uint64_t n);

// ---- engine.hpp (stochastic path) --------------------------------------------------------
enum class Exec { serial, parallel };  // accepted for signature parity; the device decides

// Device-resident SpreadTables: built once from (grid, cfg) in fp64 and kept in HBM,
// so step_stochastic(fire, tables, ...) uploads only the fire layer.
template <class S>
class SpreadTables;

template <>
class SpreadTables<double> {
 public:
  SpreadTables(const GridState& grid, const SimConfig& cfg);
  int height() const { return h_; }
  int width() const { return w_; }
  const SimConfig& config() const { return cfg_; }
  ebl_batch* device_batch(int members) const;  // shared-grid batch of `members`, cached

 private:
  int h_, w_;
  SimConfig cfg_;
  std::shared_ptr<const GridState> grid_;
  mutable std::shared_ptr<ebl_batch> cache_;
  mutable int cache_members_ = 0;
};

FireLayer step_stochastic(const FireLayer& fire, const SpreadTables<double>& tables,
                          const SimConfig& cfg, const RngKey& key, Exec exec = Exec::parallel);
FireLayer step_stochastic(const FireLayer& fire, const GridState& grid, const SimConfig& cfg,
                          const RngKey& key, Exec exec = Exec::parallel);

class WindSchedule {
 public:
  WindSchedule() = default;
  explicit WindSchedule(std::vector<WindField> winds);
  bool empty() const { return winds_.empty(); }
  std::size_t size() const { return winds_.size(); }
  const WindField& at_step(std::uint64_t t) const;

 private:
  std::vector<WindField> winds_;
};

struct StochasticRun {
  FireLayer final_state;
  std::vector<FireLayer> trajectory;
};

StochasticRun run_stochastic(const FireLayer& initial, const GridState& grid, const SimConfig& cfg,
                             RngKey key, int steps, bool record = false,
                             const WindSchedule* schedule = nullptr, Exec exec = Exec::parallel);

struct StochasticBatch {
  std::uint64_t seed = 0;
  std::uint64_t step = 0;
  struct Member {
    FireLayer fire;
    std::uint64_t stream = 0;
  };
  std::vector<Member> members;
};

StochasticBatch make_stochastic_batch(const FireLayer& initial, int count, std::uint64_t seed,
                                      std::uint64_t first_stream = 0);
void step_batch(StochasticBatch& batch, const SpreadTables<double>& tables, const SimConfig& cfg,
                Exec exec = Exec::parallel);
void step_batch(StochasticBatch& batch, const GridState& grid, const SimConfig& cfg,
                Exec exec = Exec::parallel);

struct FireFractions {
  double unburned = 0.0, burning = 0.0, burned = 0.0;
};
FireFractions fire_fraction_stats(const FireLayer& fire);

// The throughput form of StochasticBatch: members stay in HBM between steps.
class DeviceBatch {
 public:
  DeviceBatch(int n_envs, int height, int width, int device = 0, void* cuda_stream = nullptr);
  void set_config(const SimConfig& cfg);
  void set_grid(const GridState& shared_grid);
  void set_terrain(int n_grids, const std::uint8_t* fuel_class, const float* elevation,
                   int n_classes, const double* class_veg, const double* class_den,
                   double cellsize);
  void set_wind(int n_winds, const double* speed, const double* direction);
  void set_members(const std::vector<FireLayer>& layers);
  std::vector<FireLayer> members() const;
  void set_key(std::uint64_t seed, std::uint64_t step, std::uint64_t first_stream = 0);
  void step(int n_steps = 1);
  std::vector<FireFractions> fractions() const;
  ebl_batch* handle() const { return b_.get(); }

 private:
  std::shared_ptr<ebl_batch> b_;
  int n_, h_, w_;
};

// ---- engine.hpp (deterministic path, double) + calibrate.hpp -------------------------------
template <class S>
struct BasicContinuousState {
  Grid<S> p_un, p_burn, p_bd;
  int height() const { return p_un.height(); }
  int width() const { return p_un.width(); }
};
using ContinuousState = BasicContinuousState<double>;

ContinuousState state_from_fire(const FireLayer& fire);
void validate_state(const ContinuousState& state, double tol = 1e-9);
FireFractions fire_fraction_stats(const ContinuousState& state);

// step_deterministic / run_deterministic (engine.hpp:147-245) for S = double, on the device in
// the reference's fp64 arithmetic.
ContinuousState step_deterministic(const ContinuousState& state, const GridState& grid,
                                   const SimConfig& cfg, Exec exec = Exec::parallel);
struct DeterministicRun {
  ContinuousState final_state;
  std::vector<ContinuousState> trajectory;
};
DeterministicRun run_deterministic(const ContinuousState& initial, const GridState& grid,
                                   const SimConfig& cfg, int steps, bool record = false,
                                   const WindSchedule* schedule = nullptr, Exec exec = Exec::parallel);

struct DeterministicBatch {
  std::uint64_t step = 0;
  std::vector<ContinuousState> members;
};
void step_batch(DeterministicBatch& batch, const GridState& grid, const SimConfig& cfg,
                Exec exec = Exec::parallel);

inline constexpr std::size_t kParamCount = 6;
using ParamArray = std::array<double, kParamCount>;
enum ParamIndex : std::size_t {
  kParamPBase = 0, kParamAlphaW1 = 1, kParamAlphaW2 = 2, kParamAlphaS = 3, kParamAlphaGamma = 4,
  kParamPContinue = 5,
};
ParamArray params_of(const SimConfig& cfg);
SimConfig config_from_params(const ParamArray& theta, int max_steps = 200);

struct CalibrationTarget {
  Grid<double> burn_mask;
  int horizon = 0;
};
struct LossConfig {
  double bce_weight = 1.0;
  double mse_weight = 1.0;
  int pool_size = 4;
  double bce_epsilon = 1e-6;
};
struct CalibrationOptions {
  int iterations = 300;
  ParamArray init_theta = params_of(SimConfig{});
  std::array<bool, kParamCount> optimize = {true, true, true, true, true, true};
  double lr = 1e-2;
  int max_horizon = 2000;
  Exec exec = Exec::parallel;
};
struct CalibrationResult {
  ParamArray best_theta{};
  double best_loss = 0.0;
  double initial_loss = 0.0;
  std::vector<double> loss_history;
  std::vector<ParamArray> theta_history;
};

// Loss value and d loss / d theta (ParamIndex order) after `horizon` deterministic steps:
// the reference gets these from Dual<6> (calibrate.cpp:130-151); here reverse mode on device.
std::pair<double, ParamArray> loss_and_gradient(const GridState& grid, const ContinuousState& initial,
                                                const CalibrationTarget& target, const LossConfig& lc,
                                                const SimConfig& cfg);
// calibrate (calibrate.cpp:104-167); throws NumericalError on a non-finite loss/gradient.
CalibrationResult calibrate(const GridState& grid, const ContinuousState& initial,
                            const CalibrationTarget& target, const LossConfig& lc,
                            const CalibrationOptions& opts);

class NumericalError : public std::runtime_error {  // errors.hpp:14-17
 public:
  using std::runtime_error::runtime_error;
};

// ---- rl_env.hpp ---------------------------------------------------------------------------
struct EnvConfig {
  int height = 20, width = 20, window_radius = 2, water_capacity = 30;
  double burn_penalty = 0.05;
  int max_episode_steps = 120, ignition_count = 1;
  bool waste_water = true;
  double wind_speed = 1.0, wind_direction = 0.0, fuel_veg = 0.0, fuel_den = 0.0;
  SimConfig spread;
};
inline constexpr double kTerminalBonus = 10.0;
EnvConfig default_preset();
EnvConfig smoke10_preset();

enum class Move : int { North = 0, South = 1, East = 2, West = 3, Stay = 4 };
enum class Valve : int { Closed = 0, Open = 1 };
struct Action {
  Move move = Move::Stay;
  Valve valve = Valve::Closed;
  bool operator==(const Action&) const = default;
};
inline constexpr int kActionCount = 10;
inline int action_index(Action a) { return static_cast<int>(a.move) * 2 + static_cast<int>(a.valve); }
Action action_from_index(int index);

struct EnvState {
  FireLayer fire;
  CellIndex agent;
  int water = 0;
  int step = 0;
  std::uint64_t seed = 0;
  std::uint64_t stream = 0;
  bool done = false;
};

struct Observation {
  std::vector<double> values;
};
int observation_size(const EnvConfig& cfg);

struct StepResult {
  EnvState state;
  Observation observation;
  double reward = 0.0;
  bool done = false;
};

class FireSuppressionEnv {
 public:
  explicit FireSuppressionEnv(EnvConfig cfg);
  const EnvConfig& config() const { return cfg_; }
  EnvState reset(std::uint64_t seed, std::uint64_t stream) const;
  Observation observe(const EnvState& state) const;
  StepResult step(const EnvState& state, Action action) const;

 private:
  EnvConfig cfg_;
  std::shared_ptr<ebl_batch> b_;  // one-env device batch in reference RL mode
};

Action random_policy(const RngKey& key);

}  // namespace emberline
