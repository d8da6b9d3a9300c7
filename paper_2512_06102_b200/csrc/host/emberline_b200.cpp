// C++ drop-in (include/emberline_b200.hpp) over the C-ABI (include/ember_b200.h).
// Host-side value types mirror the reference's; every simulation step is a device call.
#include "emberline_b200.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numbers>

namespace emberline {

namespace {

[[noreturn]] void raise(int rc) {
  const std::string msg = ebl_last_error();
  switch (rc) {
    case EBL_EINVAL: throw std::invalid_argument(msg);
    case EBL_ELOGIC: throw std::logic_error(msg);
    case EBL_ERANGE: throw std::out_of_range(msg);
    case EBL_ENUMERIC: throw NumericalError(msg);
    default: throw std::runtime_error("ember_b200: " + msg);
  }
}

inline void ok(int rc) {
  if (rc != EBL_OK) raise(rc);
}

ebl_sim_config to_c(const SimConfig& c) {
  return ebl_sim_config{c.p_base, c.alpha_w1, c.alpha_w2, c.alpha_s, c.alpha_gamma, c.p_continue,
                        c.max_steps};
}

std::shared_ptr<ebl_batch> make_batch(int n, int h, int w, int device = 0, void* stream = nullptr) {
  ebl_batch* b = nullptr;
  ok(ebl_batch_create(&b, device, n, h, w, stream));
  return std::shared_ptr<ebl_batch>(b, ebl_batch_destroy);
}

void upload_grid(ebl_batch* b, const GridState& g) {
  const int n = g.height() * g.width();
  ok(ebl_batch_set_grid(b, 1, g.wind().speed_layer().data().data(),
                        g.wind().direction_layer().data().data(), g.fuel().veg_layer().data().data(),
                        g.fuel().den_layer().data().data(), g.slope().values().data()));
  (void)n;
}

std::vector<std::uint8_t> bytes_of(const FireLayer& f) {
  std::vector<std::uint8_t> v(f.size());
  std::memcpy(v.data(), f.data().data(), v.size());
  return v;
}

FireLayer layer_of(int h, int w, const std::uint8_t* p) {
  FireLayer f(h, w);
  std::memcpy(f.data().data(), p, static_cast<std::size_t>(h) * w);
  return f;
}

void reject_nan(const Grid<double>& g, const char* what) {
  for (double v : g.data())
    if (std::isnan(v)) throw std::invalid_argument(std::string(what) + ": NaN value in layer");
}

}  // namespace

// ---- grid.hpp --------------------------------------------------------------------------------
// The value types below reproduce the reference's constructors and validation (same checks, same
// exception types and messages, so a caller sees identical behaviour): grid.cpp:28-142.
int offset_index(NeighborOffset d) {  // grid.cpp:28-33
  for (int k = 0; k < 8; ++k)
    if (kNeighborOffsets[k] == d) return k;
  throw std::invalid_argument("offset_index: not a neighbor offset");
}

double wrap_angle(double a) {  // grid.cpp:35-42
  const double two_pi = 2.0 * std::numbers::pi;
  double w = std::fmod(a, two_pi);
  return w < 0.0 ? w + two_pi : w;
}

double offset_angle(NeighborOffset d) {  // grid.cpp:44-47
  if (d.dx < -1 || d.dx > 1 || d.dy < -1 || d.dy > 1 || (d.dx == 0 && d.dy == 0))
    throw std::invalid_argument("offset_angle: not a neighbor offset");
  return wrap_angle(std::atan2(static_cast<double>(d.dy), static_cast<double>(d.dx)));
}

// grid.cpp:49-62 (direction wrapped at construction)
WindField::WindField(Grid<double> speed, Grid<double> direction)
    : speed_(std::move(speed)), dir_(std::move(direction)) {
  if (speed_.height() != dir_.height() || speed_.width() != dir_.width())
    throw std::invalid_argument("WindField: speed and direction dimensions differ");
  for (double v : speed_.data()) {
    if (!std::isfinite(v)) throw std::invalid_argument("WindField: non-finite speed");
    if (v < 0.0) throw std::invalid_argument("WindField: negative speed");
  }
  for (double& v : dir_.data()) {
    if (!std::isfinite(v)) throw std::invalid_argument("WindField: non-finite direction");
    v = wrap_angle(v);
  }
}

WindField WindField::uniform(int h, int w, double speed, double direction) {
  return WindField(Grid<double>(h, w, speed), Grid<double>(h, w, direction));
}

// grid.cpp:68-77 (veg/den clamped to [-1, 1])
FuelField::FuelField(Grid<double> veg, Grid<double> den) : veg_(std::move(veg)), den_(std::move(den)) {
  if (veg_.height() != den_.height() || veg_.width() != den_.width())
    throw std::invalid_argument("FuelField: veg and den dimensions differ");
  reject_nan(veg_, "FuelField veg");
  reject_nan(den_, "FuelField den");
  for (double& v : veg_.data()) v = std::clamp(v, -1.0, 1.0);
  for (double& v : den_.data()) v = std::clamp(v, -1.0, 1.0);
}

FuelField FuelField::uniform(int h, int w, double veg, double den) {
  return FuelField(Grid<double>(h, w, veg), Grid<double>(h, w, den));
}

SlopeField::SlopeField(int height, int width) : h_(height), w_(width) {
  if (height < 1 || width < 1) throw std::invalid_argument("SlopeField: dimensions must be at least 1x1");
  s_.assign(static_cast<std::size_t>(h_) * w_ * 8, 0.0);
}

void SlopeField::set_toward(int r, int c, int k, double slope) {
  if (std::isnan(slope)) throw std::invalid_argument("SlopeField: NaN slope");
  s_[static_cast<std::size_t>(r * w_ + c) * 8 + k] = slope;
}

void validate_config(const SimConfig& cfg) {  // grid.cpp:107-124
  const ebl_sim_config c = to_c(cfg);
  ok(ebl_validate_config(&c));
}

// grid.cpp:126-142 (matching dimensions of every layer)
GridState::GridState(FireLayer fire, WindField wind, FuelField fuel, SlopeField slope)
    : fire_(std::move(fire)), wind_(std::move(wind)), fuel_(std::move(fuel)), slope_(std::move(slope)) {
  const int h = fire_.height(), w = fire_.width();
  if (h < 1 || w < 1) throw std::invalid_argument("GridState: empty fire layer");
  auto same = [&](int lh, int lw, const char* name) {
    if (lh != h || lw != w)
      throw std::invalid_argument(std::string("GridState: ") + name + " layer is " + std::to_string(lh) +
                                  "x" + std::to_string(lw) + ", expected " + std::to_string(h) + "x" +
                                  std::to_string(w));
  };
  same(wind_.height(), wind_.width(), "wind");
  same(fuel_.height(), fuel_.width(), "fuel");
  same(slope_.height(), slope_.width(), "slope");
  for (FireState s : fire_.data())
    if (static_cast<std::uint8_t>(s) > 2) throw std::invalid_argument("GridState: invalid fire state value");
  for (double s : slope_.values())
    if (std::isnan(s)) throw std::invalid_argument("GridState: NaN in slope layer");
}

GridState GridState::with_wind(WindField wind) const {
  if (wind.height() != height() || wind.width() != width())
    throw std::invalid_argument("GridState::with_wind: dimension mismatch");
  GridState g = *this;
  g.wind_ = std::move(wind);
  return g;
}

// ---- rng.hpp ----------------------------------------------------------------------------------
namespace {
inline std::uint64_t mix(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
}  // namespace

std::uint64_t rng_word(const RngKey& k, std::uint64_t cell, std::uint64_t draw) {
  return mix(mix(mix(mix(mix(0x243F6A8885A308D3ull ^ k.seed) ^ k.stream) ^ k.step) ^ cell) ^ draw);
}

double rng_uniform(const RngKey& k, std::uint64_t cell, std::uint64_t draw) {
  return static_cast<double>(rng_word(k, cell, draw) >> 11) * 0x1.0p-53;
}

std::uint64_t rng_below(const RngKey& k, std::uint64_t cell, std::uint64_t draw, std::uint64_t n) {
  const auto v = static_cast<std::uint64_t>(rng_uniform(k, cell, draw) * static_cast<double>(n));
  return v < n ? v : n - 1;
}

// ---- engine.hpp ---------------------------------------------------------------------------------
SpreadTables<double>::SpreadTables(const GridState& grid, const SimConfig& cfg)
    : h_(grid.height()), w_(grid.width()), cfg_(cfg), grid_(std::make_shared<GridState>(grid)) {}

ebl_batch* SpreadTables<double>::device_batch(int members) const {
  if (!cache_ || cache_members_ != members) {
    cache_ = make_batch(members, h_, w_);
    const ebl_sim_config c = to_c(cfg_);
    ok(ebl_batch_set_config(cache_.get(), &c));
    upload_grid(cache_.get(), *grid_);
    cache_members_ = members;
  }
  return cache_.get();
}

namespace {
// Steps `layers` (all on one shared grid) once on the device with per-member streams.
void device_step(const SpreadTables<double>& tables, const SimConfig& cfg, std::uint64_t seed,
                 std::uint64_t step, const std::vector<std::uint64_t>& streams,
                 std::vector<std::uint8_t>& layers) {
  ebl_batch* b = tables.device_batch(static_cast<int>(streams.size()));
  // SpreadTables carry the construction-time config for pot/gamma; the step's cfg
  // supplies p_continue (engine.cpp:18-20).  Changing only p_continue never rebuilds.
  ebl_sim_config c = to_c(tables.config());
  c.p_continue = cfg.p_continue;
  ok(ebl_batch_set_config(b, &c));
  ok(ebl_batch_set_state(b, layers.data()));
  ok(ebl_batch_set_key(b, seed, step, streams.data(), 0));
  ok(ebl_step_batch(b, 1));
  ok(ebl_batch_get_state(b, layers.data()));
}
}  // namespace

FireLayer step_stochastic(const FireLayer& fire, const SpreadTables<double>& tables,
                          const SimConfig& cfg, const RngKey& key, Exec) {
  if (fire.height() != tables.height() || fire.width() != tables.width())
    throw std::invalid_argument("step_stochastic: fire layer and tables dimensions differ");
  std::vector<std::uint8_t> v = bytes_of(fire);
  device_step(tables, cfg, key.seed, key.step, {key.stream}, v);
  return layer_of(fire.height(), fire.width(), v.data());
}

FireLayer step_stochastic(const FireLayer& fire, const GridState& grid, const SimConfig& cfg,
                          const RngKey& key, Exec exec) {
  const SpreadTables<double> tables(grid, cfg);
  return step_stochastic(fire, tables, cfg, key, exec);
}

// engine.cpp:74-86 (empty schedule is a logic_error; at_step clamps to the last entry)
WindSchedule::WindSchedule(std::vector<WindField> winds) : winds_(std::move(winds)) {
  for (std::size_t i = 1; i < winds_.size(); ++i)
    if (winds_[i].height() != winds_[0].height() || winds_[i].width() != winds_[0].width())
      throw std::invalid_argument("WindSchedule: wind field dimensions differ across steps");
}

const WindField& WindSchedule::at_step(std::uint64_t t) const {
  if (winds_.empty()) throw std::logic_error("WindSchedule::at_step on empty schedule");
  const std::uint64_t last = winds_.size() - 1;
  return winds_[t < last ? t : last];
}

StochasticRun run_stochastic(const FireLayer& initial, const GridState& grid, const SimConfig& cfg,
                             RngKey key, int steps, bool record, const WindSchedule* schedule, Exec) {
  StochasticRun out;
  const int h = initial.height(), w = initial.width();
  auto b = make_batch(1, h, w);
  const ebl_sim_config c = to_c(cfg);
  ok(ebl_batch_set_config(b.get(), &c));
  upload_grid(b.get(), grid);
  std::vector<std::uint8_t> v = bytes_of(initial);
  ok(ebl_batch_set_state(b.get(), v.data()));
  ok(ebl_batch_set_key(b.get(), key.seed, key.step, &key.stream, 0));
  if (record) out.trajectory.push_back(initial);
  if (schedule != nullptr && !schedule->empty() && steps > 0) {
    // the entries a run of `steps` from key.step can reach (engine.cpp:110-112), uploaded once;
    // the device indexes them by absolute step
    const std::uint64_t last = std::min<std::uint64_t>(key.step + steps - 1, schedule->size() - 1);
    const std::size_t n = static_cast<std::size_t>(h) * w;
    std::vector<double> sp((last + 1) * n), dr((last + 1) * n);
    for (std::uint64_t s = 0; s <= last; ++s) {
      const WindField& wf = schedule->at_step(s);
      std::memcpy(sp.data() + s * n, wf.speed_layer().data().data(), n * sizeof(double));
      std::memcpy(dr.data() + s * n, wf.direction_layer().data().data(), n * sizeof(double));
    }
    ok(ebl_batch_set_grid_wind_schedule(b.get(), static_cast<int>(last + 1), sp.data(), dr.data()));
  }
  if (steps > 0) {
    if (record) {  // every step's layer, written by the kernel as it goes
      std::vector<std::uint8_t> traj(static_cast<std::size_t>(steps) * h * w);
      ok(ebl_step_batch_record(b.get(), steps, traj.data(), 0));
      for (int t = 0; t < steps; ++t)
        out.trajectory.push_back(layer_of(h, w, traj.data() + static_cast<std::size_t>(t) * h * w));
    } else {
      ok(ebl_step_batch(b.get(), steps));  // one fused launch on the device
    }
  }
  ok(ebl_batch_get_state(b.get(), v.data()));
  out.final_state = layer_of(h, w, v.data());
  return out;
}

StochasticBatch make_stochastic_batch(const FireLayer& initial, int count, std::uint64_t seed,
                                      std::uint64_t first_stream) {
  if (count < 1) throw std::invalid_argument("make_stochastic_batch: count must be >= 1");
  StochasticBatch b;
  b.seed = seed;
  b.members.reserve(count);
  for (int j = 0; j < count; ++j) b.members.push_back({initial, first_stream + static_cast<std::uint64_t>(j)});
  return b;
}

void step_batch(StochasticBatch& batch, const SpreadTables<double>& tables, const SimConfig& cfg, Exec) {
  if (batch.members.empty()) return;
  const int h = batch.members[0].fire.height(), w = batch.members[0].fire.width();
  const std::size_t n = static_cast<std::size_t>(h) * w;
  std::vector<std::uint8_t> layers(n * batch.members.size());
  std::vector<std::uint64_t> streams(batch.members.size());
  for (std::size_t m = 0; m < batch.members.size(); ++m) {
    std::memcpy(layers.data() + m * n, batch.members[m].fire.data().data(), n);
    streams[m] = batch.members[m].stream;
  }
  device_step(tables, cfg, batch.seed, batch.step, streams, layers);
  for (std::size_t m = 0; m < batch.members.size(); ++m)
    std::memcpy(batch.members[m].fire.data().data(), layers.data() + m * n, n);
  batch.step += 1;
}

void step_batch(StochasticBatch& batch, const GridState& grid, const SimConfig& cfg, Exec exec) {
  const SpreadTables<double> tables(grid, cfg);
  step_batch(batch, tables, cfg, exec);
}

FireFractions fire_fraction_stats(const FireLayer& fire) {  // engine.cpp:185-197
  FireFractions f;
  const double n = fire.size();
  for (FireState s : fire.data()) {
    if (s == FireState::Unburned) f.unburned += 1.0;
    else if (s == FireState::Burning) f.burning += 1.0;
    else f.burned += 1.0;
  }
  f.unburned /= n;
  f.burning /= n;
  f.burned /= n;
  return f;
}

// ---- DeviceBatch ----------------------------------------------------------------------------------
DeviceBatch::DeviceBatch(int n_envs, int height, int width, int device, void* stream)
    : b_(make_batch(n_envs, height, width, device, stream)), n_(n_envs), h_(height), w_(width) {}

void DeviceBatch::set_config(const SimConfig& cfg) {
  const ebl_sim_config c = to_c(cfg);
  ok(ebl_batch_set_config(b_.get(), &c));
}

void DeviceBatch::set_grid(const GridState& g) { upload_grid(b_.get(), g); }

void DeviceBatch::set_terrain(int n_grids, const std::uint8_t* fc, const float* el, int n_classes,
                              const double* veg, const double* den, double cellsize) {
  ok(ebl_batch_set_terrain(b_.get(), n_grids, fc, el, n_classes, veg, den, cellsize));
}

void DeviceBatch::set_wind(int n_winds, const double* speed, const double* dir) {
  ok(ebl_batch_set_wind(b_.get(), n_winds, speed, dir));
}

void DeviceBatch::set_members(const std::vector<FireLayer>& layers) {
  if (static_cast<int>(layers.size()) != n_) throw std::invalid_argument("DeviceBatch: member count");
  const std::size_t n = static_cast<std::size_t>(h_) * w_;
  std::vector<std::uint8_t> v(n * n_);
  for (int m = 0; m < n_; ++m) std::memcpy(v.data() + m * n, layers[m].data().data(), n);
  ok(ebl_batch_set_state(b_.get(), v.data()));
}

std::vector<FireLayer> DeviceBatch::members() const {
  const std::size_t n = static_cast<std::size_t>(h_) * w_;
  std::vector<std::uint8_t> v(n * n_);
  ok(ebl_batch_get_state(b_.get(), v.data()));
  std::vector<FireLayer> out;
  for (int m = 0; m < n_; ++m) out.push_back(layer_of(h_, w_, v.data() + m * n));
  return out;
}

void DeviceBatch::set_key(std::uint64_t seed, std::uint64_t step, std::uint64_t first_stream) {
  ok(ebl_batch_set_key(b_.get(), seed, step, nullptr, first_stream));
}

void DeviceBatch::step(int n_steps) { ok(ebl_step_batch(b_.get(), n_steps)); }

std::vector<FireFractions> DeviceBatch::fractions() const {
  std::vector<std::int32_t> c(static_cast<std::size_t>(n_) * 4);
  ok(ebl_batch_counts(b_.get(), c.data()));
  std::vector<FireFractions> out(n_);
  const double n = static_cast<double>(h_) * w_;
  for (int m = 0; m < n_; ++m) out[m] = {c[m * 4] / n, c[m * 4 + 1] / n, c[m * 4 + 2] / n};
  return out;
}

// ---- deterministic path + calibrate -----------------------------------------------------------------
ContinuousState state_from_fire(const FireLayer& fire) {  // engine.cpp:42-52
  const int h = fire.height(), w = fire.width();
  ContinuousState s{Grid<double>(h, w), Grid<double>(h, w), Grid<double>(h, w)};
  for (int i = 0; i < h * w; ++i) {
    s.p_un[i] = fire[i] == FireState::Unburned ? 1.0 : 0.0;
    s.p_burn[i] = fire[i] == FireState::Burning ? 1.0 : 0.0;
    s.p_bd[i] = fire[i] == FireState::Burned ? 1.0 : 0.0;
  }
  return s;
}

void validate_state(const ContinuousState& s, double tol) {  // engine.cpp:54-72
  const int h = s.height(), w = s.width();
  if (s.p_burn.height() != h || s.p_burn.width() != w || s.p_bd.height() != h || s.p_bd.width() != w)
    throw std::invalid_argument("ContinuousState: component dimensions differ");
  for (int i = 0; i < h * w; ++i) {
    if (!(s.p_un[i] >= 0.0) || !(s.p_burn[i] >= 0.0) || !(s.p_bd[i] >= 0.0))
      throw std::invalid_argument("ContinuousState: negative or NaN component");
    if (std::abs(s.p_un[i] + s.p_burn[i] + s.p_bd[i] - 1.0) > tol)
      throw std::invalid_argument("ContinuousState: cell probabilities do not sum to 1");
  }
}

FireFractions fire_fraction_stats(const ContinuousState& s) {
  FireFractions f;
  const double n = s.p_un.size();
  for (int i = 0; i < s.p_un.size(); ++i) {
    f.unburned += s.p_un[i];
    f.burning += s.p_burn[i];
    f.burned += s.p_bd[i];
  }
  f.unburned /= n;
  f.burning /= n;
  f.burned /= n;
  return f;
}

namespace {
std::shared_ptr<ebl_batch> det_batch(int members, const GridState& grid, const SimConfig& cfg) {
  auto b = make_batch(members, grid.height(), grid.width());
  const ebl_sim_config c = to_c(cfg);
  ok(ebl_batch_set_config(b.get(), &c));
  upload_grid(b.get(), grid);
  return b;
}

void push_planes(ebl_batch* b, const std::vector<ContinuousState>& states) {
  const size_t n = static_cast<size_t>(states[0].height()) * states[0].width();
  std::vector<double> un(n * states.size()), bu(un.size()), bd(un.size());
  for (size_t m = 0; m < states.size(); ++m) {
    std::memcpy(un.data() + m * n, states[m].p_un.data().data(), n * sizeof(double));
    std::memcpy(bu.data() + m * n, states[m].p_burn.data().data(), n * sizeof(double));
    std::memcpy(bd.data() + m * n, states[m].p_bd.data().data(), n * sizeof(double));
  }
  ok(ebl_det_set_state(b, un.data(), bu.data(), bd.data()));
}

std::vector<ContinuousState> pull_planes(ebl_batch* b, int members, int h, int w) {
  const size_t n = static_cast<size_t>(h) * w;
  std::vector<double> un(n * members), bu(un.size()), bd(un.size());
  ok(ebl_det_get_state(b, un.data(), bu.data(), bd.data()));
  std::vector<ContinuousState> out;
  for (int m = 0; m < members; ++m) {
    ContinuousState s{Grid<double>(h, w), Grid<double>(h, w), Grid<double>(h, w)};
    std::memcpy(s.p_un.data().data(), un.data() + m * n, n * sizeof(double));
    std::memcpy(s.p_burn.data().data(), bu.data() + m * n, n * sizeof(double));
    std::memcpy(s.p_bd.data().data(), bd.data() + m * n, n * sizeof(double));
    out.push_back(std::move(s));
  }
  return out;
}
}  // namespace

DeterministicRun run_deterministic(const ContinuousState& initial, const GridState& grid,
                                   const SimConfig& cfg, int steps, bool record,
                                   const WindSchedule* schedule, Exec) {
  DeterministicRun out;
  const int h = initial.height(), w = initial.width();
  auto b = det_batch(1, grid, cfg);
  push_planes(b.get(), {initial});
  if (record) out.trajectory.push_back(initial);
  const bool sched = schedule != nullptr && !schedule->empty();
  if (!record && !sched) {
    ok(ebl_det_forward(b.get(), steps, 0));
  } else {
    for (int t = 0; t < steps; ++t) {
      if (sched) upload_grid(b.get(), grid.with_wind(schedule->at_step(static_cast<std::uint64_t>(t))));
      ok(ebl_det_forward(b.get(), 1, 0));
      if (record) out.trajectory.push_back(pull_planes(b.get(), 1, h, w)[0]);
    }
  }
  out.final_state = pull_planes(b.get(), 1, h, w)[0];
  return out;
}

ContinuousState step_deterministic(const ContinuousState& state, const GridState& grid,
                                   const SimConfig& cfg, Exec exec) {
  return run_deterministic(state, grid, cfg, 1, false, nullptr, exec).final_state;
}

void step_batch(DeterministicBatch& batch, const GridState& grid, const SimConfig& cfg, Exec) {
  if (batch.members.empty()) return;
  const int h = batch.members[0].height(), w = batch.members[0].width();
  auto b = det_batch(static_cast<int>(batch.members.size()), grid, cfg);
  push_planes(b.get(), batch.members);
  ok(ebl_det_forward(b.get(), 1, 0));
  batch.members = pull_planes(b.get(), static_cast<int>(batch.members.size()), h, w);
  batch.step += 1;
}

ParamArray params_of(const SimConfig& c) {
  return {c.p_base, c.alpha_w1, c.alpha_w2, c.alpha_s, c.alpha_gamma, c.p_continue};
}

SimConfig config_from_params(const ParamArray& t, int max_steps) {
  return SimConfig{t[0], t[1], t[2], t[3], t[4], t[5], max_steps};
}

std::pair<double, ParamArray> loss_and_gradient(const GridState& grid, const ContinuousState& initial,
                                                const CalibrationTarget& target, const LossConfig& lc,
                                                const SimConfig& cfg) {
  auto b = det_batch(1, grid, cfg);
  push_planes(b.get(), {initial});
  ok(ebl_det_forward(b.get(), target.horizon, 1));
  double l = 0.0;
  ParamArray g{};
  ok(ebl_det_loss_grad(b.get(), target.burn_mask.data().data(), lc.bce_weight, lc.mse_weight,
                       lc.pool_size, &l, g.data()));
  return {l, g};
}

CalibrationResult calibrate(const GridState& grid, const ContinuousState& initial,
                            const CalibrationTarget& target, const LossConfig& lc,
                            const CalibrationOptions& opts) {
  if (target.burn_mask.height() != grid.height() || target.burn_mask.width() != grid.width())
    throw std::invalid_argument("CalibrationTarget: mask dimensions differ from the grid");
  if (opts.iterations < 0) throw std::invalid_argument("calibrate: negative iteration count");
  auto b = det_batch(1, grid, SimConfig{});
  ebl_calib_options o{};
  ebl_default_calib_options(&o);
  o.iterations = opts.iterations;
  for (std::size_t i = 0; i < kParamCount; ++i) {
    o.init_theta[i] = opts.init_theta[i];
    o.optimize[i] = opts.optimize[i] ? 1 : 0;
  }
  o.lr = opts.lr;
  o.max_horizon = opts.max_horizon;
  CalibrationResult r;
  r.loss_history.resize(opts.iterations + 1);
  std::vector<double> th((opts.iterations + 1) * kParamCount);
  ok(ebl_calibrate(b.get(), initial.p_un.data().data(), initial.p_burn.data().data(),
                   initial.p_bd.data().data(), target.burn_mask.data().data(), target.horizon,
                   lc.bce_weight, lc.mse_weight, lc.pool_size, &o, r.loss_history.data(), th.data(),
                   r.best_theta.data(), &r.best_loss));
  for (int i = 0; i <= opts.iterations; ++i) {
    ParamArray t;
    for (std::size_t k = 0; k < kParamCount; ++k) t[k] = th[i * kParamCount + k];
    r.theta_history.push_back(t);
  }
  r.initial_loss = r.loss_history.front();
  return r;
}

// ---- rl_env.hpp ----------------------------------------------------------------------------------
namespace {
ebl_env_config env_to_c(const EnvConfig& e) {
  return ebl_env_config{e.height,         e.width,        e.window_radius,
                        e.water_capacity, e.burn_penalty, e.max_episode_steps,
                        e.ignition_count, e.waste_water ? 1 : 0, e.wind_speed,
                        e.wind_direction, e.fuel_veg,     e.fuel_den,
                        to_c(e.spread)};
}

EnvConfig env_from_c(const ebl_env_config& c) {
  EnvConfig e;
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
  e.spread = SimConfig{c.spread.p_base, c.spread.alpha_w1, c.spread.alpha_w2, c.spread.alpha_s,
                       c.spread.alpha_gamma, c.spread.p_continue, c.spread.max_steps};
  return e;
}
}  // namespace

EnvConfig default_preset() {
  ebl_env_config c;
  ebl_env_default_preset(&c);
  return env_from_c(c);
}

EnvConfig smoke10_preset() {
  ebl_env_config c;
  ebl_env_smoke10_preset(&c);
  return env_from_c(c);
}

Action action_from_index(int index) {
  if (index < 0 || index >= kActionCount)
    throw std::out_of_range("action_from_index: index " + std::to_string(index) + " outside [0, 10)");
  return Action{static_cast<Move>(index / 2), static_cast<Valve>(index % 2)};
}

int observation_size(const EnvConfig& cfg) {
  const ebl_env_config c = env_to_c(cfg);
  return ebl_env_observation_size(&c);
}

FireSuppressionEnv::FireSuppressionEnv(EnvConfig cfg) : cfg_(std::move(cfg)) {
  b_ = make_batch(1, cfg_.height > 0 ? cfg_.height : 1, cfg_.width > 0 ? cfg_.width : 1);
  const ebl_env_config c = env_to_c(cfg_);
  ok(ebl_rl_configure(b_.get(), EBL_RL_REFERENCE, &c, 0, 1, 0));
}

namespace {
void push_state(ebl_batch* b, const EnvState& s) {
  std::vector<std::uint8_t> v = bytes_of(s.fire);
  ok(ebl_batch_set_state(b, v.data()));
  const ebl_env_state es{s.agent.row, s.agent.col, s.water, s.step, s.seed, s.stream, s.done ? 1 : 0, 0};
  ok(ebl_rl_set_env_states(b, &es));
}

EnvState pull_state(ebl_batch* b, int h, int w) {
  std::vector<std::uint8_t> v(static_cast<std::size_t>(h) * w);
  ok(ebl_batch_get_state(b, v.data()));
  ebl_env_state es;
  ok(ebl_rl_get_env_states(b, &es));
  EnvState s;
  s.fire = layer_of(h, w, v.data());
  s.agent = CellIndex{es.agent_row, es.agent_col};
  s.water = es.water;
  s.step = es.step;
  s.seed = es.seed;
  s.stream = es.stream;
  s.done = es.done != 0;
  return s;
}
}  // namespace

EnvState FireSuppressionEnv::reset(std::uint64_t seed, std::uint64_t stream) const {
  ok(ebl_rl_reset(b_.get(), seed, &stream, nullptr));
  return pull_state(b_.get(), cfg_.height, cfg_.width);
}

Observation FireSuppressionEnv::observe(const EnvState& state) const {
  push_state(b_.get(), state);
  Observation o;
  o.values.resize(observation_size(cfg_));
  ok(ebl_rl_observe(b_.get(), o.values.data()));
  return o;
}

StepResult FireSuppressionEnv::step(const EnvState& state, Action action) const {
  if (state.done) throw std::logic_error("FireSuppressionEnv::step: episode already finished");
  push_state(b_.get(), state);
  const std::int32_t a = action_index(action);
  double reward = 0.0;
  std::uint8_t done = 0;
  ok(ebl_rl_step(b_.get(), &a, &reward, &done, 0));
  StepResult r;
  r.state = pull_state(b_.get(), cfg_.height, cfg_.width);
  r.observation.values.resize(observation_size(cfg_));
  ok(ebl_rl_observe(b_.get(), r.observation.values.data()));
  r.reward = reward;
  r.done = done != 0;
  return r;
}

Action random_policy(const RngKey& key) {
  return action_from_index(static_cast<int>(rng_below(key, 0, kDrawPolicy, kActionCount)));
}

}  // namespace emberline
