// Drop-in parity: the same calls made against the reference (namespace ebl_ref, the
// unmodified sources compiled in place — oracle/_ref) and against the C++ drop-in
// (include/emberline_b200.hpp, every step on the GPU), compared bit for bit.
// Mirrors the reference's own checks: test_engine.cpp:265-376, test_rl_env.cpp:234-253.
#define emberline ebl_ref
#include "emberline/calibrate.hpp"
#include "emberline/engine.hpp"
#include "emberline/reference.hpp"
#include "emberline/rl_env.hpp"
#undef emberline

#include <cstdio>
#include <cstring>
#include <functional>

#include "emberline_b200.hpp"

namespace R = ebl_ref;
namespace D = emberline;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                          \
  do {                                                                    \
    ++g_checks;                                                           \
    if (!(c)) {                                                           \
      ++g_fail;                                                           \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);   \
    }                                                                     \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

struct Layers {
  int h, w;
  std::vector<double> speed, dir, veg, den, slope8;
};

static Layers varied(std::uint64_t seed, int h, int w) {  // same RNG-driven pattern as test_engine.cpp
  Layers L{h, w};
  const R::RngKey key{seed, 0, 0};
  const int n = h * w;
  L.speed.resize(n), L.dir.resize(n), L.veg.resize(n), L.den.resize(n), L.slope8.resize(n * 8);
  for (int i = 0; i < n; ++i) {
    L.speed[i] = 2.0 * R::rng_uniform(key, i, 10);
    L.dir[i] = 6.28 * R::rng_uniform(key, i, 11);
    L.veg[i] = R::rng_uniform(key, i, 12) - 0.3;
    L.den[i] = R::rng_uniform(key, i, 13) - 0.3;
    for (int k = 0; k < 8; ++k) L.slope8[i * 8 + k] = 0.5 * R::rng_uniform(key, i, 20 + k) - 0.25;
  }
  return L;
}

static R::GridState ref_grid(const Layers& L) {
  R::Grid<double> s(L.h, L.w), d(L.h, L.w), v(L.h, L.w), e(L.h, L.w);
  R::SlopeField sl(L.h, L.w);
  for (int i = 0; i < L.h * L.w; ++i) {
    s[i] = L.speed[i], d[i] = L.dir[i], v[i] = L.veg[i], e[i] = L.den[i];
    for (int k = 0; k < 8; ++k) sl.set_toward(i / L.w, i % L.w, k, L.slope8[i * 8 + k]);
  }
  return R::new_grid(R::FireLayer(L.h, L.w), R::WindField(s, d), R::FuelField(v, e), sl);
}

static D::GridState dev_grid(const Layers& L) {
  D::Grid<double> s(L.h, L.w), d(L.h, L.w), v(L.h, L.w), e(L.h, L.w);
  D::SlopeField sl(L.h, L.w);
  for (int i = 0; i < L.h * L.w; ++i) {
    s[i] = L.speed[i], d[i] = L.dir[i], v[i] = L.veg[i], e[i] = L.den[i];
    for (int k = 0; k < 8; ++k) sl.set_toward(i / L.w, i % L.w, k, L.slope8[i * 8 + k]);
  }
  return D::new_grid(D::FireLayer(L.h, L.w), D::WindField(s, d), D::FuelField(v, e), sl);
}

static bool same(const R::FireLayer& a, const D::FireLayer& b) {
  return a.height() == b.height() && a.width() == b.width() &&
         std::memcmp(a.data().data(), b.data().data(), a.size()) == 0;
}

static D::FireLayer to_dev(const R::FireLayer& a) {
  D::FireLayer b(a.height(), a.width());
  std::memcpy(b.data().data(), a.data().data(), a.size());
  return b;
}

static void test_engine_matches_reference() {
  const Layers L = varied(47, 9, 9);
  const R::GridState rg = ref_grid(L);
  const D::GridState dg = dev_grid(L);
  R::SimConfig rc;
  rc.p_base = 0.25, rc.p_continue = 0.55;
  D::SimConfig dc;
  dc.p_base = 0.25, dc.p_continue = 0.55;
  R::FireLayer rf(9, 9, R::FireState::Unburned);
  rf(4, 4) = rf(2, 7) = R::FireState::Burning;
  D::FireLayer df = to_dev(rf);
  R::FireLayer straight = rf;
  const D::SpreadTables<double> tables(dg, dc);
  D::FireLayer dt = df;
  for (int t = 0; t < 20; ++t) {
    const R::RngKey rk{13, static_cast<std::uint64_t>(t), 2};
    const D::RngKey dk{13, static_cast<std::uint64_t>(t), 2};
    rf = R::step_stochastic(rf, rg, rc, rk);
    straight = R::reference_step_stochastic(straight, rg, rc, rk);
    df = D::step_stochastic(df, dg, dc, dk);
    dt = D::step_stochastic(dt, tables, dc, dk);
    CHECK(same(rf, df));
    CHECK(same(straight, df));
    CHECK(same(rf, dt));
  }
}

static void test_run_and_record() {
  const Layers L = varied(37, 6, 6);
  const R::GridState rg = ref_grid(L);
  const D::GridState dg = dev_grid(L);
  R::FireLayer f(6, 6, R::FireState::Unburned);
  f(3, 3) = R::FireState::Burning;
  const auto r5 = R::run_stochastic(f, rg, R::SimConfig{}, R::RngKey{4, 0, 0}, 5, true);
  const auto d5 = D::run_stochastic(to_dev(f), dg, D::SimConfig{}, D::RngKey{4, 0, 0}, 5, true);
  CHECK(d5.trajectory.size() == 6);
  for (std::size_t i = 0; i < r5.trajectory.size() && i < d5.trajectory.size(); ++i)
    CHECK(same(r5.trajectory[i], d5.trajectory[i]));
  const auto d0 = D::run_stochastic(to_dev(f), dg, D::SimConfig{}, D::RngKey{4, 0, 0}, 0);
  CHECK(same(f, d0.final_state) && d0.trajectory.empty());
  const Layers L2 = varied(41, 12, 12);
  R::SimConfig rc;
  rc.p_base = 0.2;
  D::SimConfig dc;
  dc.p_base = 0.2;
  R::FireLayer g(12, 12, R::FireState::Unburned);
  g(6, 6) = R::FireState::Burning;
  const auto a = R::run_stochastic(g, ref_grid(L2), rc, R::RngKey{3, 7, 1}, 25);
  const auto b = D::run_stochastic(to_dev(g), dev_grid(L2), dc, D::RngKey{3, 7, 1}, 25);
  CHECK(same(a.final_state, b.final_state));
}

static void test_wind_schedule() {
  const Layers L = varied(59, 8, 8);
  R::SimConfig rc;
  rc.p_base = 0.3;
  D::SimConfig dc;
  dc.p_base = 0.3;
  R::FireLayer f(8, 8, R::FireState::Unburned);
  f(4, 4) = R::FireState::Burning;
  const R::WindSchedule rs({R::WindField::uniform(8, 8, 0.5, 0.0), R::WindField::uniform(8, 8, 2.0, 1.5)});
  const D::WindSchedule ds({D::WindField::uniform(8, 8, 0.5, 0.0), D::WindField::uniform(8, 8, 2.0, 1.5)});
  const auto a = R::run_stochastic(f, ref_grid(L), rc, R::RngKey{21, 0, 0}, 4, true, &rs);
  const auto b = D::run_stochastic(to_dev(f), dev_grid(L), dc, D::RngKey{21, 0, 0}, 4, true, &ds);
  for (int i = 0; i < 5; ++i) CHECK(same(a.trajectory[i], b.trajectory[i]));
  CHECK(throws<std::logic_error>([] { D::WindSchedule(std::vector<D::WindField>{}).at_step(0); }));
}

static void test_batches() {
  const Layers L = varied(61, 10, 10);
  R::SimConfig rc;
  rc.p_base = 0.22;
  D::SimConfig dc;
  dc.p_base = 0.22;
  R::FireLayer f(10, 10, R::FireState::Unburned);
  f(5, 5) = R::FireState::Burning;
  R::StochasticBatch rb = R::make_stochastic_batch(f, 8, 123, 3);
  D::StochasticBatch db = D::make_stochastic_batch(to_dev(f), 8, 123, 3);
  const R::SpreadTables<double> rt(ref_grid(L), rc);
  const D::SpreadTables<double> dt(dev_grid(L), dc);
  for (int t = 0; t < 15; ++t) {
    R::step_batch(rb, rt, rc);
    D::step_batch(db, dt, dc);
  }
  CHECK(db.step == 15);
  for (int k = 0; k < 8; ++k) CHECK(same(rb.members[k].fire, db.members[k].fire));
  const auto rfs = R::fire_fraction_stats(rb.members[0].fire);
  const auto dfs = D::fire_fraction_stats(db.members[0].fire);
  CHECK(rfs.unburned == dfs.unburned && rfs.burning == dfs.burning && rfs.burned == dfs.burned);
  CHECK(throws<std::invalid_argument>([&] { D::make_stochastic_batch(to_dev(f), 0, 1); }));
  // DeviceBatch (members resident): equals step_batch
  D::DeviceBatch dev(8, 10, 10);
  dev.set_config(dc);
  dev.set_grid(dev_grid(L));
  dev.set_members(std::vector<D::FireLayer>(8, to_dev(f)));
  dev.set_key(123, 0, 3);
  dev.step(15);
  const auto mem = dev.members();
  for (int k = 0; k < 8; ++k) CHECK(same(rb.members[k].fire, mem[k]));
  const auto fr = dev.fractions();
  CHECK(fr[0].burned == rfs.burned && fr[0].burning == rfs.burning);
}

static void test_rl_env() {
  const R::FireSuppressionEnv renv(R::default_preset());
  const D::FireSuppressionEnv denv(D::default_preset());
  for (std::uint64_t ep = 0; ep < 4; ++ep) {
    R::EnvState rs = renv.reset(11, ep);
    D::EnvState ds = denv.reset(11, ep);
    CHECK(same(rs.fire, ds.fire) && rs.agent.row == ds.agent.row && rs.agent.col == ds.agent.col);
    CHECK(renv.observe(rs).values == denv.observe(ds).values);
    int guard = 0;
    while (!rs.done && guard++ < 500) {
      const R::Action ra = R::random_policy(R::RngKey{11, static_cast<std::uint64_t>(rs.step), ep});
      const D::Action da = D::random_policy(D::RngKey{11, static_cast<std::uint64_t>(ds.step), ep});
      CHECK(R::action_index(ra) == D::action_index(da));
      const R::StepResult rr = renv.step(rs, ra);
      const D::StepResult dr = denv.step(ds, da);
      CHECK(rr.reward == dr.reward && rr.done == dr.done);
      CHECK(same(rr.state.fire, dr.state.fire));
      CHECK(rr.state.water == dr.state.water && rr.state.step == dr.state.step);
      CHECK(rr.observation.values == dr.observation.values);
      rs = rr.state;
      ds = dr.state;
    }
    CHECK(ds.done);
    CHECK(throws<std::logic_error>([&] { denv.step(ds, D::Action{}); }));
  }
  CHECK(throws<std::out_of_range>([] { D::action_from_index(10); }));
  CHECK(D::observation_size(D::default_preset()) == R::observation_size(R::default_preset()));
}

template <class A, class B>
static double max_rel(const A& a, const B& b) {
  double m = 0.0;
  for (int i = 0; i < a.size(); ++i) {
    const double d = std::abs(a[i] - b[i]) / std::max(1e-300, std::max(std::abs(a[i]), std::abs(b[i])));
    if (std::abs(a[i] - b[i]) > 1e-15) m = std::max(m, d);
  }
  return m;
}

static void test_deterministic_and_calibrate() {
  // run_deterministic<double> (engine.hpp:225-245): the device runs the reference's fp64 arithmetic
  const Layers L = varied(29, 16, 16);
  R::SimConfig rc;
  D::SimConfig dc;
  R::FireLayer f(16, 16, R::FireState::Unburned);
  f(8, 8) = f(3, 12) = R::FireState::Burning;
  const R::ContinuousState rs = R::state_from_fire(f);
  const D::ContinuousState ds = D::state_from_fire(to_dev(f));
  const auto ra = R::run_deterministic(rs, ref_grid(L), rc, 60, true);
  const auto da = D::run_deterministic(ds, dev_grid(L), dc, 60, true);
  CHECK(da.trajectory.size() == ra.trajectory.size());
  CHECK(max_rel(ra.final_state.p_burn, da.final_state.p_burn) < 1e-12);
  CHECK(max_rel(ra.final_state.p_un, da.final_state.p_un) < 1e-12);
  CHECK(max_rel(ra.trajectory[30].p_bd, da.trajectory[30].p_bd) < 1e-12);
  const auto rf = R::fire_fraction_stats(ra.final_state);
  const auto df = D::fire_fraction_stats(da.final_state);
  CHECK(std::abs(rf.burning - df.burning) < 1e-12 && std::abs(rf.burned - df.burned) < 1e-12);
  const auto r1 = R::step_deterministic(rs, ref_grid(L), rc);
  const auto d1 = D::step_deterministic(ds, dev_grid(L), dc);
  CHECK(max_rel(r1.p_burn, d1.p_burn) == 0.0);
  R::DeterministicBatch rb;
  rb.members.assign(3, rs);
  D::DeterministicBatch db;
  db.members.assign(3, ds);
  for (int t = 0; t < 5; ++t) {
    R::step_batch(rb, ref_grid(L), rc);
    D::step_batch(db, dev_grid(L), dc);
  }
  CHECK(db.step == 5 && max_rel(rb.members[2].p_burn, db.members[2].p_burn) < 1e-12);
  CHECK(throws<std::invalid_argument>([&] {
    D::ContinuousState bad = ds;
    bad.p_un[0] = 0.5;
    D::validate_state(bad);
  }));
  // calibrate (calibrate.cpp:104-167): reference Dual<6> forward mode vs device reverse mode
  R::Grid<double> mask_r(16, 16);
  D::Grid<double> mask_d(16, 16);
  const auto tgt_run = R::run_deterministic(rs, ref_grid(L), R::config_from_params({0.22, 0.15, 0.3, 0.8, 1.1, 0.7}), 12);
  for (int i = 0; i < 256; ++i)
    mask_r[i] = mask_d[i] = (tgt_run.final_state.p_burn[i] + tgt_run.final_state.p_bd[i]) >= 0.5 ? 1.0 : 0.0;
  const R::CalibrationTarget rt{mask_r, 12};
  const D::CalibrationTarget dt{mask_d, 12};
  R::CalibrationOptions ro;
  D::CalibrationOptions dop;
  ro.iterations = dop.iterations = 8;
  ro.init_theta = {0.15, 0.2, 0.25, 1.1, 0.9, 0.6};
  dop.init_theta = {0.15, 0.2, 0.25, 1.1, 0.9, 0.6};
  const auto rres = R::calibrate(ref_grid(L), rs, rt, R::LossConfig{}, ro);
  const auto dres = D::calibrate(dev_grid(L), ds, dt, D::LossConfig{}, dop);
  CHECK(dres.loss_history.size() == rres.loss_history.size());
  for (std::size_t i = 0; i < rres.loss_history.size(); ++i)
    CHECK(std::abs(rres.loss_history[i] - dres.loss_history[i]) <= 1e-9 * std::abs(rres.loss_history[i]));
  for (int k = 0; k < 6; ++k) CHECK(std::abs(rres.best_theta[k] - dres.best_theta[k]) <= 1e-9);
  const auto lg = D::loss_and_gradient(dev_grid(L), ds, dt, D::LossConfig{}, D::config_from_params(dop.init_theta));
  CHECK(std::abs(lg.first - rres.loss_history[0]) <= 1e-12 * rres.loss_history[0]);
}

static void test_validation() {
  CHECK(throws<std::invalid_argument>([] { D::Grid<double>(0, 3); }));
  CHECK(throws<std::invalid_argument>([] { D::WindField::uniform(2, 2, -1.0, 0.0); }));
  CHECK(throws<std::invalid_argument>([] {
    D::FuelField(D::Grid<double>(2, 2, std::nan("")), D::Grid<double>(2, 2));
  }));
  D::SimConfig bad;
  bad.p_continue = 2.0;
  CHECK(throws<std::invalid_argument>([&] { D::validate_config(bad); }));
  CHECK(D::offset_index(D::NeighborOffset{-1, 1}) == 3);
  for (int k = 0; k < 8; ++k)
    CHECK(D::offset_angle(D::kNeighborOffsets[k]) == R::offset_angle(R::kNeighborOffsets[k]));
  CHECK(D::rng_word(D::RngKey{42, 7, 3}, 11, 0) == 0x9edc5135dc9b8a8eull);
}

int main() {
  test_validation();
  test_engine_matches_reference();
  test_run_and_record();
  test_wind_schedule();
  test_batches();
  test_rl_env();
  test_deterministic_and_calibrate();
  std::printf("dropin: %d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
