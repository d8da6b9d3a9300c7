/* TEST INFRASTRUCTURE ONLY — the CPU restatement ("port") of the reference's
 * batched CA fire-spread step.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it, and only as the
 * checker; the product library (libember_b200.so) never links or calls it.
 *
 * Pinned against: (1) the reference itself compiled in place
 * (oracle/_ref/libebl_ref.so, see oracle/Makefile) on every function below,
 * tests/test_oracle_pin.py; (2) the RNG known-answer vectors and C0 digests of
 * SURVEY §8(c), committed in tests/golden/.
 *
 * Conventions follow the reference: row-major H x W, row 0 = south
 * (grid.hpp:5-7), FireState uint8 {0 Unburned, 1 Burning, 2 Burned}
 * (grid.hpp:98), neighbour order E,NE,N,NW,W,SW,S,SE (grid.hpp:74-83),
 * config order (p_base, alpha_w1, alpha_w2, alpha_s, alpha_gamma, p_continue)
 * (grid.hpp:171-180). */
#ifndef EMBER_ORACLE_H
#define EMBER_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* rng.hpp:28-58 */
uint64_t ebo_rng_word(uint64_t seed, uint64_t step, uint64_t stream, uint64_t cell, uint64_t draw);
double ebo_rng_uniform(uint64_t seed, uint64_t step, uint64_t stream, uint64_t cell, uint64_t draw);
uint64_t ebo_rng_below(uint64_t seed, uint64_t step, uint64_t stream, uint64_t cell, uint64_t draw,
                       uint64_t n);

/* grid.cpp:35-47 */
double ebo_wrap_angle(double a);
double ebo_offset_angle(int k);

/* Static layers of one grid, as the reference's GridState holds them
 * (grid.hpp:105-157): per-cell wind speed/direction, veg/den, 8 slopes. */
typedef struct {
  int h, w;
  double *speed, *dir, *veg, *den, *slope8;
} ebo_grid;

/* Allocates a grid from layers (copies; wraps directions and clamps veg/den
 * exactly as WindField / FuelField construction does, grid.cpp:49-77). */
ebo_grid* ebo_grid_layers(int h, int w, const double* speed, const double* dir, const double* veg,
                          const double* den, const double* slope8);
/* Terrain form: slope from fp32 elevation (geodata.cpp:209-229), uniform wind. */
ebo_grid* ebo_grid_terrain(int h, int w, const double* veg, const double* den, const float* elev,
                           double cellsize, double speed, double dir);
void ebo_grid_free(ebo_grid* g);

/* SpreadTables<double> (engine.hpp:76-125): pot[cell*8+k], gamma[cell]. */
void ebo_tables(const ebo_grid* g, const double* cfg, double* pot, double* gamma);

/* kernel.hpp:53-78 evaluated directly (no tables) for every cell. */
void ebo_intensity(const ebo_grid* g, const double* cfg, const uint8_t* fire, double* lambda,
                   double* p);

/* One stochastic step (engine.cpp:12-38) with prebuilt tables. */
void ebo_step_tables(int h, int w, const double* pot, const double* gamma, double p_continue,
                     uint64_t seed, uint64_t step, uint64_t stream, const uint8_t* in, uint8_t* out);
/* run_stochastic (engine.cpp:101-120): tables built once, steps applied in place. */
void ebo_run(const ebo_grid* g, const double* cfg, uint64_t seed, uint64_t step0, uint64_t stream,
             int steps, uint8_t* state);
/* Per-env grids, OpenMP over envs (the C1 harness); returns wall seconds. */
double ebo_run_envs(ebo_grid* const* grids, int n_envs, const double* cfg, uint64_t seed,
                    const uint64_t* streams, int steps, uint8_t* states, int threads);

/* fire_fraction_stats counts (engine.cpp:185-198): counts[3] = U, B, X. */
void ebo_counts(const uint8_t* fire, int n, int32_t* counts);

/* ---- RL environment, reference semantics (rl_env.hpp/.cpp) ---- */
typedef struct {
  int height, width, window_radius, water_capacity;
  double burn_penalty;
  int max_episode_steps, ignition_count, waste_water;
  double wind_speed, wind_direction, fuel_veg, fuel_den;
  double spread[6];
} ebo_env_cfg;

typedef struct {
  int agent_row, agent_col, water, step;
  uint64_t seed, stream;
  int done;
} ebo_env_state;

int ebo_env_obs_size(const ebo_env_cfg* c);
void ebo_env_reset(const ebo_env_cfg* c, uint64_t seed, uint64_t stream, ebo_env_state* s,
                   uint8_t* fire);
/* returns 0, or -1 when stepping a finished episode (logic_error in the reference) */
int ebo_env_step(const ebo_env_cfg* c, const ebo_env_state* s, const uint8_t* fire, int action,
                 ebo_env_state* s_out, uint8_t* fire_out, double* reward, double* obs);
void ebo_env_observe(const ebo_env_cfg* c, const ebo_env_state* s, const uint8_t* fire,
                     double* obs);
int ebo_random_policy(uint64_t seed, uint64_t step, uint64_t stream);

/* ---- air-tanker RL step (BASELINE C2 semantics) ---- */
typedef struct {
  int ignitions;       /* ignitions per (re)set, at burnable cells */
  int max_steps;       /* episode cap (256) */
  int autoreset;       /* 1: a finished env restarts with episode+1 */
} ebo_tanker_cfg;

typedef struct {
  int step;            /* episode-local step (RNG step index) */
  uint32_t episode;    /* RNG stream = episode << 32 | env_id */
  int done;
} ebo_tanker_state;

/* Burnable = (1+veg)*(1+den) > 0 at the cell (source and gamma both > 0). */
void ebo_tanker_reset(const ebo_grid* g, const ebo_tanker_cfg* tc, uint64_t seed, uint32_t env_id,
                      uint32_t episode, ebo_tanker_state* s, uint8_t* fire, uint8_t* wet);
/* One step for one env: action = row*W + col.  tables from ebo_tables(g). */
void ebo_tanker_step(const ebo_grid* g, const double* pot, const double* gamma, double p_continue,
                     const ebo_tanker_cfg* tc, uint64_t seed, uint32_t env_id, int action,
                     ebo_tanker_state* s, uint8_t* fire, uint8_t* wet, float* reward,
                     uint8_t* done);
int ebo_tanker_policy(uint64_t seed, uint32_t env_id, const ebo_tanker_state* s, int n_cells);

/* ---- deterministic (raw-probability) mode, engine.hpp:147-175 ---- */
void ebo_det_step_tables(int h, int w, const double* pot, const double* gamma, double p_continue,
                         const double* un, const double* burn, const double* bd, double* un_o,
                         double* burn_o, double* bd_o);
/* run_deterministic<double> from an arbitrary continuous state (in place). */
void ebo_det_run(const ebo_grid* g, const double* cfg, int steps, double* un, double* burn,
                 double* bd);
/* C4 gradient oracle: run_deterministic<Dual<6>> + loss (calibrate.hpp:120-146) from a discrete
 * initial layer, theta = the 6 SimConfig fields; grad6 = d loss / d theta. */
void ebo_det_loss_grad(const ebo_grid* g, const double* cfg, int steps, const uint8_t* fire0,
                       const double* mask, double bce_w, double mse_w, int pool, double* loss_out,
                       double* grad6);

/* calibrate (calibrate.cpp:104-167): Adam on ThetaTransform-unconstrained parameters, each
 * iteration a Dual<6> deterministic rollout of `horizon` steps from the continuous initial
 * state + loss.  loss_hist [iterations+1], theta_hist [(iterations+1)*6].  0 / -1 non-finite /
 * -2 bad init_theta. */
/* serialize_snapshot (snapshot.cpp:55-70): header, H lines northmost first ({U,B,X}, other
 * bytes '?'), optional agent line (ar < 0: none).  Returns the length; writes at most cap bytes. */
long ebo_snapshot_text(int h, int w, const uint8_t* fire, uint64_t step, int ar, int ac, int water, char* out,
                       long cap);
int ebo_calibrate(const ebo_grid* g, const double* un0, const double* bu0, const double* bd0,
                  const double* mask, int horizon, double bce_w, double mse_w, int pool,
                  int iterations, const double* init_theta, const int* optimize, double lr,
                  double* loss_hist, double* theta_hist, double* best_theta, double* best_loss);

/* The benchmark's synthetic inputs (not a reference function), restated so
 * the CPU arms never load the product library; pinned to ebl_synth_terrain/_ignitions. */
void ebo_synth_terrain(uint64_t seed, uint32_t env_id0, int n_envs, int h, int w, double elev_max,
                       double wind_max, uint8_t* fuel_class, float* elevation, double* wind_speed,
                       double* wind_direction);
void ebo_worldcover_palette(int32_t* codes, double* veg, double* den);
int ebo_synth_ignitions(uint64_t seed, uint32_t env_id0, int n_envs, int h, int w,
                        const uint8_t* fuel_class, const double* class_veg, const double* class_den,
                        int count, uint8_t* states);

/* CPU-baseline harness for C2: the tanker step over n envs, OpenMP over envs (see .c). */
double ebo_tanker_run_envs(ebo_grid* const* grids, int n_envs, const double* cfg,
                           const ebo_tanker_cfg* tc, uint64_t seed, uint32_t env_id0,
                           const uint32_t* env_ids, int steps, int threads, double* reward_sum,
                           uint8_t* fire_out, uint8_t* wet_out, double* env_reward, int32_t* env_episodes);

#ifdef __cplusplus
}
#endif
#endif
