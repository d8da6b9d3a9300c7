/* ember_b200.h — C-ABI of the B200 fire-spread engine (libember_b200.so).
 *
 * The reference (emberline, /root/reference/proj) has no FFI: its interface is
 * the C++ header API in proj/include/emberline/.  Every entry point below is the
 * flat-pointer form of one reference function or type on the north-star path,
 * cited as file:line; include/emberline_b200.hpp wraps them back into the
 * reference's C++ signatures (the drop-in), and paper_2512_06102_b200/_lib.py binds
 * them with ctypes (INTEGRATION.md shows both bindings).
 *
 * Conventions (identical to the reference):
 *  - a grid is H x W row-major, index row*W + col, row 0 = south (grid.hpp:5-7,42);
 *  - cell state is uint8 {0 Unburned, 1 Burning, 2 Burned} (grid.hpp:98);
 *  - a batch is B envs stored batch-major [env][row][col] ("members", engine.hpp:250-258);
 *  - config doubles in the order of BasicSimConfig (grid.hpp:171-180);
 *  - the RNG key of env e at lockstep step t is {seed, t, stream[e]} (rng.hpp:15-19,
 *    engine.cpp:145), draw domain kDrawFireEvent, cell index = row*W + col.
 *
 * Errors: every function returning int returns 0 on success and a negative
 * EBL_E* code on failure; ebl_last_error() gives the message (thread-local).
 * The C++ wrapper rethrows the reference's exception types (std::invalid_argument
 * for EBL_EINVAL, std::logic_error for EBL_ELOGIC, std::out_of_range for
 * EBL_ERANGE), matching grid.cpp:18-24, engine.cpp:124, rl_env.cpp:60-93,173.
 * There is no CPU fallback: without a usable CUDA device ebl_batch_create fails
 * with EBL_ECUDA. */
#ifndef EMBER_B200_H
#define EMBER_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EBL_OK 0
#define EBL_EINVAL -1 /* std::invalid_argument */
#define EBL_ELOGIC -2 /* std::logic_error */
#define EBL_ERANGE -3 /* std::out_of_range */
#define EBL_ECUDA -4  /* device / driver failure */
#define EBL_ESTATE -5 /* call order (e.g. stepping before a grid is set) */
#define EBL_ENUMERIC -6 /* NumericalError (errors.hpp:14-17) */
#define EBL_EFILE -7    /* FileError (errors.hpp:9-12), e.g. an unmapped landcover code */

#define EBL_ABI_VERSION 1

typedef struct ebl_batch ebl_batch; /* opaque: one device, one stream, B envs of H x W */

/* BasicSimConfig<double> (grid.hpp:171-180). */
typedef struct {
  double p_base, alpha_w1, alpha_w2, alpha_s, alpha_gamma, p_continue;
  int max_steps;
} ebl_sim_config;

int ebl_abi_version(void);
const char* ebl_last_error(void);
/* validate_config (grid.cpp:107-124). */
int ebl_validate_config(const ebl_sim_config* cfg);
void ebl_default_config(ebl_sim_config* cfg);

/* ---- batch lifetime: the device-resident StochasticBatch (engine.hpp:250-261) ---- */
/* `cuda_stream` may be NULL (library-owned stream) or a cudaStream_t to launch on. */
int ebl_batch_create(ebl_batch** out, int device, int n_envs, int height, int width,
                     void* cuda_stream);
void ebl_batch_destroy(ebl_batch* b);
int ebl_batch_set_config(ebl_batch* b, const ebl_sim_config* cfg);

/* Static layers, form 1 — a general GridState (grid.hpp:192-211): per-cell wind
 * speed/direction, veg/den, 8 slopes per cell ([cell*8+k], kNeighborOffsets order).
 * n_grids = 1 (all members share one grid, as StochasticBatch does) or n_envs.
 * Built into SpreadTables<double> (engine.hpp:76-125) in fp64 on the host and
 * kept resident; rebuilt when the config changes. Validation as in
 * WindField/FuelField/SlopeField/GridState construction (grid.cpp:49-142). */
int ebl_batch_set_grid(ebl_batch* b, int n_grids, const double* wind_speed,
                       const double* wind_direction, const double* veg, const double* den,
                       const double* slope8);

/* Static layers, form 2 — terrain (the north-star layout): per-cell uint8 fuel
 * class into a palette of (veg, den) pairs (FuelTable, geodata.hpp:63-86), fp32
 * elevation in metres from which the 8 slopes are derived on the fly exactly as
 * slope_from_dem does (geodata.cpp:209-229) at `cellsize`.  n_grids = 1 or n_envs.
 * A NaN elevation is a DEM nodata cell: slope 0 from and toward it (geodata.cpp:214,220). */
int ebl_batch_set_terrain(ebl_batch* b, int n_grids, const uint8_t* fuel_class,
                          const float* elevation, int n_classes, const double* class_veg,
                          const double* class_den, double cellsize);
/* fuel_from_landcover / grid_from_rasters (geodata.cpp:324-369) on the device: int32
 * landcover codes [n_grids][H*W] (model order) are mapped through a FuelTable (codes[k] ->
 * (veg[k], den[k]); a repeated code keeps its last entry; optional fallback for unknown
 * codes) into the terrain form's palette.  Landcover nodata (has_nodata && code ==
 * nodata_code) and DEM nodata (NaN elevation) cells become inert (-1, -1) and the latter get
 * slope 0.  Errors: EBL_EINVAL for modifiers outside [-1, 1] (FuelTable::set), EBL_EFILE
 * naming the first unmapped code when there is no fallback (FuelTable::lookup). */
int ebl_batch_set_landcover(ebl_batch* b, int n_grids, const int32_t* landcover,
                            const float* elevation, int has_nodata, int32_t nodata_code,
                            int n_codes, const int32_t* codes, const double* veg,
                            const double* den, int has_fallback, double fallback_veg,
                            double fallback_den, double cellsize);
/* The C1 generator (ebl_synth_terrain below) run on the device straight into the batch:
 * per-env terrain (n_grids = n_envs, env e on stream env_id0 + e), the WorldCover palette,
 * per-env wind; bit-identical to ebl_synth_terrain.  n_envs <= 65535. */
int ebl_batch_synth_terrain(ebl_batch* b, uint64_t seed, uint32_t env_id0, double elev_max,
                            double wind_max, double cellsize);
/* ebl_synth_ignitions on the device into the batch state (terrain form; every env zeroed
 * first).  *placed_total (may be NULL) receives the number of ignitions placed. */
int ebl_batch_synth_ignitions(ebl_batch* b, uint64_t seed, uint32_t env_id0, int count,
                              int* placed_total);
/* Terrain-form layers back to the host: fuel_class / elevation [n_grids][H*W]; either may
 * be NULL. */
int ebl_batch_get_terrain(ebl_batch* b, uint8_t* fuel_class, float* elevation);

/* Spatially uniform wind per env (WindField::uniform, grid.cpp:64-66) for the
 * terrain form; n_winds = 1 or n_envs. */
int ebl_batch_set_wind(ebl_batch* b, int n_winds, const double* speed, const double* direction);

/* Member fire layers, host <-> device, [n_envs][H*W] uint8.  Like the reference's FireLayer
 * they are not validated: a byte other than 1 (Burning) / 2 (Burned) steps as Unburned
 * (engine.cpp:15-25) and is written back as 0 or 1. */
int ebl_batch_set_state(ebl_batch* b, const uint8_t* states);
int ebl_batch_get_state(ebl_batch* b, uint8_t* states);
/* Same, device pointers (no host round trip). */
int ebl_batch_set_state_device(ebl_batch* b, const void* d_states);
int ebl_batch_get_state_device(ebl_batch* b, void* d_states);
/* Device pointer of the current state buffer (valid until the next step). */
void* ebl_batch_state_device_ptr(ebl_batch* b);

/* RNG identity: StochasticBatch::seed/step and Member::stream (engine.hpp:250-258).
 * streams == NULL means stream[e] = first_stream + e (make_stochastic_batch,
 * engine.cpp:122-132). */
int ebl_batch_set_key(ebl_batch* b, uint64_t seed, uint64_t step, const uint64_t* streams,
                      uint64_t first_stream);
uint64_t ebl_batch_step_index(const ebl_batch* b);

/* step_batch (engine.cpp:134-159) applied n_steps times: step t uses key
 * {seed, step+t, stream[e]}; the batch step counter advances by n_steps. */
int ebl_step_batch(ebl_batch* b, int n_steps);

/* make_stochastic_batch + step_batch x n_steps + reading the members back (engine.cpp:122-159,
 * emberline_main.cpp:417-424), from and to HOST buffers [n_envs][H*W]: identical to
 * ebl_batch_set_state + ebl_step_batch + ebl_batch_get_state, but pipelined over env chunks
 * (chunk c's host->device copy, its fused launch and its device->host copy overlap the other
 * chunks' work).  Returns when final_states is written.  Pinned host memory makes the copies
 * asynchronous. */
int ebl_batch_run(ebl_batch* b, const uint8_t* initial, int n_steps, uint8_t* final_states);
/* Number of env chunks ebl_batch_run pipelines over (0 = auto, 4; 1 = no pipelining). */
int ebl_batch_set_pipeline(ebl_batch* b, int chunks);

/* run_stochastic(record=true) (engine.cpp:108,116): ebl_step_batch that also stores the layers
 * after every step into traj [n_steps][n_envs][H*W] (device pointer when on_device, else host;
 * the initial layers are the caller's).  The blocked kernel writes them from shared memory as
 * it goes: no per-step launches or host syncs. */
int ebl_step_batch_record(ebl_batch* b, int n_steps, void* traj, int on_device);

/* WindSchedule (engine.hpp:188-199, engine.cpp:74-86) on the device: step t of a run uses the
 * entry min(t, n_sched - 1) of the absolute step index t (run_stochastic, engine.cpp:110-112).
 * Terrain form: uniform winds speed/dir [n_sched][n_winds] (n_winds = 1 or n_envs); n_sched = 0
 * sets a constant wind.  General form: per-cell WindFields [n_sched][n_grids][H*W]; the fp64
 * SpreadTables are built once per entry. */
int ebl_batch_set_wind_schedule(ebl_batch* b, int n_sched, int n_winds, const double* speed,
                                const double* direction);
int ebl_batch_set_grid_wind_schedule(ebl_batch* b, int n_sched, const double* speed,
                                     const double* direction);

/* Kernel selection for ebl_step_batch (results are identical by construction):
 *  AUTO      the warp-local kernel: one CTA per env with all n steps fused when an env fits
 *            shared memory (H*W <= 65536), else light-cone-halo tiles, 8 steps per launch;
 *            rows dealt to warps, each warp deciding its own rows' active cells, one block
 *            barrier per step; regions without a burning cell skip their steps, and tiles
 *            quiet for two launches of one call are skipped outright;
 *  WARP      the same as AUTO;
 *  TILED     the per-cell tile kernel, one step per launch (independent implementation);
 *  RESIDENT  the pooled-list blocked kernel, whole env per CTA (error if it does not fit);
 *  BLOCKED   the pooled-list blocked kernel with halo tiles even when the env would fit. */
#define EBL_KERNEL_AUTO 0
#define EBL_KERNEL_TILED 1
#define EBL_KERNEL_RESIDENT 2
#define EBL_KERNEL_BLOCKED 3
#define EBL_KERNEL_WARP 6
/* (4, 5 and 7 named kernel variants measured slower than WARP and removed; set_kernel rejects
 * them with EBL_EINVAL) */
int ebl_batch_set_kernel(ebl_batch* b, int which);
/* Explicit tiling of the blocked kernel (tile_h rows x tile_w cols, tile_w a multiple of
 * 32, `halo` rows of light cone = steps per launch); tile_h == 0 restores planning. */
int ebl_batch_set_tiling(ebl_batch* b, int tile_h, int tile_w, int halo);

/* ---- row-sharded landscapes (BASELINE C3) ----
 * A shard's layer holds global rows [row_off, row_off + H): its band plus light-cone halo
 * rows.  The RNG cell index stays global ((row_off + r) * W + c), so a sharded run is
 * bit-identical to the unsharded one. */
int ebl_batch_set_row_offset(ebl_batch* b, int64_t row_off);
/* Layer rows [row_lo, row_hi) this shard owns (its band; the rest of its layer is halo). */
int ebl_batch_set_band(ebl_batch* b, int row_lo, int row_hi);
/* Steps n_shards row shards of one landscape (bands in order, one env each, halo-tiled blocked
 * kernel with `halo` rows of light cone) by n_steps, `halo` steps per launch, with the halo
 * exchange fused into the kernels: each launch stores the band rows its neighbours hold as halo
 * straight into their output layers (peer stores over NVLink between GPUs), and each shard's
 * stream waits on its neighbours' previous launch (events, no host synchronisation).
 * Bit-identical to the unsharded run.  Replaces the step + ebl_batch_copy_rows loop. */
int ebl_shards_step(ebl_batch** shards, int n_shards, int n_steps, int halo);
/* Copies rows [src_row, src_row+n) of every member of `src` into rows [dst_row, ...) of `dst`
 * (same width and member count); batches on different devices copy peer-to-peer over
 * NVLink (cudaMemcpyPeerAsync) on dst's stream after src's stream has drained. */
int ebl_batch_copy_rows(ebl_batch* dst, int dst_row, const ebl_batch* src, int src_row, int n_rows);
/* Rows [row0, row0+n) of every member to (to_batch = 0) or from (1) a device buffer
 * [n_envs][n][W] (e.g. a torch tensor exchanged with NCCL send/recv between processes). */
int ebl_batch_rows_device(ebl_batch* b, int row0, int n_rows, void* dptr, int to_batch);

/* fire_fraction_stats (engine.cpp:185-198) as integer counts of the current
 * state, out[e*4 + {0,1,2,3}] = {unburned, burning, burned, newly ignited in the
 * last step}. */
int ebl_batch_counts(ebl_batch* b, int32_t* out);

/* Per-cell arrival intensity and ignition probability of the current state
 * (kernel.hpp:53-78, the fp32 fast path): lambda/p [n_envs][H*W] float. */
int ebl_batch_intensity(ebl_batch* b, float* lambda, float* p);
/* The same probe for one fp32 form of the terrain path: record_form = 1 the slope / source-class
 * record form the resident kernels use (the ebl_batch_intensity default when the palette has <= 32
 * classes), 0 the on-the-fly form from the elevation layer (halo tiles, tiled kernel). */
int ebl_batch_intensity_form(ebl_batch* b, int record_form, float* lambda, float* p);

/* Diagnostics since the last reset: [0] draws decided in the fp64 guard band,
 * [1] draws within 1e-12 of their fp64 threshold ("ambiguous": a flip vs the
 * CPU reference is only possible here), [2] steps, [3] kernel
 * launches issued. */
int ebl_batch_diag(ebl_batch* b, uint64_t* out4, int reset);
/* Tile statistics of the warp-local kernel since the last reset: [0] regions (CTAs) that loaded
 * and stepped or stored their tile, [1] regions launched (the rest were quiet tiles skipped
 * outright).  Their ratio is the share of the dense cell-updates actually visited. */
int ebl_batch_tile_stats(ebl_batch* b, uint64_t* out2, int reset);
/* Phase profile of the resident blocked kernel (diagnostic builds with -DEBL_PHASE_PROF=1 only;
 * otherwise set_profiling(on) fails with EBL_ESTATE): each launch stores per env int64
 * [n_envs][10] = {P1 cycles (to the first barrier), P2 cycles (to the second), active cells,
 * steps, slowest warp's dense-pass cycles, slowest warp's list-build cycles, slowest warp's P2
 * work cycles, candidate decisions, list build: count done, reservation done}, summed over the
 * launch's steps (clock64, the env's CTA). */
int ebl_batch_set_profiling(ebl_batch* b, int on);
int ebl_batch_profile(ebl_batch* b, int64_t* out);
/* rng_word (rng.hpp:38-46) evaluated ON THE DEVICE for n keys
 * keys5[i*5 + {0..4}] = {seed, step, stream, cell, draw}; the parity probe of the
 * device generator (device 0). */
int ebl_device_rng_words(int n, const uint64_t* keys5, uint64_t* out);

/* serialize_snapshot (snapshot.cpp:55-70) of n layers, concatenated: "emberline-snapshot v1 H W
 * step", H lines of W chars from {U,B,X} (northmost row first; other byte values '?'), then
 * "agent row col water" when agents[3*i] >= 0.  layers_dev: n_layers device layers of the batch's
 * H x W (e.g. an ebl_step_batch_record trajectory), or NULL for the batch's current layers
 * (n_layers ignored).  steps[i] (NULL: the batch step).  *len = the text's bytes; out = NULL
 * queries the size; cap < *len is EBL_ERANGE.  Bodies are rendered on the device. */
int ebl_batch_snapshot_text(ebl_batch* b, const void* layers_dev, int n_layers, const uint64_t* steps,
                            const int32_t* agents, char* out, size_t cap, size_t* len);
/* parse_snapshot (snapshot.cpp:74-121) of one snapshot text: dimensions, step, layer (row 0 =
 * south; NULL to validate only), agent (has_agent).  FileError cases -> EBL_EFILE with the
 * reference's messages. */
int ebl_snapshot_parse(const char* text, size_t text_len, int* h, int* w, uint64_t* step, uint8_t* layer,
                       size_t layer_cap, int32_t* agent3, int* has_agent);

/* Pinned, mapped host staging memory in 2 MiB transparent huge pages for the host-buffer entry
 * points (ebl_batch_run, set/get_state): robust full-rate DMA, and ebl_batch_run writes the final
 * layers into it straight from the kernel.  No reference counterpart (the reference is host-only). */
int ebl_host_alloc(size_t bytes, void** out);
int ebl_host_free(void* p);
int ebl_batch_sync(ebl_batch* b);

/* ---- one-shot entry points (exact reference signatures, host buffers) ---- */
/* step_stochastic(fire, grid, cfg, key) (engine.hpp:204-207) on general layers. */
int ebl_step_stochastic(int height, int width, const uint8_t* fire, const double* wind_speed,
                        const double* wind_direction, const double* veg, const double* den,
                        const double* slope8, const ebl_sim_config* cfg, uint64_t seed,
                        uint64_t step, uint64_t stream, uint8_t* out);
/* run_stochastic(initial, grid, cfg, key, steps) (engine.hpp:215-217), final state only. */
int ebl_run_stochastic(int height, int width, const uint8_t* initial, const double* wind_speed,
                       const double* wind_direction, const double* veg, const double* den,
                       const double* slope8, const ebl_sim_config* cfg, uint64_t seed,
                       uint64_t step, uint64_t stream, int steps, uint8_t* out);

/* ---- deterministic (raw-probability) mode and its gradient (BASELINE C4) -------- */
/* BasicContinuousState (engine.hpp:27-37) of every env as fp64 planes [n_envs][H*W]. */
int ebl_det_set_state(ebl_batch* b, const double* p_un, const double* p_burn, const double* p_bd);
/* state_from_fire (engine.cpp:42-52) of the batch's current fire layers. */
int ebl_det_set_state_from_fire(ebl_batch* b);
int ebl_det_get_state(ebl_batch* b, double* p_un, double* p_burn, double* p_bd);
/* run_deterministic (engine.hpp:225-245) for n_steps on the terrain statics, in the
 * reference's fp64 arithmetic on the device (DESIGN.md §4 explains why not fp32); record = 1
 * keeps (p_un, p_burn) of every step in HBM for ebl_det_loss_grad. */
/* Where the terrain-form SpreadTables<double> of the deterministic path are built: on the device
 * (default: the config-free fp64 slopes cached once per terrain, pot = (source kappa_wind)
 * exp(alpha_s S) with a restatement of the reference libm's exp, bit-identical to the host build,
 * so calibration iterations need no host table build) or on the host (on_device = 0). */
int ebl_batch_set_det_tables(ebl_batch* b, int on_device);
int ebl_det_forward(ebl_batch* b, int n_steps, int record);
/* loss = bce_w * BCE(clamp(pred)) + mse_w * MSE(avgpool(pred, pool), avgpool(mask, pool)),
 * pred = p_burn + p_bd (calibrate.hpp:86-146), per env, and its gradient with respect to
 * the six SimConfig fields in ParamIndex order (calibrate.hpp:21-28) by reverse mode
 * through the recorded steps (the reference computes it forward-mode with Dual<6>,
 * calibrate.cpp:130-162).  mask [n_envs][H*W], or NULL for the target ebl_det_set_mask made
 * resident (a calibration's fixed target: uploaded once, not per iteration); loss [n_envs];
 * grad6 [n_envs*6]. */
/* Upload the target burn mask [n_envs][H*W] (CalibrationTarget::burn_mask) once. */
int ebl_det_set_mask(ebl_batch* b, const double* mask);
int ebl_det_loss_grad(ebl_batch* b, const double* mask, double bce_w, double mse_w, int pool,
                      double* loss, double* grad6);

/* CalibrationOptions (calibrate.hpp:158-166). */
typedef struct {
  int iterations;
  double init_theta[6]; /* constrained space, ParamIndex order */
  int optimize[6];
  double lr;
  int max_horizon;
} ebl_calib_options;
void ebl_default_calib_options(ebl_calib_options* o);
/* calibrate(grid, initial, target, lc, opts) (calibrate.cpp:104-167): Adam on the
 * ThetaTransform-unconstrained parameters; every iteration a device deterministic rollout of
 * `horizon` steps from the continuous initial state [n_envs][H*W], the loss and its reverse-mode
 * gradient (summed over the batch's envs, which share theta; n_envs = 1 is the reference's call).
 * loss_hist [iterations+1], theta_hist [(iterations+1)*6].  Errors as the reference:
 * EBL_EINVAL (invalid_argument), EBL_ENUMERIC (NumericalError).  Restores the batch config. */
int ebl_calibrate(ebl_batch* b, const double* p_un, const double* p_burn, const double* p_bd,
                  const double* mask, int horizon, double bce_w, double mse_w, int pool,
                  const ebl_calib_options* opt, double* loss_hist, double* theta_hist,
                  double* best_theta, double* best_loss);

/* ---- RL (rl_env.hpp) ---------------------------------------------------------- */
/* EnvConfig (rl_env.hpp:24-40). */
typedef struct {
  int height, width, window_radius, water_capacity;
  double burn_penalty;
  int max_episode_steps, ignition_count, waste_water;
  double wind_speed, wind_direction, fuel_veg, fuel_den;
  ebl_sim_config spread;
} ebl_env_config;

/* EnvState minus the fire layer (rl_env.hpp:67-75). */
typedef struct {
  int32_t agent_row, agent_col, water, step;
  uint64_t seed, stream;
  int32_t done;
  uint32_t episode; /* tanker episode counter (RNG stream = episode << 32 | env id) */
} ebl_env_state;

#define EBL_RL_REFERENCE 0 /* FireSuppressionEnv semantics: Move x Valve, single-cell douse */
#define EBL_RL_TANKER 1    /* BASELINE C2: (x,y) action, 3x3 extinguish+wet, auto-reset */

void ebl_env_default_preset(ebl_env_config* c); /* default_preset, rl_env.cpp:10-27 */
void ebl_env_smoke10_preset(ebl_env_config* c); /* smoke10_preset, rl_env.cpp:29-57 */
int ebl_env_observation_size(const ebl_env_config* c); /* rl_env.cpp:73-76 */

/* Puts the batch in RL mode.  EBL_RL_REFERENCE: the batch's statics become the
 * config's flat terrain (rl_env.cpp:99-105).  EBL_RL_TANKER: statics must be
 * set (terrain form), `ignitions` per reset at burnable cells, `max_steps` cap,
 * auto-reset on.  Env e has id env_id0 + e. */
int ebl_rl_configure(ebl_batch* b, int variant, const ebl_env_config* c, int tanker_ignitions,
                     int tanker_max_steps, uint32_t env_id0);
/* FireSuppressionEnv::reset (rl_env.cpp:125-145) of every env (mask[e] != 0, or all
 * when mask == NULL).  REFERENCE: streams[e] (NULL: env id). TANKER: episode 0. */
int ebl_rl_reset(ebl_batch* b, uint64_t seed, const uint64_t* streams, const uint8_t* mask);
/* One step of every env: FireSuppressionEnv::step (rl_env.cpp:172-210) or the tanker
 * step.  actions[e]: REFERENCE action_index (rl_env.hpp:62-64) in [0,10);
 * TANKER row*W+col.  actions == NULL: the device-side random policy
 * (random_policy, rl_env.cpp:237-239 / uniform (x,y) for TANKER).  reward/done
 * may be NULL; host pointers unless `device_io` is 1.  Returns EBL_ELOGIC if a
 * REFERENCE env is already done (rl_env.cpp:173).  TANKER: the layers stay bit-resident
 * between consecutive calls; any other call that reads or writes them rebuilds the bytes;
 * host reward/done buffers in mapped pinned memory (ebl_host_alloc) are written by the kernel
 * through the mapping (no copy after the step); either way they are complete on return. */
int ebl_rl_step(ebl_batch* b, const int32_t* actions, double* reward, uint8_t* done, int device_io);
/* Tanker fused rollout: n_steps random-policy steps on device, rewards summed
 * into reward_sum[e] (host), episodes finished counted into episodes[e]. */
int ebl_rl_rollout(ebl_batch* b, int n_steps, double* reward_sum, int32_t* episodes);
/* Observation (rl_env.cpp:147-170): [n_envs][observation_size] doubles (REFERENCE). */
int ebl_rl_observe(ebl_batch* b, double* obs);
int ebl_rl_get_env_states(ebl_batch* b, ebl_env_state* out);
int ebl_rl_set_env_states(ebl_batch* b, const ebl_env_state* in);
int ebl_rl_get_wet(ebl_batch* b, uint8_t* wet);
/* TANKER observation for a learner on the device: [n_envs][H][W] bytes into out_dev (device
 * memory), FireState in bits 0-1, wet flag in bit 2; asynchronous on the batch stream, reads the
 * bit-resident state without invalidating it.  With ebl_rl_step(device_io = 1) the whole
 * act -> step -> observe loop stays on the device (no host round trip). */
int ebl_rl_observe_device(ebl_batch* b, void* out_dev);

/* ---- input preparation (BASELINE configs; not part of the reference API) ---- */
/* Synthetic per-env terrain for C1-C4: landcover class from
 * 4-octave value noise thresholded at 11 equal quantiles into the WorldCover codes,
 * fractal elevation in [0, elev_max] m, per-env uniform wind V~U(0,vmax),
 * dir~U(0,2pi), all keyed by the reference RNG in domain kDrawSynthesis.
 * fuel_class [n_envs][H*W] holds palette indices 0..10 (codes 10..100); wind may be
 * NULL. Env e uses stream env_id0 + e. */
int ebl_synth_terrain(uint64_t seed, uint32_t env_id0, int n_envs, int height, int width,
                      double elev_max, double wind_max, uint8_t* fuel_class, float* elevation,
                      double* wind_speed, double* wind_direction);
/* The WorldCover palette of default_worldcover_table (geodata.cpp:305-319):
 * codes[11], veg[11], den[11]. */
void ebl_worldcover_palette(int32_t* codes, double* veg, double* den);
/* `count` ignitions at uniform burnable cells (veg>-1, den>-1 after lookup) per
 * env via rng_below(key{seed,0,env_id0+e}, counter++, kDrawEnvSetup, H*W),
 * redrawing duplicates; states [n_envs][H*W] are zeroed first. */
int ebl_synth_ignitions(uint64_t seed, uint32_t env_id0, int n_envs, int height, int width,
                        const uint8_t* fuel_class, const double* class_veg,
                        const double* class_den, int count, uint8_t* states);

#ifdef __cplusplus
}
#endif
#endif /* EMBER_B200_H */
