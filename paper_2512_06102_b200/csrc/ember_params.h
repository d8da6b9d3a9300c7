// Launch parameter blocks shared by the host launcher (ember_capi.cu) and the
// kernels (ember_kernels.cu).  Plain structs, passed by value as kernel params.
#pragma once
#include <cstddef>
#include <cstdint>

namespace ebl {

enum StaticMode : int { kStaticNone = 0, kStaticTables = 1, kStaticTerrain = 2 };

// Everything one stochastic step of the whole batch needs.  Per-env statics are
// addressed as base + env * stride (stride 0 = one grid shared by all members,
// the StochasticBatch layout of engine.hpp:250-258).
struct StepArgs {
  int h, w, n_envs;
  uint64_t seed;
  uint64_t step;                  // lockstep step index t (RngKey::step)
  long long row_off;              // global row of layer row 0 (row shards): RNG cell = (row_off+r)*W+c
  const uint64_t* streams;        // [n_envs] Member::stream
  uint64_t pc_thr;                // Burning survives iff (word>>11) < pc_thr (= ceil(p_continue*2^53))
  const uint8_t* in;              // [n_envs][h*w]
  uint8_t* out;
  int32_t* counts;                // [n_envs][4] U,B,X,newly (nullable)
  // halo-tiled launches: per-tile activity records [env][tile] {bit0 burning in the output tile,
  // bits 1-2 quiet streak (saturating at 2), U, B, X}; read from the previous launch (null: no
  // valid records), written for the next.  Tiles whose output rows reach outside
  // [keep_lo, keep_hi) (row shards: halo rows a neighbour writes) are never skipped outright.
  const int32_t* tflag_in;        // int4 records
  int32_t* tflag_out;
  unsigned long long* diag;       // [4] fp64 fallbacks, ambiguous draws, tiles processed, launched
  // general form (SpreadTables)
  const double* pot;              // [grid][h*w*8]
  const double* gamma;            // [grid][h*w]
  size_t tab_stride;              // cells per grid, or 0
  // terrain form
  const uint8_t* fuel;            // [grid][h*w]
  const float* elev;              // [grid][h*w]
  const float* slope32;           // [grid][h*w][8] fp32 slope table (terrain form) or null
  const uint2* nfuel;             // [grid][h*w] fuel classes of the 8 sources u_k = v - d_k (bytes k)
  const float* pot32t;            // [env][h*w][8] fp32 pot of source u_k into target v (terrain form,
                                  // one wind per env; null with a wind schedule): the lambda terms
  size_t pot32t_stride;           // floats per env of pot32t (0: one table for all envs)
  int n_pal;                      // palette entries in use (terrain form)
  float alpha_s_l2;               // alpha_s * log2(e): kappa_slope = 2^(alpha_s_l2 * S)
  int rec_probe;                  // k_intensity: report the record form (1) or the elevation form (0)
  size_t ter_stride;
  const float* pal32;             // [2][256] src32, gam32
  const double* pal64;            // [2][256] src64, gam64
  const float* kw32;              // [wind][8]
  const double* kw64;
  int kw_stride;                  // 8 or 0
  int sched_len;                  // wind schedule entries (0/1: constant wind)
  size_t kw_sched_stride;         // kw elements per schedule entry (terrain form)
  size_t pot_sched_stride;        // pot elements per schedule entry (general form)
  uint8_t* traj;                  // [step][env][cell] states after each step (record), or null
  size_t traj_t0;                 // trajectory slot of this launch's first step
  float alpha_s32;
  double alpha_s;
  float inv_dist32[2];
  double dist64[2];
  int force64;
  long long* prof;                // [n_envs][10] phase profile (EBL_PHASE_PROF builds), or null
  uint8_t* out2;                  // [n_envs][h*w] second copy of the output (e.g. mapped pinned host memory), or null
  // row shards (ebl_shards_step): the layer rows this launch writes back, and up to two peer
  // layers (a neighbour shard's output buffer, possibly on another GPU over NVLink) that receive
  // rows [peer_lo, peer_hi) of this layer at their row peer_dst -- the halo exchange fused into
  // the producing kernel's store
  int store_lo, store_hi;
  int keep_lo, keep_hi;           // rows outside: halo rows written by neighbour shards (exposed tiles
                                  // unless halo_marked)
  // work-list runs of halo tiles (one batch, ebl_step_batch): list_mode 1 = grid launch, 2 = the
  // launch runs the tiles of tile_list[0 .. *tile_count) on persistent CTAs (list_cursor: the
  // claim counter); both keep the tile records in place (trec, int4 per tile) and append the next
  // launch's tiles to next_list / next_count, deduplicated by stamping queued[tile] = list_stamp
  int list_mode;
  int32_t* trec;
  int32_t* queued;
  int32_t list_stamp;
  int32_t* next_list;
  int32_t* next_count;
  const int32_t* tile_list;
  const int32_t* tile_count;
  int32_t* list_cursor;
  int32_t* list_zero0;            // counters the launch after next uses: zeroed by this launch
  int32_t* list_zero1;
  int tiles_x, tiles_y, tiles_total;
  int early_exit;                 // whole-env C1/64^2 launches: the instantiation that leaves its step
                                  // loop once no cell burns (ember_warp.cu)
  int n_peers;
  uint8_t* peer_out[2];
  int peer_lo[2], peer_hi[2], peer_dst[2];
  // row shards on work lists (ebl_shards_step): the activity records travel with the halo rows.  A
  // tile with a burning cell that stores rows into neighbour p also enqueues, into p's next work
  // list (stamp peer_stamp), p's tiles whose regions reach those rows (peer_queued null: no marks).
  // halo_marked = both neighbours do so for this shard, so its halo tiles need no exposure rule.
  int halo_marked;
  int32_t* peer_queued[2];
  int32_t* peer_next_list[2];
  int32_t* peer_next_count[2];
  int32_t peer_stamp[2];
  int peer_tiles_x[2], peer_tiles_y[2], peer_tile_h[2], peer_tile_w[2], peer_halo_r[2], peer_halo_c[2];
};

// Tiling of the blocked kernel (ember_blocked.cu): tiles of tile_h x tile_w cells with
// halo_rows / halo_cols of light-cone halo; n_steps per launch (<= halo_rows when halos
// exist); row_off = global row of buffer row 0 (the RNG cell index is global).
struct BlockGeom {
  int tile_h, tile_w, halo_rows, halo_cols;
  int n_steps;
  int row_off;
  int list_cap;      // active-list entries per CTA (all its envs)
  int fixed_region;  // every tile's region is (tile + 2 halo) in both dims, clamped inside the layer
                     // (edge tiles take more halo inward): compile-time words per row for tiles
  int envs_per_cta;  // 1 (the blocked kernel's env pooling was measured slower and removed)
};

// Row shards sharing one device (ebl_shards_step): one work-list launch for all of them -- the
// persistent CTAs take tiles from the shards' lists in order (k_step_warp_shards), so a chunk costs
// one launch instead of one per shard.  Passed as a __grid_constant__ kernel parameter.
constexpr int kMaxShardLaunch = 8;
struct ShardsLaunch {
  StepArgs sa[kMaxShardLaunch];
  BlockGeom g[kMaxShardLaunch];
  int n;
  int all_tiles;  // first launch of a call (list_mode 1): every tile of every shard, no lists read
};

// Deterministic mode + adjoint (ember_det.cu).  fp64 planes [env][cell] (the
// reference's trajectory is ulp-sensitive, so parity needs its exact fp64 arithmetic).
struct DetArgs {
  StepArgs s;                     // statics (terrain form), dims
  const double* un;               // current state
  const double* burn;
  const double* bd;
  double* un_o;                   // next state
  double* burn_o;
  double* bd_o;
  const double* pot;              // [table][cell][8] SpreadTables<double>::pot (host-built, exact)
  const double* gam;              // [table][cell]
  const double* potT;             // [table][cell][8] target-ordered pot: potT[v][k] = pot[v - d_k][k]
                                  // (0 toward out-of-bounds sources), or null
  size_t tab_stride;              // cells per table (0: one table for all envs)
  double pc;
  double* traj_un;                // [T][env][cell] state before step t (record mode)
  double* traj_burn;
  double* traj_lam;               // [T][env][cell] lambda of step t (saves back1 the pot gather)
  double inv_p_base;              // 1 / p_base: dpot/dp_base = pot / p_base (terrain form)
  const double* mask;             // [env][cell] target burn mask
  double bce_w, mse_w;
  int pool;
  double* A_un;                   // adjoints of the state after step t
  double* A_burn;
  double* A_bd;
  double* a_lam;                  // adjoint of lambda (unused by the fused k_det_back)
  double* A_un_o;                 // adjoints of the state before step t (k_det_back writes these;
  double* A_burn_o;               // the A_* above are read only: neighbours' tiles read them too)
  double* acc;                    // [env][block][8] gradient partials (fixed order)
  double* loss;                   // [env]
  double* grad;                   // [env][6]
  const double* V;                // [wind] wind speed
  const double* align;            // [wind][8] cos(phi_k - theta) - 1
  int wind_stride;                // 1 (per env) or 0 (shared)
  // general form (per-cell layers): host-built derivative factors per table cell, else null
  const double* fac_F;            // [table][cell] (1+veg)(1+den)
  const double* fac_pb;           // [table][cell][8] dpot/dp_base = F kw ks
  const double* fac_V;            // [table][cell] V
  const double* fac_Va;           // [table][cell][8] V (cos(phi_k - theta) - 1)
  const double* fac_S;            // [table][cell][8] slope S
};

// Per-env RL record (rl_env.hpp:67-75 EnvState minus the layer, plus the tanker
// episode counter).
struct RlEnv {
  int32_t row, col, water, step;
  uint64_t seed, stream;
  int32_t done;
  uint32_t episode;
};

struct RlArgs {
  StepArgs s;                     // statics, streams unused (per-env stream in RlEnv)
  RlEnv* env;                     // [n_envs]
  uint8_t* state;                 // [n_envs][h*w], updated in place
  uint8_t* wet;                   // [n_envs][h*w] (tanker)
  const int32_t* actions;         // [n_envs] or null (device random policy)
  double* reward;                 // [n_envs] (nullable)
  uint8_t* done;                  // [n_envs] (nullable)
  int32_t* error;                 // set to 1 when a finished REFERENCE env is stepped
  // reference variant
  int water_capacity, max_episode_steps, waste_water;
  double burn_penalty;
  // tanker variant
  int ignitions, max_steps;
  uint32_t env_id0;
  uint64_t seed;
  int n_steps;                    // fused rollout length (tanker)
  double* reward_sum;             // [n_envs] (rollout)
  int32_t* episodes;              // [n_envs] (rollout)
  // bit-resident tanker state (warp-local tanker kernel): [n_envs][3 planes B, X, WET][h][wpr] words;
  // bits_in: load from it (else from the byte layers); the kernel always stores it (not the bytes)
  uint32_t* bits;
  int bits_in;
};

}  // namespace ebl
