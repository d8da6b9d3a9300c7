// Launchers exported by ember_kernels.cu / ember_blocked.cu to the C-ABI layer.
#pragma once
#include <cuda_runtime.h>

#include "ember_params.h"

namespace ebl {

constexpr int kTileW = 64;        // general tiled step: CTA tile 16 x 64 cells,
constexpr int kTileH = 16;        // 256 threads x 4 cells
constexpr int kTileThreads = 256;
constexpr int kRlThreads = 256;   // RL kernels: one CTA per env
constexpr int kRlMaxCells = 16384;  // env layer(s) resident in shared memory
constexpr int kResThreads = 128;    // blocked kernel: one CTA per tile (whole env if it fits)
constexpr size_t kResMaxSmem = 200 * 1024;
constexpr int kBlockTileH = 32;     // tiled runs (large grids): 32 x 128 tiles with a 16-row / 32-column
constexpr int kBlockTileW = 128;    // light-cone halo, 16 steps per launch (C3 sweeps: scripts/c3_tiles.sh,
constexpr int kBlockHalo = 16;      // scripts/c3_halo_sweep.sh)

bool phase_prof_built();
// Host-side launch helpers with per-(kernel, device) caches: the dynamic shared-memory opt-in is
// set once per larger size, the occupancy and SM count are queried once (both cost microseconds of
// host time per call, which bounds launch-heavy paths such as row shards).
cudaError_t smem_opt_in(const void* kernel, size_t smem);
cudaError_t resident_ctas(const void* kernel, int threads, size_t smem, int* ctas_per_gpu);
size_t blocked_smem_bytes(int region_h, int region_w, int list_cap, int envs_per_cta);
bool resident_fits(int h, int w);
BlockGeom plan_blocks(int buf_h, int w, int n_steps, bool force_tiles, int row_off, int n_envs,
                      int envs_per_cta);
cudaError_t launch_step_blocked(const StepArgs& a, int mode, const BlockGeom& g, cudaStream_t s);
// warp-local resident kernel (ember_warp.cu): whole env per CTA, one barrier per step
size_t warp_smem_bytes(int h, int w);
bool warp_fits(int h, int w);
cudaError_t launch_step_warp(const StepArgs& a, int mode, const BlockGeom& g, cudaStream_t s);
cudaError_t launch_step_warp_shards(const ShardsLaunch& p, int mode, cudaStream_t s);
cudaError_t launch_tile_init(const uint8_t* in, uint8_t* out, int h, int w, int n_envs, int tile_h, int tile_w,
                             int32_t* trec, int32_t* queued, int32_t stamp, int32_t* next_list, int32_t* next_count,
                             int count_lo, int count_hi, cudaStream_t s);
cudaError_t launch_mark_halo(const uint8_t* layer, int n_envs, size_t ncell, int w, int row0, int n_rows,
                             int32_t* tflags, int tile_h, int tile_w, int ntx, int nty, cudaStream_t s);
cudaError_t launch_tile_counts(const int32_t* trec, int n_envs, int tiles_per_env, int32_t* counts, cudaStream_t s);

cudaError_t launch_det_forward(const DetArgs& d, int t, cudaStream_t s);
cudaError_t launch_det_bd_run(const double* bd0, double* bd_out, const double* traj_burn, size_t n, int n_steps,
                              double pc, cudaStream_t s);
cudaError_t launch_pot_target(const double* pot, double* potT, int n_tables, int h, int w, cudaStream_t s);
cudaError_t launch_det_tables_terrain(const double* S, const uint8_t* fuel, const double* pal64, const double* kw64,
                                      double alpha_s, int n_tables, size_t ncell, size_t grid_stride, int wind_stride,
                                      double* pot, cudaStream_t s);
cudaError_t launch_det_loss(const DetArgs& d, cudaStream_t s);
cudaError_t launch_det_from_fire(const uint8_t* st, double* un, double* bu, double* bd, size_t n,
                                 cudaStream_t s);
cudaError_t launch_det_backward(const DetArgs& d, int t, cudaStream_t s);
cudaError_t launch_det_reduce(const DetArgs& d, cudaStream_t s);
int det_blocks_per_env(int h, int w);  // gradient partials per env of the fused backward
cudaError_t launch_rng_probe(int n, const uint64_t* keys5, uint64_t* out, cudaStream_t s);
cudaError_t launch_step_tile(const StepArgs& a, int mode, cudaStream_t s);
cudaError_t launch_intensity(const StepArgs& a, int mode, float* lam, float* p, cudaStream_t s);
cudaError_t launch_counts(const uint8_t* st, int n_envs, int ncell, int32_t* counts, cudaStream_t s);
cudaError_t launch_rl_ref_step(const RlArgs& g, int mode, cudaStream_t s);
cudaError_t launch_rl_observe(const uint8_t* state, const RlEnv* envs, int n_envs, int h, int w,
                              int radius, int capacity, double* obs, cudaStream_t s);
cudaError_t launch_rl_tanker(const RlArgs& g, int mode, cudaStream_t s);
constexpr int kRlBitsThreads = 128;  // bit-plane tanker kernel: one CTA per env
size_t rl_bits_smem_bytes(int h, int w);
bool rl_bits_fits(int h, int w);
cudaError_t launch_rl_tanker_bits(const RlArgs& g, int mode, cudaStream_t s);
size_t rl_warp_smem_bytes(int h, int w);
cudaError_t launch_rl_tanker_warp(const RlArgs& g, int mode, cudaStream_t s);
cudaError_t launch_rl_observe_planes(const uint32_t* bits, const uint8_t* state, const uint8_t* wet, uint8_t* out,
                                     int n_envs, int h, int w, cudaStream_t s);
cudaError_t launch_rl_bits_to_bytes(const uint32_t* bits, uint8_t* state, uint8_t* wet, int n_envs, int h, int w,
                                    cudaStream_t s);
cudaError_t launch_rl_tanker_reset(const RlArgs& g, int mode, const uint8_t* mask, cudaStream_t s);

// ---- environment construction (ember_synth.cu) ----
struct SynthArgs {
  uint64_t seed;
  uint32_t env_id0;
  int n_envs, h, w;       // n_envs <= 65535 (grid.y)
  int lc_base, el_base;   // lattice periods (ember_host.cpp synth_one)
  double elev_max;
  uint8_t* fuel;          // [n_envs][h*w] palette index 0..10
  float* elev;            // [n_envs][h*w]
  double* scratch;        // [n_envs][h*w]
  unsigned long long* mm; // [n_envs][4] landcover lo, hi, elevation lo, hi (IEEE bits)
  unsigned int* hist;     // [n_envs][4096]
  int* thr;               // [n_envs][10]
};
cudaError_t launch_synth_terrain(const SynthArgs& a, cudaStream_t s);

struct IgniteArgs {
  uint64_t seed;
  uint32_t env_id0;
  int n_envs, h, w, count;
  const uint8_t* fuel;
  size_t fuel_stride;      // 0 (shared terrain) or h*w
  const double* burnable;  // [256] 1.0 / 0.0 per palette entry
  uint8_t* states;         // [n_envs][h*w], zeroed by the launcher
  int* placed;             // [n_envs]
};
cudaError_t launch_synth_ignitions(const IgniteArgs& a, cudaStream_t s);

struct LandcoverArgs {
  size_t n;
  const int32_t* landcover;  // [n] codes
  const float* elev;         // [n] or null; NaN = DEM nodata
  const int32_t* codes;      // sorted FuelTable codes, n_codes <= 254
  int n_codes, fallback_index, nodata_index, has_nodata;
  int32_t nodata_code;
  uint8_t* fuel;             // [n] palette index
  unsigned long long* missing;  // first cell with an unmapped code (init ~0)
};
cudaError_t launch_landcover_map(const LandcoverArgs& a, cudaStream_t s);
// fp32 slope table [grid][cell][8] (terrain form, built with the layers; ember_synth.cu)
cudaError_t launch_snapshot_text(const uint8_t* layers, int n, int h, int w, const char* meta,
                                 const unsigned long long* off, char* out, cudaStream_t s);
cudaError_t launch_pot32t(const float* slope32, const uint2* nfuel, const uint8_t* fuel, const float* pal32,
                          const float* kw32, int n_envs, size_t ncell, size_t ter_stride, int kw_stride, float alpha_l2,
                          float* out, cudaStream_t s);
cudaError_t launch_slope_table(const float* elev, const uint8_t* fuel, size_t n_grids, int h, int w, float inv_d0,
                               float inv_d1, float* out, uint2* nfuel, cudaStream_t s);

}  // namespace ebl
