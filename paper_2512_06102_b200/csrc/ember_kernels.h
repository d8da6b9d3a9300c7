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
constexpr int kBlockTileH = 64;     // tiled blocked kernel (large grids): 64 x 256 tiles,
constexpr int kBlockTileW = 256;    // 8-row / 32-column light-cone halo, 8 steps per launch
constexpr int kBlockHalo = 8;

size_t blocked_smem_bytes(int region_h, int region_w, int list_cap);
bool resident_fits(int h, int w);
BlockGeom plan_blocks(int buf_h, int w, int n_steps, bool force_tiles, int row_off);
cudaError_t launch_step_blocked(const StepArgs& a, int mode, const BlockGeom& g, cudaStream_t s);

cudaError_t launch_det_forward(const DetArgs& d, int t, cudaStream_t s);
cudaError_t launch_det_loss(const DetArgs& d, cudaStream_t s);
cudaError_t launch_det_backward(const DetArgs& d, int t, cudaStream_t s);
cudaError_t launch_det_reduce(const DetArgs& d, cudaStream_t s);
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
cudaError_t launch_rl_tanker_reset(const RlArgs& g, int mode, const uint8_t* mask, cudaStream_t s);

}  // namespace ebl
