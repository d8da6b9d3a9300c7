// Launchers exported by ember_kernels.cu / ember_resident.cu to the C-ABI layer.
#pragma once
#include <cuda_runtime.h>

#include "ember_params.h"

namespace ebl {

constexpr int kTileW = 64;        // general tiled step: CTA tile 16 x 64 cells,
constexpr int kTileH = 16;        // 256 threads x 4 cells
constexpr int kTileThreads = 256;
constexpr int kRlThreads = 256;   // RL kernels: one CTA per env
constexpr int kRlMaxCells = 16384;  // env layer(s) resident in shared memory
constexpr int kResThreads = 256;    // fused env-resident kernel: one CTA per env
constexpr size_t kResMaxSmem = 200 * 1024;

size_t resident_smem_bytes(int h, int w);
bool resident_fits(int h, int w);
cudaError_t launch_step_resident(const StepArgs& a, int mode, int n_steps, cudaStream_t s);

cudaError_t launch_rng_probe(int n, const uint64_t* keys5, uint64_t* out, cudaStream_t s);
cudaError_t launch_step_tile(const StepArgs& a, int mode, cudaStream_t s);
cudaError_t launch_intensity(const StepArgs& a, int mode, float* lam, float* p, cudaStream_t s);
cudaError_t launch_counts(const uint8_t* st, int n_envs, int ncell, int32_t* counts, cudaStream_t s);
cudaError_t launch_rl_ref_step(const RlArgs& g, int mode, cudaStream_t s);
cudaError_t launch_rl_observe(const uint8_t* state, const RlEnv* envs, int n_envs, int h, int w,
                              int radius, int capacity, double* obs, cudaStream_t s);
cudaError_t launch_rl_tanker(const RlArgs& g, int mode, cudaStream_t s);
cudaError_t launch_rl_tanker_reset(const RlArgs& g, int mode, const uint8_t* mask, cudaStream_t s);

}  // namespace ebl
