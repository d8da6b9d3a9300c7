// C-ABI implementation (include/ember_b200.h): the device-resident batch object,
// static-layer management, launch sequencing and error convention.
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <cmath>
#include <cstdlib>
#include <cstdint>
#include <algorithm>
#include <cstring>
#include <limits>
#include <memory>
#include <charconv>
#include <mutex>
#include <sstream>
#include <unordered_map>
#include <string>
#include <vector>

#include "../../include/ember_b200.h"
#include "ember_host.h"
#include "ember_kernels.h"
#include "ember_params.h"

using ebl::Cfg6;

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define EBL_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return set_err(EBL_ECUDA, std::string(#call ": ") + cudaGetErrorString(e_));       \
  } while (0)

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  ~DevBuf() { reset(); }
  void reset() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  cudaError_t alloc(size_t count) {
    if (count == n && p) return cudaSuccess;
    reset();
    n = count;
    return cudaMalloc(&p, count * sizeof(T) + 16);
  }
};


}  // namespace

struct ebl_batch {
  int device = 0;
  int n_envs = 0, h = 0, w = 0;
  size_t ncell = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ebl_sim_config cfg{};

  DevBuf<uint8_t> state[2];
  int cur = 0;
  int kernel = EBL_KERNEL_AUTO;
  int tile_h = 0, tile_w = 0, tile_halo = 0;  // explicit blocked tiling (tests); 0 = planned
  bool counts_valid = false;
  DevBuf<int32_t> counts;
  DevBuf<unsigned long long> diag;
  DevBuf<long long> prof;           // phase profile of the blocked kernel (ebl_batch_set_profiling)
  int band_lo = -1, band_hi = -1;   // layer rows owned by this row shard (ebl_batch_set_band)
  cudaEvent_t shard_ev[2] = {nullptr, nullptr};  // completion of this shard's launch of chunk c, slot c & 1
  bool profiling = false;
  uint64_t launches = 0, steps_done = 0;

  uint64_t seed = 0, step = 0;
  int64_t row_off = 0;  // global row of layer row 0 (row-sharded landscapes)
  int sched_len = 0;    // wind schedule entries (0: constant wind)
  uint8_t* traj_out = nullptr;  // device trajectory of the ebl_step_batch in flight (record)
  std::vector<double> g_sched_speed, g_sched_dir;  // general form: [S][grid][cell]
  bool streams_uploaded = false;
  std::vector<uint64_t> h_streams;
  DevBuf<uint64_t> streams;

  int mode = ebl::kStaticNone;
  int n_grids = 0;
  // general form
  std::vector<double> g_speed, g_dir, g_veg, g_den, g_slope;
  bool tables_dirty = false;
  DevBuf<double> pot, gamma;
  // terrain form
  DevBuf<uint8_t> fuel;
  DevBuf<float> elev;
  DevBuf<float> slope32;            // [grid][cell][8] fp32 slopes of the layers (built by prepare)
  DevBuf<uint2> nfuel;              // [grid][cell] fuel classes of the 8 sources (built with slope32)
  DevBuf<float> pot32t;             // [env or 1][cell][8] fp32 lambda terms (built by prepare)
  DevBuf<int32_t> tflags[2];           // per-tile activity records of halo-tiled runs (ping-pong)
  // records of the last launch kept across ebl_step_batch calls: tiles count (-1: none), which
  // buffer holds them, and the tile geometry they describe.  Any entry point other than stepping,
  // reads, and halo-row writes outside the band drops them (check_batch / check_sync).
  mutable int tf_carry_tiles = -1;
  int tf_carry_par = 0, tf_carry_th = 0, tf_carry_tw = 0;
  // work-list runs (C3-like single landscapes): in-place tile records, dedup stamps, two lists and
  // their counters [count0, count1, cursor]
  DevBuf<int32_t> trec, tqueued, tlist[2], tcount;
  int32_t list_stamp = 0;
  DevBuf<char> snap_text, snap_meta;  // snapshot rendering staging (grow-only)
  DevBuf<unsigned long long> snap_off;
  bool pot32t_valid = false;
  bool slope_dirty = false;
  std::vector<double> pal_veg, pal_den;
  double cellsize = 30.0;
  int n_winds = 0;
  std::vector<double> wind_speed, wind_dir;
  bool derived_dirty = false;
  DevBuf<float> pal32, kw32;
  DevBuf<double> pal64, kw64;

  // RL
  int rl_variant = -1;
  ebl_env_config env_cfg{};
  int tanker_ignitions = 5, tanker_max_steps = 256;
  uint32_t env_id0 = 0;
  uint64_t rl_seed = 0;
  DevBuf<ebl::RlEnv> rl_env;
  // bit-resident tanker state (warp-local tanker kernel): rl_bits_valid = the bits equal the
  // current layers; rl_bits_truth = the bits are newer than the byte layers (rebuilt on demand)
  DevBuf<uint32_t> rl_bits;
  bool rl_bits_valid = false, rl_bits_truth = false;
  DevBuf<uint8_t> wet, done, mask;
  DevBuf<double> reward, reward_sum;
  DevBuf<int32_t> actions, error, episodes;
  DevBuf<double> obs;

  // deterministic mode (C4), fp64
  DevBuf<double> det[6];            // un, burn, bd x2 (double buffer)
  int det_cur = 0;
  bool det_ready = false;
  DevBuf<double> det_pot, det_gam, det_fac, det_V, det_align, traj, adj, det_mask, acc, det_loss, det_grad, det_init;
  DevBuf<double> det_potT;          // target-ordered copy of det_pot for the forward (EBL_DET_POTT)
  DevBuf<double> det_S;             // [grid][cell][8] cached fp64 slopes (host atan, once per terrain)
  bool det_S_valid = false;
  bool det_dev_tables = true;       // terrain-form SpreadTables built on the device (ebl_batch_set_det_tables)
  int det_tables = 0;
  bool det_tables_valid = false;
  ebl_sim_config det_cfg{};
  bool det_mask_set = false;        // det_mask holds the ebl_det_set_mask target
  int traj_steps = -1;              // steps recorded by the last ebl_det_forward(record=1)
  std::vector<uint8_t> h_fuel;      // host copies of the terrain (exact host-built tables)
  std::vector<float> h_elev;
  bool h_terrain_stale = false;     // device terrain newer than h_fuel/h_elev (device-built)

  // host-buffer pipeline (ebl_batch_run): copy-in stream, per-chunk compute streams, copy-out
  int pipe_chunks = 0;              // 0 = auto
  cudaStream_t pipe_in = nullptr, pipe_out = nullptr;
  std::vector<cudaStream_t> pipe_comp;
  std::vector<cudaEvent_t> pipe_ev_in, pipe_ev_done;
  cudaEvent_t pipe_ev_start = nullptr, pipe_ev_end = nullptr;

  ~ebl_batch() {
    for (cudaStream_t s : pipe_comp) cudaStreamDestroy(s);
    for (cudaEvent_t e : pipe_ev_in) cudaEventDestroy(e);
    for (cudaEvent_t e : pipe_ev_done) cudaEventDestroy(e);
    if (pipe_in) cudaStreamDestroy(pipe_in);
    if (pipe_out) cudaStreamDestroy(pipe_out);
    if (pipe_ev_start) cudaEventDestroy(pipe_ev_start);
    if (pipe_ev_end) cudaEventDestroy(pipe_ev_end);
    for (cudaEvent_t e : shard_ev)
      if (e) cudaEventDestroy(e);
  }
};

namespace {

Cfg6 cfg6(const ebl_sim_config& c) {
  return Cfg6{c.p_base, c.alpha_w1, c.alpha_w2, c.alpha_s, c.alpha_gamma, c.p_continue};
}

// Every entry point that works on a batch makes the batch's device current for the call and
// restores the caller's device on return (a process may drive batches on several GPUs, and the
// caller's own CUDA context -- e.g. torch's current device -- must not move under it).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (dev < 0 || cudaGetDevice(&prev) != cudaSuccess) {
      prev = -1;
      cudaGetLastError();
      return;
    }
    if (prev == dev) prev = -1;
    else if (cudaSetDevice(dev) != cudaSuccess) cudaGetLastError();
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};
#define EBL_DEVICE_GUARD(b) DeviceGuard ebl_device_guard_((b) ? (b)->device : -1)

int check_batch(const ebl_batch* b, bool keep_records = false) {
  if (!b) return set_err(EBL_EINVAL, "null batch");
  if (!keep_records) b->tf_carry_tiles = -1;
  return EBL_OK;
}

// Byte layers up to date before any access other than the warp-local tanker kernel: rebuild them
// from the bit-resident tanker state when that is newer, and treat the bits as stale afterwards
// (the caller may write the bytes).
int rl_sync_bytes(ebl_batch* b) {
  if (b->rl_bits_truth) {
    EBL_CUDA(cudaSetDevice(b->device));
    EBL_CUDA(ebl::launch_rl_bits_to_bytes(b->rl_bits.p, b->state[b->cur].p, b->wet.p, b->n_envs, b->h, b->w,
                                          b->stream));
    b->rl_bits_truth = false;
  }
  b->rl_bits_valid = false;
  return EBL_OK;
}

// check_batch + rl_sync_bytes: the entry of every public call that touches the layers
int check_sync(ebl_batch* b, bool keep_records = false) {
  if (int e = check_batch(b, keep_records)) return e;
  return rl_sync_bytes(b);
}

// Brings the derived device-side statics in line with (config, layers).
int prepare(ebl_batch* b) {
  if (b->mode == ebl::kStaticNone) return set_err(EBL_ESTATE, "no grid or terrain set on the batch");
  EBL_CUDA(cudaSetDevice(b->device));
  const Cfg6 c = cfg6(b->cfg);
  const bool pot32t_stale = b->mode == ebl::kStaticTerrain && (b->derived_dirty || b->slope_dirty);
  if (b->mode == ebl::kStaticTables && b->tables_dirty) {
    const size_t n = b->ncell * b->n_grids;
    const int S = std::max(1, b->sched_len);  // one table per wind-schedule entry
    std::vector<double> pot(n * 8 * S), gam(n);
    for (int s = 0; s < S; ++s) {
      const double* sp = b->sched_len ? b->g_sched_speed.data() + s * n : b->g_speed.data();
      const double* dr = b->sched_len ? b->g_sched_dir.data() + s * n : b->g_dir.data();
      ebl::build_tables(n, sp, dr, b->g_veg.data(), b->g_den.data(), b->g_slope.data(), c,
                        pot.data() + s * n * 8, gam.data());
    }
    EBL_CUDA(b->pot.alloc(n * 8 * S));
    EBL_CUDA(b->gamma.alloc(n));
    EBL_CUDA(cudaMemcpyAsync(b->pot.p, pot.data(), pot.size() * sizeof(double), cudaMemcpyHostToDevice, b->stream));
    EBL_CUDA(cudaMemcpyAsync(b->gamma.p, gam.data(), n * sizeof(double), cudaMemcpyHostToDevice, b->stream));
    EBL_CUDA(cudaStreamSynchronize(b->stream));
    b->tables_dirty = false;
  }
  if (b->mode == ebl::kStaticTerrain && b->derived_dirty) {
    if (b->n_winds == 0) return set_err(EBL_ESTATE, "terrain form needs ebl_batch_set_wind");
    std::vector<float> p32(768, 0.f);
    std::vector<double> p64(1024, 0.0);
    for (size_t k = 0; k < b->pal_veg.size(); ++k) {
      const double v = ebl::clamp_fuel(b->pal_veg[k]), d = ebl::clamp_fuel(b->pal_den[k]);
      p64[k] = (c.p_base * (1.0 + v)) * (1.0 + d);            // kernel.hpp:39-40
      p64[256 + k] = (c.alpha_gamma * (1.0 + v)) * (1.0 + d);  // kernel.hpp:75-76
      p64[512 + k] = (1.0 + v) * (1.0 + d) > 0.0 ? 1.0 : 0.0;
      p64[768 + k] = (1.0 + v) * (1.0 + d);  // F, for the deterministic adjoint
      p32[k] = static_cast<float>(p64[k]);
      p32[256 + k] = static_cast<float>(p64[256 + k]);
      p32[512 + k] = static_cast<float>((1.0 + v) * (1.0 + d));  // F = (1+veg)(1+den), deterministic adjoint
    }
    // kappa_wind of every wind [schedule entry][wind set] (wind_speed holds S * n_winds entries)
    const size_t nw = b->wind_speed.size();
    std::vector<double> k64(nw * 8);
    std::vector<float> k32(k64.size());
    for (size_t e = 0; e < nw; ++e) ebl::kappa_wind8(b->wind_speed[e], b->wind_dir[e], c, &k64[e * 8]);
    for (size_t i = 0; i < k64.size(); ++i) k32[i] = static_cast<float>(k64[i]);
    EBL_CUDA(b->pal32.alloc(768));
    EBL_CUDA(b->pal64.alloc(1024));
    EBL_CUDA(b->kw32.alloc(k32.size()));
    EBL_CUDA(b->kw64.alloc(k64.size()));
    EBL_CUDA(cudaMemcpyAsync(b->pal32.p, p32.data(), 768 * sizeof(float), cudaMemcpyHostToDevice, b->stream));
    EBL_CUDA(cudaMemcpyAsync(b->pal64.p, p64.data(), 1024 * sizeof(double), cudaMemcpyHostToDevice, b->stream));
    EBL_CUDA(cudaMemcpyAsync(b->kw32.p, k32.data(), k32.size() * sizeof(float), cudaMemcpyHostToDevice, b->stream));
    EBL_CUDA(cudaMemcpyAsync(b->kw64.p, k64.data(), k64.size() * sizeof(double), cudaMemcpyHostToDevice, b->stream));
    EBL_CUDA(cudaStreamSynchronize(b->stream));
    b->derived_dirty = false;
  }
  if (b->mode == ebl::kStaticTerrain && b->slope_dirty) {  // slope_from_dem of the layers (GridState)
    const double d0 = b->cellsize * 1.0, d1 = b->cellsize * 1.41421356237309504880;
    EBL_CUDA(b->slope32.alloc(b->ncell * b->n_grids * 8));
    EBL_CUDA(b->nfuel.alloc(b->ncell * b->n_grids));
    EBL_CUDA(ebl::launch_slope_table(b->elev.p, b->fuel.p, b->n_grids, b->h, b->w, static_cast<float>(1.0 / d0),
                                     static_cast<float>(1.0 / d1), b->slope32.p, b->nfuel.p, b->stream));
    b->slope_dirty = false;
  }
  if (pot32t_stale) {  // the per-candidate lambda terms (one wind per env; none under a schedule)
    b->pot32t_valid = false;
    if (b->sched_len <= 1) {
      const bool per_env = b->n_grids > 1 || b->n_winds > 1;
      const int n_tab = per_env ? b->n_envs : 1;
      EBL_CUDA(b->pot32t.alloc(b->ncell * n_tab * 8));
      EBL_CUDA(ebl::launch_pot32t(b->slope32.p, b->nfuel.p, b->fuel.p, b->pal32.p, b->kw32.p, n_tab, b->ncell,
                                  b->n_grids > 1 ? b->ncell : 0, b->n_winds > 1 ? 8 : 0,
                                  static_cast<float>(b->cfg.alpha_s * 1.4426950408889634), b->pot32t.p, b->stream));
      b->pot32t_valid = true;
    }
  }
  return EBL_OK;
}

ebl::StepArgs step_args(const ebl_batch* b) {
  ebl::StepArgs a{};
  a.h = b->h;
  a.w = b->w;
  a.n_envs = b->n_envs;
  a.seed = b->seed;
  a.step = b->step;
  a.row_off = b->row_off;
  a.streams = b->streams.p;
  a.pc_thr = ebl::continue_threshold(b->cfg.p_continue);
  a.in = b->state[b->cur].p;
  a.out = b->state[b->cur ^ 1].p;
  a.diag = b->diag.p;
  a.pot = b->pot.p;
  a.gamma = b->gamma.p;
  a.tab_stride = b->n_grids > 1 ? b->ncell : 0;
  a.fuel = b->fuel.p;
  a.elev = b->elev.p;
  a.slope32 = b->mode == ebl::kStaticTerrain ? b->slope32.p : nullptr;
  a.nfuel = b->mode == ebl::kStaticTerrain ? b->nfuel.p : nullptr;
  a.pot32t = b->mode == ebl::kStaticTerrain && b->pot32t_valid && b->sched_len <= 1 ? b->pot32t.p : nullptr;
  a.pot32t_stride = b->n_grids > 1 || b->n_winds > 1 ? b->ncell * 8 : 0;
  a.n_pal = static_cast<int>(b->pal_veg.size());
  a.alpha_s_l2 = static_cast<float>(b->cfg.alpha_s * 1.4426950408889634);
  a.ter_stride = b->n_grids > 1 ? b->ncell : 0;
  a.pal32 = b->pal32.p;
  a.pal64 = b->pal64.p;
  a.kw32 = b->kw32.p;
  a.kw64 = b->kw64.p;
  a.kw_stride = b->n_winds > 1 ? 8 : 0;
  a.sched_len = b->sched_len;
  a.kw_sched_stride = static_cast<size_t>(b->n_winds) * 8;
  a.pot_sched_stride = b->ncell * b->n_grids * 8;
  a.alpha_s = b->cfg.alpha_s;
  a.alpha_s32 = static_cast<float>(b->cfg.alpha_s);
  const double d0 = b->cellsize * 1.0, d1 = b->cellsize * 1.41421356237309504880;  // geodata.cpp:222-223
  a.dist64[0] = d0;
  a.dist64[1] = d1;
  a.inv_dist32[0] = static_cast<float>(1.0 / d0);
  a.inv_dist32[1] = static_cast<float>(1.0 / d1);
  // the fp32 guard band (1e-4 relative) holds while |alpha_s * slope| stays O(10)
  a.force64 = !(std::fabs(b->cfg.alpha_s) <= 50.0);
  a.prof = b->profiling ? b->prof.p : nullptr;
  a.store_lo = 0;
  a.store_hi = b->h;
  a.keep_lo = b->band_lo >= 0 ? b->band_lo : 0;
  a.keep_hi = b->band_lo >= 0 ? b->band_hi : b->h;
  a.n_peers = 0;
  return a;
}

// StepArgs of the env sub-range [off, off + n) of a batch (per-env pointers advanced).
ebl::StepArgs chunk_args(const ebl_batch* b, ebl::StepArgs a, int off, int n) {
  const size_t o = static_cast<size_t>(off);
  a.n_envs = n;
  a.in += o * b->ncell;
  a.out += o * b->ncell;
  a.streams += o;
  if (a.counts) a.counts += o * 4;
  if (a.prof) a.prof += o * 10;
  if (a.out2) a.out2 += o * b->ncell;
  if (a.tab_stride) {
    a.pot += o * a.tab_stride * 8;
    a.gamma += o * a.tab_stride;
  }
  if (a.ter_stride) {
    a.fuel += o * a.ter_stride;
    a.elev += o * a.ter_stride;
    if (a.slope32) a.slope32 += o * a.ter_stride * 8;
    if (a.nfuel) a.nfuel += o * a.ter_stride;
  }
  if (a.kw_stride) {
    a.kw32 += o * a.kw_stride;
    a.kw64 += o * a.kw_stride;
  }
  if (a.pot32t) a.pot32t += o * a.pot32t_stride;
  return a;
}

// The warp-local kernel runs every one-env-per-CTA geometry (whole env or halo tiles) under AUTO
// (C1: 0.63 ms vs 0.77 ms for the pooled-list blocked kernel, which EBL_KERNEL_RESIDENT /
// EBL_KERNEL_BLOCKED keep selectable).
bool use_warp(const ebl_batch* b) { return b->kernel == EBL_KERNEL_WARP || b->kernel == EBL_KERNEL_AUTO; }

// Halo-tiled warp-kernel runs (default 32 x 128 tiles) on terrain layers at least one region large:
// every tile's region is the full (tile + halo) -- 48 x 192 by default, clamped inside the layer:
// edge tiles take their halo inward -- so all tiles take compile-time words per row and the
// branch-free decide pass.
// EBL_FIXED_REGION=0: edge regions cut at the layer edge (the generic path).
void apply_fixed_regions(const ebl_batch* b, ebl::BlockGeom& g) {
  static const bool on = [] {
    const char* e = std::getenv("EBL_FIXED_REGION");
    return !e || std::atoi(e) != 0;
  }();
  if (!on || !use_warp(b) || b->mode != ebl::kStaticTerrain) return;
  const int rw = g.tile_w + 2 * g.halo_cols;  // the compile-time region widths (ember_warp.cu)
  if (g.halo_rows < 1 || g.halo_rows > 32 || g.halo_cols != 32 || !(rw == 128 || rw == 192 || rw == 320)) return;
  if (b->h < g.tile_h + 2 * g.halo_rows || b->w < g.tile_w + 2 * g.halo_cols || (b->w % 32) != 0) return;
  g.fixed_region = 1;
}

// EBL_TILE_INIT=0: work-list runs start with a grid launch over every tile instead of k_tile_init
bool tile_init_on() {
  static const bool on = [] {
    const char* e = std::getenv("EBL_TILE_INIT");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

// EBL_HALO_MARKS=0: row shards' halo tiles are exposed (never skipped) instead of marked
bool halo_marks_on() {
  static const bool on = [] {
    const char* e = std::getenv("EBL_HALO_MARKS");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

// Halo rows [row0, row0 + n) of a row shard were just written from outside (a neighbour's band):
// their burning cells mark the carried tile records, so the skip rule sees them (ember_warp.cu).
cudaError_t mark_halo_rows(ebl_batch* b, int row0, int n) {
  if (b->tf_carry_tiles <= 0 || b->tf_carry_th <= 0 || b->tf_carry_tw <= 0) return cudaSuccess;
  const int ntx = (b->w + b->tf_carry_tw - 1) / b->tf_carry_tw, nty = (b->h + b->tf_carry_th - 1) / b->tf_carry_th;
  if (ntx * nty != b->tf_carry_tiles) return cudaSuccess;
  return ebl::launch_mark_halo(b->state[b->cur].p, b->n_envs, b->ncell, b->w, row0, n, b->tflags[b->tf_carry_par].p,
                               b->tf_carry_th, b->tf_carry_tw, ntx, nty, b->stream);
}

cudaError_t launch_ca(const ebl_batch* b, const ebl::StepArgs& a, const ebl::BlockGeom& g, cudaStream_t s) {
  if (use_warp(b)) return ebl::launch_step_warp(a, b->mode, g, s);
  return ebl::launch_step_blocked(a, b->mode, g, s);
}

int ensure_pipeline(ebl_batch* b, int chunks) {
  if (!b->pipe_in) {
    EBL_CUDA(cudaStreamCreateWithFlags(&b->pipe_in, cudaStreamNonBlocking));
    EBL_CUDA(cudaStreamCreateWithFlags(&b->pipe_out, cudaStreamNonBlocking));
    EBL_CUDA(cudaEventCreateWithFlags(&b->pipe_ev_start, cudaEventDisableTiming));
    EBL_CUDA(cudaEventCreateWithFlags(&b->pipe_ev_end, cudaEventDisableTiming));
  }
  while (static_cast<int>(b->pipe_comp.size()) < chunks) {
    cudaStream_t s;
    cudaEvent_t e0, e1;
    EBL_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    EBL_CUDA(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
    EBL_CUDA(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
    b->pipe_comp.push_back(s);
    b->pipe_ev_in.push_back(e0);
    b->pipe_ev_done.push_back(e1);
  }
  return EBL_OK;
}

}  // namespace

extern "C" {

int ebl_abi_version(void) { return EBL_ABI_VERSION; }
const char* ebl_last_error(void) { return g_err.c_str(); }

void ebl_default_config(ebl_sim_config* c) {
  *c = ebl_sim_config{0.12, 0.2, 0.4, 1.0, 1.0, 0.6, 200};  // grid.hpp:173-179
}

int ebl_validate_config(const ebl_sim_config* c) {  // grid.cpp:107-124
  auto finite = [](double v) { return std::isfinite(v); };
  if (!finite(c->p_base) || c->p_base <= 0.0) return set_err(EBL_EINVAL, "SimConfig: p_base must be > 0");
  if (!finite(c->alpha_gamma) || c->alpha_gamma <= 0.0)
    return set_err(EBL_EINVAL, "SimConfig: alpha_gamma must be > 0");
  if (!finite(c->p_continue) || c->p_continue < 0.0 || c->p_continue > 1.0)
    return set_err(EBL_EINVAL, "SimConfig: p_continue must be in [0, 1]");
  if (!finite(c->alpha_w1) || !finite(c->alpha_w2) || !finite(c->alpha_s))
    return set_err(EBL_EINVAL, "SimConfig: wind/slope parameters must be finite");
  if (c->max_steps < 1) return set_err(EBL_EINVAL, "SimConfig: max_steps must be positive");
  return EBL_OK;
}

int ebl_batch_create(ebl_batch** out, int device, int n_envs, int height, int width, void* stream) {
  if (!out) return set_err(EBL_EINVAL, "null out");
  *out = nullptr;
  if (height < 1 || width < 1) return set_err(EBL_EINVAL, "Grid: dimensions must be at least 1x1");
  if (n_envs < 1) return set_err(EBL_EINVAL, "make_stochastic_batch: count must be >= 1");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return set_err(EBL_ECUDA, "no CUDA device available (the engine has no CPU path)");
  if (device < 0 || device >= ndev) return set_err(EBL_EINVAL, "device ordinal out of range");
  DeviceGuard guard(device);
  auto b = std::make_unique<ebl_batch>();
  b->device = device;
  b->n_envs = n_envs;
  b->h = height;
  b->w = width;
  b->ncell = static_cast<size_t>(height) * width;
  if (stream) {
    b->stream = static_cast<cudaStream_t>(stream);
  } else {
    EBL_CUDA(cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking));
    b->own_stream = true;
  }
  ebl_default_config(&b->cfg);
  const size_t total = b->ncell * n_envs;
  EBL_CUDA(b->state[0].alloc(total));
  EBL_CUDA(b->state[1].alloc(total));
  EBL_CUDA(cudaMemsetAsync(b->state[0].p, 0, total, b->stream));
  EBL_CUDA(b->counts.alloc(static_cast<size_t>(n_envs) * 4));
  EBL_CUDA(b->diag.alloc(4));  // fp64 fallbacks, ambiguous draws, tiles processed, tiles launched
  EBL_CUDA(cudaMemsetAsync(b->diag.p, 0, 4 * sizeof(unsigned long long), b->stream));
  EBL_CUDA(b->streams.alloc(n_envs));
  b->h_streams.resize(n_envs);
  for (int e = 0; e < n_envs; ++e) b->h_streams[e] = static_cast<uint64_t>(e);
  EBL_CUDA(cudaMemcpyAsync(b->streams.p, b->h_streams.data(), n_envs * sizeof(uint64_t),
                           cudaMemcpyHostToDevice, b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  b->streams_uploaded = true;
  *out = b.release();
  return EBL_OK;
}

void ebl_batch_destroy(ebl_batch* b) {
  if (!b) return;
  EBL_DEVICE_GUARD(b);
  cudaStreamSynchronize(b->stream);
  if (b->own_stream) cudaStreamDestroy(b->stream);
  delete b;
}

int ebl_batch_set_config(ebl_batch* b, const ebl_sim_config* c) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (!c) return set_err(EBL_EINVAL, "null config");
  // pot/gamma/kappa depend on every field but p_continue and max_steps
  const bool statics = c->p_base != b->cfg.p_base || c->alpha_w1 != b->cfg.alpha_w1 ||
                       c->alpha_w2 != b->cfg.alpha_w2 || c->alpha_s != b->cfg.alpha_s ||
                       c->alpha_gamma != b->cfg.alpha_gamma ||
                       std::memcmp(&c->p_base, &b->cfg.p_base, 5 * sizeof(double)) != 0;
  b->cfg = *c;
  if (statics) {
    b->tables_dirty = b->tables_dirty || b->mode == ebl::kStaticTables;
    b->derived_dirty = b->derived_dirty || b->mode == ebl::kStaticTerrain;
  }
  return EBL_OK;
}

int ebl_batch_set_grid(ebl_batch* b, int n_grids, const double* speed, const double* dir,
                       const double* veg, const double* den, const double* slope8) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (n_grids != 1 && n_grids != b->n_envs) return set_err(EBL_EINVAL, "n_grids must be 1 or n_envs");
  if (!speed || !dir || !veg || !den || !slope8) return set_err(EBL_EINVAL, "null layer");
  const size_t n = b->ncell * n_grids;
  for (size_t i = 0; i < n; ++i) {  // grid.cpp:49-62, 68-77, 86-90
    if (!std::isfinite(speed[i])) return set_err(EBL_EINVAL, "WindField: non-finite speed");
    if (speed[i] < 0.0) return set_err(EBL_EINVAL, "WindField: negative speed");
    if (!std::isfinite(dir[i])) return set_err(EBL_EINVAL, "WindField: non-finite direction");
    if (std::isnan(veg[i])) return set_err(EBL_EINVAL, "FuelField veg: NaN value in layer");
    if (std::isnan(den[i])) return set_err(EBL_EINVAL, "FuelField den: NaN value in layer");
  }
  for (size_t i = 0; i < n * 8; ++i)
    if (std::isnan(slope8[i])) return set_err(EBL_EINVAL, "SlopeField: NaN slope");
  b->g_speed.assign(speed, speed + n);
  b->g_dir.assign(dir, dir + n);
  b->g_veg.assign(veg, veg + n);
  b->g_den.assign(den, den + n);
  b->g_slope.assign(slope8, slope8 + n * 8);
  b->mode = ebl::kStaticTables;
  b->n_grids = n_grids;
  b->sched_len = 0;
  b->g_sched_speed.clear();
  b->g_sched_dir.clear();
  b->tables_dirty = true;
  b->det_tables_valid = false;
  b->fuel.reset();
  b->elev.reset();
  return EBL_OK;
}

int ebl_batch_set_terrain(ebl_batch* b, int n_grids, const uint8_t* fuel_class, const float* elevation,
                          int n_classes, const double* class_veg, const double* class_den,
                          double cellsize) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (n_grids != 1 && n_grids != b->n_envs) return set_err(EBL_EINVAL, "n_grids must be 1 or n_envs");
  if (n_classes < 1 || n_classes > 256) return set_err(EBL_EINVAL, "n_classes must be in [1, 256]");
  if (!(cellsize > 0.0) || !std::isfinite(cellsize))
    return set_err(EBL_EINVAL, "raster_from_model: cellsize must be positive");
  for (int k = 0; k < n_classes; ++k)
    if (std::isnan(class_veg[k]) || std::isnan(class_den[k]))
      return set_err(EBL_EINVAL, "FuelField: NaN value in layer");
  const size_t n = b->ncell * n_grids;
  for (size_t i = 0; i < n; ++i) {
    if (fuel_class[i] >= n_classes) return set_err(EBL_EINVAL, "fuel class outside the palette");
    if (std::isinf(elevation[i])) return set_err(EBL_EINVAL, "elevation must be finite or NaN (nodata)");
  }
  EBL_CUDA(cudaSetDevice(b->device));
  EBL_CUDA(b->fuel.alloc(n));
  EBL_CUDA(b->elev.alloc(n));
  EBL_CUDA(cudaMemcpyAsync(b->fuel.p, fuel_class, n, cudaMemcpyHostToDevice, b->stream));
  EBL_CUDA(cudaMemcpyAsync(b->elev.p, elevation, n * sizeof(float), cudaMemcpyHostToDevice, b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  b->pal_veg.assign(class_veg, class_veg + n_classes);
  b->h_fuel.assign(fuel_class, fuel_class + n);
  b->h_elev.assign(elevation, elevation + n);
  b->h_terrain_stale = false;
  b->pal_den.assign(class_den, class_den + n_classes);
  b->cellsize = cellsize;
  b->mode = ebl::kStaticTerrain;
  b->n_grids = n_grids;
  b->derived_dirty = true;
  b->slope_dirty = true;
  b->det_tables_valid = false;
  b->det_S_valid = false;
  b->pot.reset();
  b->gamma.reset();
  if (b->n_winds == 0) {  // calm air until set
    b->n_winds = 1;
    b->wind_speed.assign(1, 0.0);
    b->wind_dir.assign(1, 0.0);
  }
  return EBL_OK;
}

namespace {
// Terrain-form bookkeeping once fuel/elev hold device-built layers for n_grids grids.
void adopt_device_terrain(ebl_batch* b, int n_grids, std::vector<double> veg, std::vector<double> den,
                          double cellsize) {
  b->pal_veg = std::move(veg);
  b->pal_den = std::move(den);
  b->h_fuel.clear();
  b->h_elev.clear();
  b->h_terrain_stale = true;
  b->cellsize = cellsize;
  b->mode = ebl::kStaticTerrain;
  b->n_grids = n_grids;
  b->derived_dirty = true;
  b->slope_dirty = true;
  b->det_tables_valid = false;
  b->det_S_valid = false;
  b->pot.reset();
  b->gamma.reset();
  if (b->n_winds == 0) {
    b->n_winds = 1;
    b->wind_speed.assign(1, 0.0);
    b->wind_dir.assign(1, 0.0);
  }
}
}  // namespace

int ebl_batch_synth_terrain(ebl_batch* b, uint64_t seed, uint32_t env_id0, double elev_max,
                            double wind_max, double cellsize) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (!(cellsize > 0.0) || !std::isfinite(cellsize))
    return set_err(EBL_EINVAL, "raster_from_model: cellsize must be positive");
  if (!std::isfinite(elev_max)) return set_err(EBL_EINVAL, "elev_max must be finite");
  if (!std::isfinite(wind_max)) return set_err(EBL_EINVAL, "WindField: non-finite speed");
  if (wind_max < 0.0) return set_err(EBL_EINVAL, "WindField: negative speed");
  if (b->h < 2 || b->w < 2) return set_err(EBL_EINVAL, "synth_terrain: need n_envs >= 1, dims >= 2");
  if (b->n_envs > 65535) return set_err(EBL_EINVAL, "device terrain synthesis supports at most 65535 envs per batch");
  EBL_CUDA(cudaSetDevice(b->device));
  const size_t n = b->ncell * b->n_envs;
  EBL_CUDA(b->fuel.alloc(n));
  EBL_CUDA(b->elev.alloc(n));
  DevBuf<double> scratch;
  DevBuf<unsigned long long> mm;
  DevBuf<unsigned int> hist;
  DevBuf<int> thr;
  EBL_CUDA(scratch.alloc(n));
  EBL_CUDA(mm.alloc(static_cast<size_t>(b->n_envs) * 4));
  EBL_CUDA(hist.alloc(static_cast<size_t>(b->n_envs) * 4096));
  EBL_CUDA(thr.alloc(static_cast<size_t>(b->n_envs) * 10));
  ebl::SynthArgs a{};
  a.seed = seed;
  a.env_id0 = env_id0;
  a.n_envs = b->n_envs;
  a.h = b->h;
  a.w = b->w;
  a.lc_base = std::min(64, std::max(4, std::min(b->h, b->w) / 4));   // ember_host.cpp synth_one
  a.el_base = std::min(128, std::max(8, std::min(b->h, b->w) / 2));
  a.elev_max = elev_max;
  a.fuel = b->fuel.p;
  a.elev = b->elev.p;
  a.scratch = scratch.p;
  a.mm = mm.p;
  a.hist = hist.p;
  a.thr = thr.p;
  EBL_CUDA(ebl::launch_synth_terrain(a, b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  std::vector<double> veg(11), den(11);
  ebl::worldcover_palette(nullptr, veg.data(), den.data());
  adopt_device_terrain(b, b->n_envs, std::move(veg), std::move(den), cellsize);
  // per-env wind exactly as the host generator draws it
  std::vector<double> speed(b->n_envs), dir(b->n_envs);
  for (int e = 0; e < b->n_envs; ++e) {
    const uint64_t stream = env_id0 + static_cast<uint64_t>(e);
    speed[e] = wind_max * ebl::rng_uniform(seed, 3000, stream, 0, 3);
    dir[e] = 2.0 * 3.14159265358979323846 * ebl::rng_uniform(seed, 3000, stream, 1, 3);
  }
  b->n_winds = b->n_envs;
  b->sched_len = 0;
  b->wind_speed = std::move(speed);
  b->wind_dir = std::move(dir);
  return EBL_OK;
}

int ebl_batch_synth_ignitions(ebl_batch* b, uint64_t seed, uint32_t env_id0, int count, int* placed_total) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_sync(b)) return e;
  if (b->mode != ebl::kStaticTerrain) return set_err(EBL_ESTATE, "ignitions need terrain-form static layers");
  if (count < 0) return set_err(EBL_EINVAL, "EnvConfig: ignition_count must be >= 0");
  if (int e = prepare(b)) return e;  // burnable flags live in pal64[512..767]
  DevBuf<int> placed;
  EBL_CUDA(placed.alloc(b->n_envs));
  ebl::IgniteArgs a{};
  a.seed = seed;
  a.env_id0 = env_id0;
  a.n_envs = b->n_envs;
  a.h = b->h;
  a.w = b->w;
  a.count = count;
  a.fuel = b->fuel.p;
  a.fuel_stride = b->n_grids > 1 ? b->ncell : 0;
  a.burnable = b->pal64.p + 512;
  a.states = b->state[b->cur].p;
  a.placed = placed.p;
  EBL_CUDA(ebl::launch_synth_ignitions(a, b->stream));
  std::vector<int> h(b->n_envs);
  EBL_CUDA(cudaMemcpyAsync(h.data(), placed.p, h.size() * sizeof(int), cudaMemcpyDeviceToHost, b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  b->counts_valid = false;
  if (placed_total) {
    long long t = 0;
    for (int v : h) t += v;
    *placed_total = static_cast<int>(t);
  }
  return EBL_OK;
}

int ebl_batch_get_terrain(ebl_batch* b, uint8_t* fuel_class, float* elevation) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (b->mode != ebl::kStaticTerrain) return set_err(EBL_ESTATE, "no terrain-form static layers on the batch");
  EBL_CUDA(cudaSetDevice(b->device));
  const size_t n = b->ncell * b->n_grids;
  if (fuel_class) EBL_CUDA(cudaMemcpyAsync(fuel_class, b->fuel.p, n, cudaMemcpyDeviceToHost, b->stream));
  if (elevation) EBL_CUDA(cudaMemcpyAsync(elevation, b->elev.p, n * sizeof(float), cudaMemcpyDeviceToHost, b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  return EBL_OK;
}

int ebl_batch_set_landcover(ebl_batch* b, int n_grids, const int32_t* landcover, const float* elevation,
                            int has_nodata, int32_t nodata_code, int n_codes, const int32_t* codes,
                            const double* veg, const double* den, int has_fallback, double fallback_veg,
                            double fallback_den, double cellsize) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (n_grids != 1 && n_grids != b->n_envs) return set_err(EBL_EINVAL, "n_grids must be 1 or n_envs");
  if (!landcover || !elevation) return set_err(EBL_EINVAL, "null layer");
  if (n_codes < 0 || n_codes > 254) return set_err(EBL_EINVAL, "a fuel table holds at most 254 codes");
  if (n_codes > 0 && (!codes || !veg || !den)) return set_err(EBL_EINVAL, "null fuel table");
  if (!(cellsize > 0.0) || !std::isfinite(cellsize))
    return set_err(EBL_EINVAL, "raster_from_model: cellsize must be positive");
  auto in_range = [](double v) { return std::isfinite(v) && v >= -1.0 && v <= 1.0; };
  // FuelTable::set / set_fallback (geodata.cpp:231-247); a repeated code keeps the last entry
  std::vector<std::pair<int32_t, int>> order;
  for (int k = 0; k < n_codes; ++k) {
    if (!in_range(veg[k]) || !in_range(den[k]))
      return set_err(EBL_EINVAL, "FuelTable: modifiers for code " + std::to_string(codes[k]) +
                                     " must lie in [-1, 1]");
    order.emplace_back(codes[k], k);
  }
  if (has_fallback && (!in_range(fallback_veg) || !in_range(fallback_den)))
    return set_err(EBL_EINVAL, "FuelTable: fallback modifiers must lie in [-1, 1]");
  std::stable_sort(order.begin(), order.end(), [](auto& x, auto& y) { return x.first < y.first; });
  std::vector<int32_t> sorted;
  std::vector<double> pv, pd;
  for (size_t i = 0; i < order.size(); ++i) {
    if (i + 1 < order.size() && order[i + 1].first == order[i].first) continue;  // last set wins
    sorted.push_back(order[i].first);
    pv.push_back(veg[order[i].second]);
    pd.push_back(den[order[i].second]);
  }
  const int nc = static_cast<int>(sorted.size());
  const int fallback_index = has_fallback ? nc : -1;
  if (has_fallback) {
    pv.push_back(fallback_veg);
    pd.push_back(fallback_den);
  }
  const int nodata_index = static_cast<int>(pv.size());
  pv.push_back(-1.0);  // nodata cells are inert (geodata.cpp:330-334)
  pd.push_back(-1.0);
  const size_t n = b->ncell * n_grids;
  for (size_t i = 0; i < n; ++i)
    if (std::isinf(elevation[i])) return set_err(EBL_EINVAL, "elevation must be finite or NaN (nodata)");
  EBL_CUDA(cudaSetDevice(b->device));
  DevBuf<int32_t> lc, dcodes;
  DevBuf<unsigned long long> missing;
  EBL_CUDA(lc.alloc(n));
  EBL_CUDA(dcodes.alloc(std::max(1, nc)));
  EBL_CUDA(missing.alloc(1));
  EBL_CUDA(b->fuel.alloc(n));
  EBL_CUDA(b->elev.alloc(n));
  EBL_CUDA(cudaMemcpyAsync(lc.p, landcover, n * sizeof(int32_t), cudaMemcpyHostToDevice, b->stream));
  EBL_CUDA(cudaMemcpyAsync(b->elev.p, elevation, n * sizeof(float), cudaMemcpyHostToDevice, b->stream));
  if (nc) EBL_CUDA(cudaMemcpyAsync(dcodes.p, sorted.data(), nc * sizeof(int32_t), cudaMemcpyHostToDevice, b->stream));
  EBL_CUDA(cudaMemsetAsync(missing.p, 0xff, sizeof(unsigned long long), b->stream));
  ebl::LandcoverArgs a{};
  a.n = n;
  a.landcover = lc.p;
  a.elev = b->elev.p;
  a.codes = dcodes.p;
  a.n_codes = nc;
  a.fallback_index = fallback_index;
  a.nodata_index = nodata_index;
  a.has_nodata = has_nodata;
  a.nodata_code = nodata_code;
  a.fuel = b->fuel.p;
  a.missing = missing.p;
  EBL_CUDA(ebl::launch_landcover_map(a, b->stream));
  unsigned long long miss = 0;
  EBL_CUDA(cudaMemcpyAsync(&miss, missing.p, sizeof(miss), cudaMemcpyDeviceToHost, b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  if (miss != ~0ull) {
    b->mode = ebl::kStaticNone;  // layers half-built: the batch has no usable statics
    return set_err(EBL_EFILE, "fuel table has no entry for landcover code " + std::to_string(landcover[miss]));
  }
  adopt_device_terrain(b, n_grids, std::move(pv), std::move(pd), cellsize);
  return EBL_OK;
}

int ebl_batch_set_wind(ebl_batch* b, int n_winds, const double* speed, const double* dir) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (n_winds != 1 && n_winds != b->n_envs) return set_err(EBL_EINVAL, "n_winds must be 1 or n_envs");
  for (int i = 0; i < n_winds; ++i) {
    if (!std::isfinite(speed[i])) return set_err(EBL_EINVAL, "WindField: non-finite speed");
    if (speed[i] < 0.0) return set_err(EBL_EINVAL, "WindField: negative speed");
    if (!std::isfinite(dir[i])) return set_err(EBL_EINVAL, "WindField: non-finite direction");
  }
  b->n_winds = n_winds;
  b->sched_len = 0;
  b->wind_speed.assign(speed, speed + n_winds);
  b->wind_dir.assign(dir, dir + n_winds);
  b->derived_dirty = true;
  b->det_tables_valid = false;
  return EBL_OK;
}

int ebl_batch_set_wind_schedule(ebl_batch* b, int n_sched, int n_winds, const double* speed,
                                const double* dir) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (n_sched == 0) return ebl_batch_set_wind(b, n_winds, speed, dir);  // constant wind
  if (n_sched < 0) return set_err(EBL_EINVAL, "schedule length must be >= 0");
  if (n_winds != 1 && n_winds != b->n_envs) return set_err(EBL_EINVAL, "n_winds must be 1 or n_envs");
  const size_t m = static_cast<size_t>(n_sched) * n_winds;
  for (size_t i = 0; i < m; ++i) {
    if (!std::isfinite(speed[i])) return set_err(EBL_EINVAL, "WindField: non-finite speed");
    if (speed[i] < 0.0) return set_err(EBL_EINVAL, "WindField: negative speed");
    if (!std::isfinite(dir[i])) return set_err(EBL_EINVAL, "WindField: non-finite direction");
  }
  b->n_winds = n_winds;
  b->sched_len = n_sched;
  b->wind_speed.assign(speed, speed + m);
  b->wind_dir.assign(dir, dir + m);
  b->derived_dirty = true;
  b->det_tables_valid = false;
  return EBL_OK;
}

int ebl_batch_set_grid_wind_schedule(ebl_batch* b, int n_sched, const double* speed, const double* dir) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (b->mode != ebl::kStaticTables) return set_err(EBL_ESTATE, "a per-cell wind schedule needs ebl_batch_set_grid first");
  if (n_sched < 0) return set_err(EBL_EINVAL, "schedule length must be >= 0");
  const size_t m = static_cast<size_t>(n_sched) * b->ncell * b->n_grids;
  for (size_t i = 0; i < m; ++i) {  // WindSchedule of WindFields (engine.cpp:74-86, grid.cpp:49-62)
    if (!std::isfinite(speed[i])) return set_err(EBL_EINVAL, "WindField: non-finite speed");
    if (speed[i] < 0.0) return set_err(EBL_EINVAL, "WindField: negative speed");
    if (!std::isfinite(dir[i])) return set_err(EBL_EINVAL, "WindField: non-finite direction");
  }
  b->sched_len = n_sched;
  b->g_sched_speed.assign(speed, speed + m);
  b->g_sched_dir.assign(dir, dir + m);
  b->tables_dirty = true;
  return EBL_OK;
}

int ebl_step_batch_record(ebl_batch* b, int n_steps, void* traj, int on_device) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_sync(b)) return e;
  if (n_steps < 0 || (n_steps > 0 && !traj)) return set_err(EBL_EINVAL, "bad trajectory arguments");
  if (n_steps == 0) return EBL_OK;
  const size_t bytes = static_cast<size_t>(n_steps) * b->n_envs * b->ncell;
  DevBuf<uint8_t> tmp;
  uint8_t* dst = static_cast<uint8_t*>(traj);
  if (!on_device) {
    EBL_CUDA(tmp.alloc(bytes));
    dst = tmp.p;
  }
  b->traj_out = dst;
  const int rc = ebl_step_batch(b, n_steps);
  b->traj_out = nullptr;
  if (rc) return rc;
  if (!on_device) {
    EBL_CUDA(cudaMemcpyAsync(traj, tmp.p, bytes, cudaMemcpyDeviceToHost, b->stream));
    EBL_CUDA(cudaStreamSynchronize(b->stream));
  }
  return EBL_OK;
}

int ebl_batch_set_state(ebl_batch* b, const uint8_t* states) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_sync(b)) return e;
  // Like the reference's FireLayer (a plain Grid<FireState>, grid.hpp:100) member layers are
  // not validated; a byte other than 1/2 takes the Unburned path as in engine.cpp:15-25.
  const size_t total = b->ncell * b->n_envs;
  EBL_CUDA(cudaSetDevice(b->device));
  EBL_CUDA(cudaMemcpyAsync(b->state[b->cur].p, states, total, cudaMemcpyHostToDevice, b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  b->counts_valid = false;
  return EBL_OK;
}

int ebl_batch_get_state(ebl_batch* b, uint8_t* states) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_sync(b, true)) return e;
  EBL_CUDA(cudaSetDevice(b->device));
  EBL_CUDA(cudaMemcpyAsync(states, b->state[b->cur].p, b->ncell * b->n_envs, cudaMemcpyDeviceToHost, b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  return EBL_OK;
}

int ebl_batch_set_state_device(ebl_batch* b, const void* d) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_sync(b)) return e;
  EBL_CUDA(cudaMemcpyAsync(b->state[b->cur].p, d, b->ncell * b->n_envs, cudaMemcpyDeviceToDevice, b->stream));
  b->counts_valid = false;
  return EBL_OK;
}

int ebl_batch_get_state_device(ebl_batch* b, void* d) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_sync(b)) return e;
  EBL_CUDA(cudaMemcpyAsync(d, b->state[b->cur].p, b->ncell * b->n_envs, cudaMemcpyDeviceToDevice, b->stream));
  return EBL_OK;
}

void* ebl_batch_state_device_ptr(ebl_batch* b) {
  if (!b || rl_sync_bytes(b) != EBL_OK) return nullptr;
  return b->state[b->cur].p;
}

int ebl_batch_set_key(ebl_batch* b, uint64_t seed, uint64_t step, const uint64_t* streams,
                      uint64_t first_stream) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  b->seed = seed;
  b->step = step;
  bool changed = false;
  for (int e = 0; e < b->n_envs; ++e) {
    const uint64_t s = streams ? streams[e] : first_stream + e;
    changed |= b->h_streams[e] != s;
    b->h_streams[e] = s;
  }
  if (!changed && b->streams_uploaded) return EBL_OK;  // seed/step travel as kernel arguments
  EBL_CUDA(cudaSetDevice(b->device));
  EBL_CUDA(cudaMemcpyAsync(b->streams.p, b->h_streams.data(), b->n_envs * sizeof(uint64_t),
                           cudaMemcpyHostToDevice, b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  b->streams_uploaded = true;
  return EBL_OK;
}

uint64_t ebl_batch_step_index(const ebl_batch* b) { return b ? b->step : 0; }

int ebl_batch_set_kernel(ebl_batch* b, int which) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (which < EBL_KERNEL_AUTO || which > EBL_KERNEL_WARP || which == 4 || which == 5)
    return set_err(EBL_EINVAL, "unknown kernel");
  if (which == EBL_KERNEL_RESIDENT && !ebl::resident_fits(b->h, b->w))
    return set_err(EBL_EINVAL, "env too large for the resident kernel");
  b->kernel = which;
  return EBL_OK;
}

int ebl_step_batch(ebl_batch* b, int n_steps) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_sync(b, true)) return e;
  if (n_steps < 0) return set_err(EBL_EINVAL, "n_steps must be >= 0");
  if (n_steps == 0) return EBL_OK;
  if (int e = prepare(b)) return e;
  if (b->kernel == EBL_KERNEL_TILED) {  // one step per launch (the simple per-cell kernel)
    for (int t = 0; t < n_steps; ++t) {
      ebl::StepArgs a = step_args(b);
      if (t == n_steps - 1) {
        EBL_CUDA(cudaMemsetAsync(b->counts.p, 0, b->n_envs * 4 * sizeof(int32_t), b->stream));
        a.counts = b->counts.p;
      }
      EBL_CUDA(ebl::launch_step_tile(a, b->mode, b->stream));
      b->cur ^= 1;
      b->step += 1;
      b->launches += 1;
      if (b->traj_out) {  // record: this step's layers
        const size_t layer = b->ncell * b->n_envs;
        EBL_CUDA(cudaMemcpyAsync(b->traj_out + t * layer, b->state[b->cur].p, layer,
                                 cudaMemcpyDeviceToDevice, b->stream));
      }
    }
  } else {  // bit-sliced blocked kernel: whole env per CTA when it fits, else halo tiles
    const bool force_tiles = b->kernel == EBL_KERNEL_BLOCKED;
    // tile activity records: valid from the 2nd launch of this call, or carried over from the
    // previous call when nothing but stepping / reads / halo-row writes happened in between
    int tf_par = b->tf_carry_par, tf_tiles = b->tf_carry_tiles;
    b->tf_carry_tiles = -1;
    int list_launch = -1;  // work-list run of this call: index of the launch, -1 = grid launches
    size_t list_tiles = 0;
    for (int done = 0; done < n_steps;) {
      ebl::BlockGeom g = ebl::plan_blocks(b->h, b->w, n_steps - done, force_tiles, 0, b->n_envs, 1);
      if (b->tile_h > 0) {  // test hook: explicit tiling
        g.envs_per_cta = 1;
        g.tile_h = b->tile_h;
        g.tile_w = b->tile_w;
        g.halo_rows = b->tile_halo;
        g.halo_cols = g.tile_w >= b->w ? 0 : 32;
        g.n_steps = std::min(n_steps - done, std::max(1, b->tile_halo));
        const int rh = std::min(b->h, g.tile_h + 2 * g.halo_rows);
        const int rw = std::min(b->w, g.tile_w + 2 * g.halo_cols);
        g.list_cap = std::max(1, rh * rw / 4);
      }
      apply_fixed_regions(b, g);
      ebl::StepArgs a = step_args(b);
      if (done + g.n_steps == n_steps) {
        EBL_CUDA(cudaMemsetAsync(b->counts.p, 0, b->n_envs * 4 * sizeof(int32_t), b->stream));
        a.counts = b->counts.p;
      }
      a.traj = b->traj_out;  // record: the kernel stores every step's tile (no extra launches)
      a.traj_t0 = static_cast<size_t>(done);
      {  // quiet-tile skipping (warp-local kernel, halo inside the 8 neighbour tiles, no recording)
        const int tx = (b->w + g.tile_w - 1) / g.tile_w, ty = (b->h + g.tile_h - 1) / g.tile_h;
        const bool exposed = a.keep_lo > 0 || a.keep_hi < b->h;  // halo rows of a row shard
        // (exposed halo tiles need tile_h >= 3 halo for the distance argument; marked ones do not)
        const bool tiled = tx * ty > 1 && g.halo_rows <= g.tile_h && g.halo_cols <= g.tile_w && !a.traj &&
                           use_warp(b) && (!exposed || halo_marks_on() || g.tile_h >= 3 * g.halo_rows);
        // work-list run: the whole call on one unsharded batch with no records carried in; after the
        // first (grid) launch only the tiles the skip rule would not skip are launched, on persistent
        // CTAs (EBL_WORK_LIST=0 keeps grid launches with per-CTA skipping)
        static const bool work_list = [] {
          const char* e = std::getenv("EBL_WORK_LIST");
          return !e || std::atoi(e) != 0;
        }();
        if (tiled && work_list && !exposed && (list_launch >= 0 || (tf_tiles < 0 && n_steps > g.n_steps))) {
          const size_t nt = static_cast<size_t>(tx) * ty * b->n_envs;
          if (b->trec.n < nt * 4 || b->tqueued.n < nt) {
            EBL_CUDA(b->trec.alloc(nt * 4));
            EBL_CUDA(b->tqueued.alloc(nt));
            EBL_CUDA(cudaMemsetAsync(b->tqueued.p, 0, nt * sizeof(int32_t), b->stream));
            b->list_stamp = 0;
          }
          for (auto& l : b->tlist)
            if (l.n < nt) EBL_CUDA(l.alloc(nt));
          if (b->tcount.n < 6) EBL_CUDA(b->tcount.alloc(6));  // append counters [3] + cursors [3]
          list_launch += 1;
          list_tiles = nt;
          if (list_launch == 0) EBL_CUDA(cudaMemsetAsync(b->tcount.p, 0, 6 * sizeof(int32_t), b->stream));
          // the run's first launch over every tile is replaced by k_tile_init (copy + records + the
          // first list): the first step launch already runs a work list (EBL_TILE_INIT=0: grid launch)
          if (list_launch == 0 && tile_init_on()) {
            const int32_t stamp0 = ++b->list_stamp;
            EBL_CUDA(ebl::launch_tile_init(b->state[b->cur].p, b->state[b->cur ^ 1].p, b->h, b->w, b->n_envs, g.tile_h,
                                           g.tile_w, b->trec.p, b->tqueued.p, stamp0, b->tlist[1].p, b->tcount.p + 1,
                                           a.store_lo, a.store_hi, b->stream));
            b->launches += 1;
            list_launch = 1;
          }
          const int cur_l = list_launch & 1, nxt = cur_l ^ 1, c3 = list_launch % 3;
          a.list_mode = list_launch == 0 ? 1 : 2;
          a.trec = b->trec.p;
          a.queued = b->tqueued.p;
          a.list_stamp = ++b->list_stamp;
          a.next_list = b->tlist[nxt].p;
          a.next_count = b->tcount.p + (c3 + 1) % 3;
          a.tile_list = b->tlist[cur_l].p;
          a.tile_count = b->tcount.p + c3;
          a.list_cursor = b->tcount.p + 3 + c3;
          a.list_zero0 = b->tcount.p + (c3 + 2) % 3;      // zeroed by this launch for the one after next
          a.list_zero1 = b->tcount.p + 3 + (c3 + 1) % 3;  // the next launch's cursor
          a.tiles_x = tx;
          a.tiles_y = ty;
          a.tiles_total = static_cast<int>(nt);
          tf_tiles = -1;
        } else if (tiled) {
          const size_t n = static_cast<size_t>(tx) * ty * b->n_envs * 4;
          for (auto& f : b->tflags)
            if (f.n < n) {
              EBL_CUDA(f.alloc(n));
              tf_tiles = -1;
            }
          const bool same = tf_tiles == tx * ty && b->tf_carry_th == g.tile_h && b->tf_carry_tw == g.tile_w;
          a.tflag_in = same ? b->tflags[tf_par].p : nullptr;
          // no records carried in (a call's or a row shard's first launch): k_tile_init writes them
          // from the layer (copy + {burning, streak 2 when canonical, U/B/X}) instead of the launch
          // stepping every tile -- the per-rank C3 form stepped 3.3 % of its tiles, 0.2 % after
          if (!same && tile_init_on()) {
            EBL_CUDA(ebl::launch_tile_init(b->state[b->cur].p, b->state[b->cur ^ 1].p, b->h, b->w, b->n_envs,
                                           g.tile_h, g.tile_w, b->tflags[tf_par].p, nullptr, 0, nullptr, nullptr,
                                           a.store_lo, a.store_hi, b->stream));
            b->launches += 1;
            a.tflag_in = b->tflags[tf_par].p;
          }
          a.tflag_out = b->tflags[tf_par ^ 1].p;
          // halo rows written between calls mark the records they reach (mark_halo_rows), so a
          // row shard's halo tiles follow the skip rule too (EBL_HALO_MARKS=0: exposed instead)
          a.halo_marked = halo_marks_on() ? 1 : 0;
          tf_par ^= 1;
          tf_tiles = tx * ty;
          b->tf_carry_th = g.tile_h;
          b->tf_carry_tw = g.tile_w;
        } else {
          tf_tiles = -1;
        }
      }
      // whole-env launches leave the step loop once the fire is out: C1 kernel 0.495 -> 0.476 ms
      // (a separate instantiation: the host-buffer pipeline measured better on the plain one,
      // ebl_batch_run e2e 4.38e12 vs 4.30e12; scripts/lib_ab.sh)
      a.early_exit = g.tile_h >= b->h && g.tile_w >= b->w;
      EBL_CUDA(launch_ca(b, a, g, b->stream));
      b->cur ^= 1;
      b->step += g.n_steps;
      b->launches += 1;
      done += g.n_steps;
      if (list_launch >= 0 && done == n_steps) {  // U/B/X of every tile from the in-place records
        EBL_CUDA(ebl::launch_tile_counts(b->trec.p, b->n_envs, static_cast<int>(list_tiles / b->n_envs),
                                         b->counts.p, b->stream));
        b->launches += 1;
      }
    }
    b->tf_carry_tiles = tf_tiles;
    b->tf_carry_par = tf_par;
  }
  b->steps_done += n_steps;
  b->counts_valid = true;
  return EBL_OK;
}

int ebl_batch_set_pipeline(ebl_batch* b, int chunks) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (chunks < 0 || chunks > 256) return set_err(EBL_EINVAL, "pipeline chunks must be in [0, 256]");
  b->pipe_chunks = chunks;
  return EBL_OK;
}

// set_state + step_batch x n_steps + get_state from/to HOST buffers, pipelined over env chunks:
// chunk c's H2D copy (copy-in stream, in order), its fused n-step launch (own stream, after the
// copy), its D2H copy (copy-out stream, after the launch) -- transfers of later/earlier chunks
// overlap the compute of the others.  Identical results to the unpipelined sequence (envs are
// independent; the RNG is keyed by stream, not by launch).  Pinned host buffers are needed for
// the copies to be asynchronous.
int ebl_batch_run(ebl_batch* b, const uint8_t* initial, int n_steps, uint8_t* final_states) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_sync(b)) return e;
  if (!initial || !final_states) return set_err(EBL_EINVAL, "null state buffer");
  if (n_steps < 0) return set_err(EBL_EINVAL, "n_steps must be >= 0");
  if (int e = prepare(b)) return e;
  const bool resident = b->kernel != EBL_KERNEL_TILED && b->kernel != EBL_KERNEL_BLOCKED &&
                        b->tile_h == 0 && ebl::resident_fits(b->h, b->w);
  int chunks = b->pipe_chunks > 0 ? b->pipe_chunks : 4;  // C1 e2e: 4 chunks 0.84 ms, 8: 0.92, 2: 0.89
  chunks = std::min(chunks, b->n_envs);
  if (!resident || n_steps == 0 || chunks <= 1) {  // one launch per step set: plain sequence
    int rc;
    if ((rc = ebl_batch_set_state(b, initial))) return rc;
    if ((rc = ebl_step_batch(b, n_steps))) return rc;
    return ebl_batch_get_state(b, final_states);
  }
  EBL_CUDA(cudaSetDevice(b->device));
  if (int e = ensure_pipeline(b, chunks)) return e;
  const ebl::BlockGeom g = ebl::plan_blocks(b->h, b->w, n_steps, false, 0, b->n_envs, 1);
  ebl::StepArgs a = step_args(b);
  a.counts = b->counts.p;
  // everything earlier on the batch stream (state/key uploads, statics) happens first
  EBL_CUDA(cudaEventRecord(b->pipe_ev_start, b->stream));
  EBL_CUDA(cudaStreamWaitEvent(b->pipe_in, b->pipe_ev_start, 0));
  for (int c = 0; c < chunks; ++c) EBL_CUDA(cudaStreamWaitEvent(b->pipe_comp[c], b->pipe_ev_start, 0));
  // chunk boundaries: weight of chunk c = ratio^c, equal chunks by default (measured best:
  // scripts/pipeline_ratio_sweep.sh; EBL_PIPE_RATIO < 1 makes the later chunks smaller)
  std::vector<int> bound(chunks + 1, 0);
  {
    static const double ratio = [] {
      const char* e = std::getenv("EBL_PIPE_RATIO");
      return e ? std::atof(e) : 1.0;  // C1 e2e, 4 chunks: equal 4.12e12, 0.7: 3.95e12, 0.5: 3.79e12
    }();
    std::vector<double> wgt(chunks);
    double tot = 0.0, acc = 0.0;
    for (int c = 0; c < chunks; ++c) tot += (wgt[c] = std::pow(ratio, c));
    for (int c = 0; c < chunks; ++c) {
      acc += wgt[c];
      bound[c + 1] = std::min(b->n_envs, static_cast<int>(std::lround(acc / tot * b->n_envs)));
    }
    bound[chunks] = b->n_envs;
  }
  // the final layers straight into the caller's buffer when it is mapped pinned memory: each CTA
  // writes its env as it finishes, no device -> host copy after the chunk's launch
  // (the kernels store 16-byte vectors: an unaligned mapping falls back to the DMA copy)
  uint8_t* host_dev = nullptr;
  {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, final_states) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
        pa.devicePointer && (reinterpret_cast<uintptr_t>(pa.devicePointer) & 15) == 0)
      host_dev = static_cast<uint8_t*>(pa.devicePointer);
    cudaGetLastError();
  }
  a.out2 = host_dev;
  // trailing chunks with zero-copy output: the later half by default (C1 e2e, 4 chunks: all 4.07e12,
  // last 1 4.11e12, last 2 4.29e12; scripts/pipeline_zc_sweep.sh); EBL_PIPE_ZC overrides
  static const int zc_env = [] {
    const char* e = std::getenv("EBL_PIPE_ZC");
    return e ? std::atoi(e) : -1;
  }();
  const int zc_keep = zc_env >= 0 ? zc_env : (chunks + 1) / 2;
  const int zc_from = host_dev ? std::max(0, chunks - zc_keep) : chunks;
  static const int pipe_exit = [] {  // the early-exit instantiation for the pipeline's launches too
    const char* e = std::getenv("EBL_PIPE_EXIT");
    return e ? std::atoi(e) : 0;
  }();
  a.early_exit = pipe_exit;
  for (int c = 0; c < chunks; ++c) {
    const int off = bound[c], n = bound[c + 1] - off;
    if (n <= 0) continue;
    const size_t bytes = static_cast<size_t>(n) * b->ncell, boff = static_cast<size_t>(off) * b->ncell;
    EBL_CUDA(cudaMemcpyAsync(b->state[b->cur].p + boff, initial + boff, bytes, cudaMemcpyHostToDevice, b->pipe_in));
    EBL_CUDA(cudaEventRecord(b->pipe_ev_in[c], b->pipe_in));
  }
  for (int c = 0; c < chunks; ++c) {
    const int off = bound[c], n = bound[c + 1] - off;
    if (n <= 0) continue;
    cudaStream_t s = b->pipe_comp[c];
    EBL_CUDA(cudaStreamWaitEvent(s, b->pipe_ev_in[c], 0));
    EBL_CUDA(cudaMemsetAsync(b->counts.p + static_cast<size_t>(off) * 4, 0, static_cast<size_t>(n) * 4 * sizeof(int32_t), s));
    // mapped output: only the chunks whose envs can still be running after the last input copy
    // write their layers over PCIe from the kernel (zero_copy_from on); earlier chunks are copied
    // back by DMA once the inputs are all in, so their results do not share the link with the
    // input stream
    ebl::StepArgs ca = chunk_args(b, a, off, n);
    if (c < zc_from) ca.out2 = nullptr;
    EBL_CUDA(launch_ca(b, ca, g, s));
    EBL_CUDA(cudaEventRecord(b->pipe_ev_done[c], s));
  }
  EBL_CUDA(cudaStreamWaitEvent(b->pipe_out, b->pipe_ev_in[chunks - 1], 0));
  for (int c = 0; c < chunks; ++c) {
    const int off = bound[c], n = bound[c + 1] - off;
    if (n <= 0) continue;
    const size_t bytes = static_cast<size_t>(n) * b->ncell, boff = static_cast<size_t>(off) * b->ncell;
    EBL_CUDA(cudaStreamWaitEvent(b->pipe_out, b->pipe_ev_done[c], 0));
    if (!host_dev || c < zc_from)
      EBL_CUDA(cudaMemcpyAsync(final_states + boff, b->state[b->cur ^ 1].p + boff, bytes, cudaMemcpyDeviceToHost,
                               b->pipe_out));
  }
  EBL_CUDA(cudaEventRecord(b->pipe_ev_end, b->pipe_out));
  EBL_CUDA(cudaStreamWaitEvent(b->stream, b->pipe_ev_end, 0));  // later batch work follows the run
  EBL_CUDA(cudaStreamSynchronize(b->pipe_out));
  b->cur ^= 1;
  b->step += n_steps;
  b->launches += chunks;
  b->steps_done += n_steps;
  b->counts_valid = true;
  return EBL_OK;
}

int ebl_batch_set_row_offset(ebl_batch* b, int64_t row_off) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (row_off < 0) return set_err(EBL_EINVAL, "row offset must be >= 0");
  b->row_off = row_off;
  return EBL_OK;
}

int ebl_batch_copy_rows(ebl_batch* dst, int dst_row, const ebl_batch* src, int src_row, int n_rows) {
  EBL_DEVICE_GUARD(dst);
  // the source is only read; halo-row writes outside the destination's band keep its records
  const bool halo_only = dst && dst->band_lo >= 0 && (dst_row + n_rows <= dst->band_lo || dst_row >= dst->band_hi);
  if (int e = check_sync(dst, halo_only)) return e;
  if (int e = check_sync(const_cast<ebl_batch*>(src), true)) return e;
  if (dst->w != src->w || dst->n_envs != src->n_envs) return set_err(EBL_EINVAL, "copy_rows: widths/env counts differ");
  if (n_rows < 0 || dst_row < 0 || src_row < 0 || dst_row + n_rows > dst->h || src_row + n_rows > src->h)
    return set_err(EBL_EINVAL, "copy_rows: row range outside a layer");
  if (n_rows == 0) return EBL_OK;
  EBL_CUDA(cudaSetDevice(src->device));
  EBL_CUDA(cudaStreamSynchronize(src->stream));  // src rows final
  EBL_CUDA(cudaSetDevice(dst->device));
  if (dst->device != src->device) {  // direct NVLink peer access when the pair supports it
    int can = 0;
    if (cudaDeviceCanAccessPeer(&can, dst->device, src->device) == cudaSuccess && can) {
      const cudaError_t pe = cudaDeviceEnablePeerAccess(src->device, 0);
      if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) return set_err(EBL_ECUDA, cudaGetErrorString(pe));
      cudaGetLastError();  // clear "already enabled"
    }
  }
  const size_t bytes = static_cast<size_t>(n_rows) * dst->w;
  for (int e = 0; e < dst->n_envs; ++e) {
    uint8_t* d = dst->state[dst->cur].p + e * dst->ncell + static_cast<size_t>(dst_row) * dst->w;
    const uint8_t* s = src->state[src->cur].p + e * src->ncell + static_cast<size_t>(src_row) * src->w;
    if (dst->device == src->device) {
      EBL_CUDA(cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice, dst->stream));
    } else {  // NVLink peer copy
      EBL_CUDA(cudaMemcpyPeerAsync(d, dst->device, s, src->device, bytes, dst->stream));
    }
  }
  if (halo_only) EBL_CUDA(mark_halo_rows(dst, dst_row, n_rows));
  dst->counts_valid = false;
  return EBL_OK;
}

int ebl_batch_set_band(ebl_batch* b, int row_lo, int row_hi) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (row_lo < 0 || row_hi > b->h || row_lo >= row_hi) return set_err(EBL_EINVAL, "band outside the layer");
  b->band_lo = row_lo;
  b->band_hi = row_hi;
  return EBL_OK;
}

// Row shards stepped together with the halo exchange fused into the kernels: every K-step launch
// of shard s stores its band rows that neighbour s+-1 holds as halo straight into the neighbour's
// output layer (peer stores over NVLink when the shards sit on different GPUs); shard s waits
// (stream events, no host sync) for its neighbours' previous launches before the next one.
int ebl_shards_step(ebl_batch** shards, int n_shards, int n_steps, int halo) {
  if (!shards || n_shards < 1) return set_err(EBL_EINVAL, "no shards");
  EBL_DEVICE_GUARD(shards[0]);
  if (n_steps < 0) return set_err(EBL_EINVAL, "n_steps must be >= 0");
  if (halo < 1) return set_err(EBL_EINVAL, "halo must be >= 1");
  for (int s = 0; s < n_shards; ++s) {
    ebl_batch* b = shards[s];
    if (int e = check_sync(b)) return e;
    if (b->n_envs != 1 || b->w != shards[0]->w) return set_err(EBL_EINVAL, "shards: one env each, equal widths");
    if (b->band_lo < 0) return set_err(EBL_ESTATE, "shards: ebl_batch_set_band first");
    if (b->kernel == EBL_KERNEL_TILED) return set_err(EBL_EINVAL, "shards: blocked kernel only");
    // every side with a neighbour must hold the light cone of one chunk (k <= halo steps), or
    // reach the landscape's edge there
    const int k0 = n_shards > 1 ? std::min(halo, std::max(n_steps, 1)) : 0;
    const int64_t global_h = shards[n_shards - 1]->row_off + shards[n_shards - 1]->h;
    if ((s > 0 && b->band_lo < k0 && b->row_off > 0) ||
        (s + 1 < n_shards && b->h - b->band_hi < k0 && b->row_off + b->h < global_h))
      return set_err(EBL_EINVAL, "shards: a shard holds fewer halo rows than `halo` on a side with a neighbour");
    if (s > 0 && b->row_off + b->band_lo != shards[s - 1]->row_off + shards[s - 1]->band_hi)
      return set_err(EBL_EINVAL, "shards: bands must tile the landscape in order");
    if (int e = prepare(b)) return e;
    EBL_CUDA(cudaSetDevice(b->device));
    for (cudaEvent_t& e : b->shard_ev)
      if (!e) EBL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (int q = s - 1; q <= s + 1; q += 2) {  // NVLink peer access to the neighbours' layers
      if (q < 0 || q >= n_shards || shards[q]->device == b->device) continue;
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, b->device, shards[q]->device) != cudaSuccess || !can)
        return set_err(EBL_ECUDA, "shards: no peer access between neighbour GPUs");
      const cudaError_t pe = cudaDeviceEnablePeerAccess(shards[q]->device, 0);
      if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) return set_err(EBL_ECUDA, cudaGetErrorString(pe));
      cudaGetLastError();
    }
  }
  std::vector<uint8_t*> outs(n_shards);
  std::vector<ebl::BlockGeom> geo(n_shards);
  // quiet-tile records per shard across the chunks of this call; on work lists the neighbours
  // enqueue each other's tiles next to the halo rows they store (else those tiles are exposed:
  // never skipped; ember_warp.cu)
  std::vector<int> tf_par(n_shards, 0), tf_tiles(n_shards, -1);
  std::vector<int> list_launch(n_shards, -1);  // work-list runs per shard (ebl_step_batch's scheme)
  static const bool work_list = [] {
    const char* e = std::getenv("EBL_WORK_LIST");
    return !e || std::atoi(e) != 0;
  }();
  const bool halo_marks = halo_marks_on();
  const bool tile_init = tile_init_on();
  std::vector<ebl::StepArgs> args(n_shards);
  std::vector<char> listed(n_shards, 0);
  // shards sharing one device run on shard 0's stream (stream order replaces the per-chunk
  // events), and a chunk whose shards are all on work lists is ONE launch (k_step_warp_shards)
  bool single = n_shards <= ebl::kMaxShardLaunch;
  for (int s = 1; s < n_shards; ++s) single = single && shards[s]->device == shards[0]->device;
  cudaStream_t S0 = shards[0]->stream;
  auto strm = [&](int s) { return single ? S0 : shards[s]->stream; };
  if (single)
    for (int s = 1; s < n_shards; ++s) {  // the shards' pending work precedes the call
      EBL_CUDA(cudaEventRecord(shards[s]->shard_ev[0], shards[s]->stream));
      EBL_CUDA(cudaStreamWaitEvent(S0, shards[s]->shard_ev[0], 0));
    }
  EBL_CUDA(cudaSetDevice(shards[0]->device));
  int cur_dev = shards[0]->device;
  auto set_dev = [&](int d) -> cudaError_t {
    if (d == cur_dev) return cudaSuccess;
    cur_dev = d;
    return cudaSetDevice(d);
  };
  int chunk = 0;
  for (int done = 0; done < n_steps; ++chunk) {
    int k = n_shards > 1 ? std::min(halo, n_steps - done) : n_steps - done;
    for (int s = 0; s < n_shards; ++s) {  // tiling per shard; a chunk never outruns a light cone
      const ebl_batch* b = shards[s];
      ebl::BlockGeom g = ebl::plan_blocks(b->h, b->w, k, b->kernel == EBL_KERNEL_BLOCKED, 0, 1, 1);
      if (b->tile_h > 0) {
        g.envs_per_cta = 1;
        g.tile_h = b->tile_h;
        g.tile_w = b->tile_w;
        g.halo_rows = b->tile_halo;
        g.halo_cols = g.tile_w >= b->w ? 0 : 32;
        const int rh = std::min(b->h, g.tile_h + 2 * g.halo_rows);
        const int rw = std::min(b->w, g.tile_w + 2 * g.halo_cols);
        g.list_cap = std::max(1, rh * rw / 4);
      }
      apply_fixed_regions(b, g);
      if (g.halo_rows > 0 || g.halo_cols > 0) k = std::min(k, std::max(1, g.halo_rows));
      geo[s] = g;
    }
    for (int s = 0; s < n_shards; ++s) outs[s] = shards[s]->state[shards[s]->cur ^ 1].p;
    // pass 1: waits, counters and each shard's own launch parameters (list stamps included, which
    // the neighbours' marks need)
    for (int s = 0; s < n_shards; ++s) {
      ebl_batch* b = shards[s];
      EBL_CUDA(set_dev(b->device));
      // the neighbours' launches of the previous chunk (all waits precede this chunk's records)
      for (int q = s - 1; q <= s + 1 && chunk > 0 && !single; q += 2)
        if (q >= 0 && q < n_shards)
          EBL_CUDA(cudaStreamWaitEvent(b->stream, shards[q]->shard_ev[(chunk - 1) & 1], 0));
      ebl::BlockGeom& g = geo[s];
      g.n_steps = k;
      ebl::StepArgs a = step_args(b);
      if (done + k == n_steps) {  // counts of the last launch only
        EBL_CUDA(cudaMemsetAsync(b->counts.p, 0, 4 * sizeof(int32_t), strm(s)));
        a.counts = b->counts.p;
      }
      a.store_lo = b->band_lo;
      a.store_hi = b->band_hi;
      listed[s] = 0;
      {
        const int tx = (b->w + g.tile_w - 1) / g.tile_w, ty = (b->h + g.tile_h - 1) / g.tile_h;
        const bool exposed = a.keep_lo > 0 || a.keep_hi < b->h;
        // (exposed halo tiles need tile_h >= 3 halo; on work lists the neighbours mark them instead)
        const bool tiled = tx * ty > 1 && g.halo_rows <= g.tile_h && g.halo_cols <= g.tile_w && use_warp(b) &&
                           k <= std::max(1, g.halo_rows) &&
                           (!exposed || (work_list && halo_marks) || g.tile_h >= 3 * g.halo_rows);
        if (tiled && work_list && (list_launch[s] >= 0 || n_steps > k)) {
          // work list (halo tiles: marked by the neighbours, or exposed -- ember_warp.cu)
          const size_t nt = static_cast<size_t>(tx) * ty * b->n_envs;
          if (b->trec.n < nt * 4 || b->tqueued.n < nt) {
            EBL_CUDA(b->trec.alloc(nt * 4));
            EBL_CUDA(b->tqueued.alloc(nt));
            EBL_CUDA(cudaMemsetAsync(b->tqueued.p, 0, nt * sizeof(int32_t), strm(s)));
            b->list_stamp = 0;
          }
          for (auto& l : b->tlist)
            if (l.n < nt) EBL_CUDA(l.alloc(nt));
          if (b->tcount.n < 6) EBL_CUDA(b->tcount.alloc(6));
          int L = ++list_launch[s];
          if (L == 0) EBL_CUDA(cudaMemsetAsync(b->tcount.p, 0, 6 * sizeof(int32_t), strm(s)));
          if (L == 0 && tile_init) {  // records + first list instead of a grid launch (ebl_step_batch);
            // the shard's layer holds its halo rows' initial fire, so its own init lists those tiles
            const int32_t stamp0 = ++b->list_stamp;
            EBL_CUDA(ebl::launch_tile_init(b->state[b->cur].p, b->state[b->cur ^ 1].p, b->h, b->w, b->n_envs,
                                           g.tile_h, g.tile_w, b->trec.p, b->tqueued.p, stamp0, b->tlist[1].p,
                                           b->tcount.p + 1, a.store_lo, a.store_hi, strm(s)));
            L = list_launch[s] = 1;
          }
          const int c3 = L % 3;
          a.list_mode = L == 0 ? 1 : 2;
          a.trec = b->trec.p;
          a.queued = b->tqueued.p;
          a.list_stamp = ++b->list_stamp;
          a.next_list = b->tlist[(L & 1) ^ 1].p;
          a.next_count = b->tcount.p + (c3 + 1) % 3;
          a.tile_list = b->tlist[L & 1].p;
          a.tile_count = b->tcount.p + c3;
          a.list_cursor = b->tcount.p + 3 + c3;
          a.list_zero0 = b->tcount.p + (c3 + 2) % 3;
          a.list_zero1 = b->tcount.p + 3 + (c3 + 1) % 3;
          a.tiles_x = tx;
          a.tiles_y = ty;
          a.tiles_total = static_cast<int>(nt);
          tf_tiles[s] = -1;
          listed[s] = 1;
        } else if (tiled) {
          list_launch[s] = -1;
          const size_t n = static_cast<size_t>(tx) * ty * b->n_envs * 4;
          for (auto& f : b->tflags)
            if (f.n < n) {
              EBL_CUDA(f.alloc(n));
              tf_tiles[s] = -1;
            }
          a.tflag_in = tf_tiles[s] == tx * ty ? b->tflags[tf_par[s]].p : nullptr;
          a.tflag_out = b->tflags[tf_par[s] ^ 1].p;
          tf_par[s] ^= 1;
          tf_tiles[s] = tx * ty;
        } else {
          list_launch[s] = -1;
          tf_tiles[s] = -1;
        }
      }
      args[s] = a;
    }
    // the listed shards' first-launch counter resets are on their own streams: a neighbour's first
    // marks wait for them (slot 1 plays "chunk -1")
    if (chunk == 0 && !single)
      for (int s = 0; s < n_shards; ++s) {
        EBL_CUDA(set_dev(shards[s]->device));
        EBL_CUDA(cudaEventRecord(shards[s]->shard_ev[1], shards[s]->stream));
      }
    // one launch for the chunk: every shard on the same device and on its work list
    bool fused_launch = single && n_shards > 1 && use_warp(shards[0]);
    for (int s = 0; s < n_shards && fused_launch; ++s)
      fused_launch = listed[s] && args[s].list_mode == args[0].list_mode && use_warp(shards[s]) &&
                     shards[s]->mode == shards[0]->mode;
    ebl::ShardsLaunch multi{};
    multi.all_tiles = args[0].list_mode == 1;
    // pass 2: peer stores and marks, launch
    for (int s = 0; s < n_shards; ++s) {
      ebl_batch* b = shards[s];
      EBL_CUDA(set_dev(b->device));
      if (chunk == 0 && !single)
        for (int q = s - 1; q <= s + 1; q += 2)
          if (q >= 0 && q < n_shards) EBL_CUDA(cudaStreamWaitEvent(b->stream, shards[q]->shard_ev[1], 0));
      const ebl::BlockGeom& g = geo[s];
      ebl::StepArgs a = args[s];
      bool marked = listed[s] != 0;
      const int64_t g0 = b->row_off + b->band_lo, g1 = b->row_off + b->band_hi;
      for (int q = s - 1; q <= s + 1; q += 2) {
        if (q < 0 || q >= n_shards) continue;
        const ebl_batch* nb = shards[q];
        // shard q's halo tiles lose their exposure only when q marks ours and we mark q's
        if (!listed[q]) marked = false;
        const int64_t lo = std::max(g0, nb->row_off), hi = std::min(g1, nb->row_off + static_cast<int64_t>(nb->h));
        if (hi <= lo) continue;
        const int p = a.n_peers++;
        a.peer_out[p] = outs[q];
        a.peer_lo[p] = static_cast<int>(lo - b->row_off);
        a.peer_hi[p] = static_cast<int>(hi - b->row_off);
        a.peer_dst[p] = static_cast<int>(lo - nb->row_off);
        a.peer_queued[p] = nullptr;
        if (listed[s] && listed[q]) {  // our burning tiles enqueue q's tiles that read these rows
          const ebl::StepArgs& aq = args[q];
          a.peer_queued[p] = aq.queued;
          a.peer_next_list[p] = aq.next_list;
          a.peer_next_count[p] = aq.next_count;
          a.peer_stamp[p] = aq.list_stamp;
          a.peer_tiles_x[p] = aq.tiles_x;
          a.peer_tiles_y[p] = aq.tiles_y;
          a.peer_tile_h[p] = geo[q].tile_h;
          a.peer_tile_w[p] = geo[q].tile_w;
          a.peer_halo_r[p] = geo[q].halo_rows;
          a.peer_halo_c[p] = geo[q].halo_cols;
        }
      }
      a.halo_marked = marked && halo_marks ? 1 : 0;
      if (!halo_marks)
        for (int p = 0; p < a.n_peers; ++p) a.peer_queued[p] = nullptr;
      if (fused_launch) {
        multi.sa[s] = a;
        multi.g[s] = g;
        multi.n = s + 1;
        continue;
      }
      EBL_CUDA(launch_ca(b, a, g, strm(s)));
      if (list_launch[s] >= 0 && done + k == n_steps) {  // U/B/X of the band from the in-place records
        const int tx = (b->w + g.tile_w - 1) / g.tile_w, ty = (b->h + g.tile_h - 1) / g.tile_h;
        EBL_CUDA(ebl::launch_tile_counts(b->trec.p, b->n_envs, tx * ty, b->counts.p, strm(s)));
      }
      if (!single) EBL_CUDA(cudaEventRecord(b->shard_ev[chunk & 1], b->stream));
    }
    if (fused_launch) {
      EBL_CUDA(ebl::launch_step_warp_shards(multi, shards[0]->mode, S0));
      for (int s = 0; s < n_shards && done + k == n_steps; ++s) {
        const ebl_batch* b = shards[s];
        const ebl::BlockGeom& g = geo[s];
        const int tx = (b->w + g.tile_w - 1) / g.tile_w, ty = (b->h + g.tile_h - 1) / g.tile_h;
        EBL_CUDA(ebl::launch_tile_counts(b->trec.p, b->n_envs, tx * ty, b->counts.p, S0));
      }
    }
    for (int s = 0; s < n_shards; ++s) {
      ebl_batch* b = shards[s];
      b->cur ^= 1;
      b->step += k;
      b->launches += 1;
      b->steps_done += k;
      b->counts_valid = true;
    }
    done += k;
  }
  // the last launches' peer rows land before anything else on each shard's stream
  if (single) {
    EBL_CUDA(cudaEventRecord(shards[0]->shard_ev[0], S0));
    for (int s = 1; s < n_shards; ++s) EBL_CUDA(cudaStreamWaitEvent(shards[s]->stream, shards[0]->shard_ev[0], 0));
    return EBL_OK;
  }
  for (int s = 0; s < n_shards && chunk > 0; ++s) {
    EBL_CUDA(cudaSetDevice(shards[s]->device));
    for (int q = s - 1; q <= s + 1; q += 2)
      if (q >= 0 && q < n_shards)
        EBL_CUDA(cudaStreamWaitEvent(shards[s]->stream, shards[q]->shard_ev[(chunk - 1) & 1], 0));
  }
  return EBL_OK;
}

int ebl_batch_rows_device(ebl_batch* b, int row0, int n_rows, void* dptr, int to_batch) {
  EBL_DEVICE_GUARD(b);
  // reads, and writes of halo rows outside the shard's band, keep the tile activity records
  const bool halo_only = b && b->band_lo >= 0 && (row0 + n_rows <= b->band_lo || row0 >= b->band_hi);
  if (int e = check_sync(b, !to_batch || halo_only)) return e;
  if (n_rows < 0 || row0 < 0 || row0 + n_rows > b->h) return set_err(EBL_EINVAL, "rows: range outside the layer");
  EBL_CUDA(cudaSetDevice(b->device));
  const size_t bytes = static_cast<size_t>(n_rows) * b->w;
  for (int e = 0; e < b->n_envs; ++e) {
    uint8_t* layer = b->state[b->cur].p + e * b->ncell + static_cast<size_t>(row0) * b->w;
    uint8_t* ext = static_cast<uint8_t*>(dptr) + e * bytes;
    if (to_batch) EBL_CUDA(cudaMemcpyAsync(layer, ext, bytes, cudaMemcpyDeviceToDevice, b->stream));
    else EBL_CUDA(cudaMemcpyAsync(ext, layer, bytes, cudaMemcpyDeviceToDevice, b->stream));
  }
  if (to_batch && halo_only) EBL_CUDA(mark_halo_rows(b, row0, n_rows));
  if (to_batch) b->counts_valid = false;
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  return EBL_OK;
}

int ebl_batch_set_tiling(ebl_batch* b, int tile_h, int tile_w, int halo) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (tile_h == 0) {
    b->tile_h = 0;
    return EBL_OK;
  }
  if (tile_h < 1 || tile_w < 32 || (tile_w & 31) || halo < 0 || halo > 32 ||
      (halo == 0 && (tile_h < b->h || tile_w < b->w)))
    return set_err(EBL_EINVAL, "tiling: tile_w a positive multiple of 32, halo in [1,32] unless one tile");
  const int rh = std::min(b->h, tile_h + 2 * halo), rw = std::min(b->w, tile_w + (tile_w >= b->w ? 0 : 64));
  if (rh * rw > 65536 || ebl::blocked_smem_bytes(rh, rw, std::max(1, rh * rw / 4), 1) > ebl::kResMaxSmem)
    return set_err(EBL_EINVAL, "tiling: region exceeds shared memory");
  b->tile_h = tile_h;
  b->tile_w = tile_w;
  b->tile_halo = halo;
  return EBL_OK;
}

int ebl_batch_counts(ebl_batch* b, int32_t* out) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_sync(b, true)) return e;
  EBL_CUDA(cudaSetDevice(b->device));
  if (!b->counts_valid) {
    EBL_CUDA(cudaMemsetAsync(b->counts.p, 0, b->n_envs * 4 * sizeof(int32_t), b->stream));
    EBL_CUDA(ebl::launch_counts(b->state[b->cur].p, b->n_envs, static_cast<int>(b->ncell), b->counts.p, b->stream));
    b->counts_valid = true;
  }
  EBL_CUDA(cudaMemcpyAsync(out, b->counts.p, b->n_envs * 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  return EBL_OK;
}

int ebl_batch_intensity(ebl_batch* b, float* lambda, float* p) {
  return ebl_batch_intensity_form(b, 1, lambda, p);
}

int ebl_batch_intensity_form(ebl_batch* b, int record_form, float* lambda, float* p) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_sync(b)) return e;
  if (int e = prepare(b)) return e;
  const size_t total = b->ncell * b->n_envs;
  DevBuf<float> dl, dp;
  EBL_CUDA(dl.alloc(total));
  EBL_CUDA(dp.alloc(total));
  ebl::StepArgs a = step_args(b);
  a.rec_probe = record_form;
  EBL_CUDA(ebl::launch_intensity(a, b->mode, dl.p, dp.p, b->stream));
  EBL_CUDA(cudaMemcpyAsync(lambda, dl.p, total * sizeof(float), cudaMemcpyDeviceToHost, b->stream));
  EBL_CUDA(cudaMemcpyAsync(p, dp.p, total * sizeof(float), cudaMemcpyDeviceToHost, b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  return EBL_OK;
}

int ebl_batch_set_profiling(ebl_batch* b, int on) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  EBL_CUDA(cudaSetDevice(b->device));
  if (on && !ebl::phase_prof_built())
    return set_err(EBL_ESTATE, "library built without EBL_PHASE_PROF (scripts/build_variant.sh)");
  if (on) {
    EBL_CUDA(b->prof.alloc(static_cast<size_t>(b->n_envs) * 10));
    EBL_CUDA(cudaMemsetAsync(b->prof.p, 0, static_cast<size_t>(b->n_envs) * 10 * sizeof(long long), b->stream));
  }
  b->profiling = on != 0;
  return EBL_OK;
}

int ebl_batch_profile(ebl_batch* b, int64_t* out) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (!b->profiling) return set_err(EBL_ESTATE, "profiling is off (ebl_batch_set_profiling)");
  EBL_CUDA(cudaMemcpyAsync(out, b->prof.p, static_cast<size_t>(b->n_envs) * 10 * sizeof(long long),
                           cudaMemcpyDeviceToHost, b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  return EBL_OK;
}


int ebl_batch_diag(ebl_batch* b, uint64_t* out4, int reset) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b, true)) return e;
  unsigned long long d[2];
  EBL_CUDA(cudaMemcpyAsync(d, b->diag.p, sizeof d, cudaMemcpyDeviceToHost, b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  out4[0] = d[0];
  out4[1] = d[1];
  out4[2] = b->steps_done;
  out4[3] = b->launches;
  if (reset) {
    EBL_CUDA(cudaMemsetAsync(b->diag.p, 0, sizeof d, b->stream));
    b->steps_done = 0;
    b->launches = 0;
  }
  return EBL_OK;
}

int ebl_batch_tile_stats(ebl_batch* b, uint64_t* out2, int reset) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b, true)) return e;
  if (!out2) return set_err(EBL_EINVAL, "null out");
  unsigned long long d[2];
  EBL_CUDA(cudaMemcpyAsync(d, b->diag.p + 2, sizeof d, cudaMemcpyDeviceToHost, b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  out2[0] = d[0];
  out2[1] = d[1];
  if (reset) EBL_CUDA(cudaMemsetAsync(b->diag.p + 2, 0, sizeof d, b->stream));
  return EBL_OK;
}

// ---- snapshots (snapshot.hpp / snapshot.cpp) --------------------------------------------------
int ebl_batch_snapshot_text(ebl_batch* b, const void* layers_dev, int n_layers, const uint64_t* steps,
                            const int32_t* agents, char* out, size_t cap, size_t* len) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_sync(b)) return e;
  if (!len) return set_err(EBL_EINVAL, "ebl_batch_snapshot_text: len is NULL");
  const int n = layers_dev ? n_layers : b->n_envs;
  if (n < 0) return set_err(EBL_EINVAL, "ebl_batch_snapshot_text: negative layer count");
  // headers and agent lines formatted here (serialize_snapshot, snapshot.cpp:55-70), the bodies
  // rendered on the device
  std::string meta;
  std::vector<unsigned long long> off(4 * static_cast<size_t>(n));
  size_t total = 0;
  const size_t body = static_cast<size_t>(b->h) * (b->w + 1);
  for (int i = 0; i < n; ++i) {
    const std::string hdr = "emberline-snapshot v1 " + std::to_string(b->h) + " " + std::to_string(b->w) + " " +
                            std::to_string(steps ? steps[i] : b->step) + "\n";
    std::string ag;
    if (agents && agents[3 * i] >= 0)
      ag = "agent " + std::to_string(agents[3 * i]) + " " + std::to_string(agents[3 * i + 1]) + " " +
           std::to_string(agents[3 * i + 2]) + "\n";
    off[4 * i] = total;
    off[4 * i + 1] = meta.size();
    off[4 * i + 2] = hdr.size();
    off[4 * i + 3] = ag.size();
    meta += hdr;
    meta += ag;
    total += hdr.size() + body + ag.size();
  }
  *len = total;
  if (!out) return EBL_OK;  // size query
  if (cap < total) return set_err(EBL_ERANGE, "ebl_batch_snapshot_text: the text needs " + std::to_string(total) + " bytes");
  if (n == 0) return EBL_OK;
  EBL_CUDA(cudaSetDevice(b->device));
  if (b->snap_text.n < total) EBL_CUDA(b->snap_text.alloc(total));
  if (b->snap_meta.n < meta.size()) EBL_CUDA(b->snap_meta.alloc(meta.size()));
  if (b->snap_off.n < off.size()) EBL_CUDA(b->snap_off.alloc(off.size()));
  EBL_CUDA(cudaMemcpyAsync(b->snap_meta.p, meta.data(), meta.size(), cudaMemcpyHostToDevice, b->stream));
  EBL_CUDA(cudaMemcpyAsync(b->snap_off.p, off.data(), off.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice,
                           b->stream));
  const uint8_t* L = layers_dev ? static_cast<const uint8_t*>(layers_dev) : b->state[b->cur].p;
  EBL_CUDA(ebl::launch_snapshot_text(L, n, b->h, b->w, b->snap_meta.p, b->snap_off.p, b->snap_text.p, b->stream));
  EBL_CUDA(cudaMemcpyAsync(out, b->snap_text.p, total, cudaMemcpyDeviceToHost, b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  b->launches += 1;
  return EBL_OK;
}

}  // extern "C"

namespace {
// parse_snapshot's token rules (snapshot.cpp:34-53): whitespace split; integers by from_chars over
// the whole token
std::vector<std::string> snap_split_ws(const std::string& line) {
  std::vector<std::string> out;
  std::istringstream iss(line);
  std::string tok;
  while (iss >> tok) out.push_back(tok);
  return out;
}
template <class T>
bool snap_int(const std::string& tok, const char* what, T* v) {
  const char* e = tok.data() + tok.size();
  const auto r = std::from_chars(tok.data(), e, *v);
  if (r.ec != std::errc() || r.ptr != e) return set_err(EBL_EFILE, std::string("snapshot: invalid ") + what + " '" + tok + "'"), false;
  return true;
}
}  // namespace

extern "C" {

int ebl_snapshot_parse(const char* text, size_t text_len, int* h, int* w, uint64_t* step, uint8_t* layer,
                       size_t layer_cap, int32_t* agent3, int* has_agent) {
  if (!text || !h || !w || !step) return set_err(EBL_EINVAL, "ebl_snapshot_parse: null argument");
  // parse_snapshot (snapshot.cpp:74-121), line by line as std::getline
  size_t pos = 0;
  auto getline = [&](std::string& line) -> bool {
    if (pos >= text_len) return false;
    const void* nl = std::memchr(text + pos, '\n', text_len - pos);
    const size_t end = nl ? static_cast<size_t>(static_cast<const char*>(nl) - text) : text_len;
    line.assign(text + pos, end - pos);
    pos = nl ? end + 1 : text_len;
    return true;
  };
  std::string line;
  if (!getline(line)) return set_err(EBL_EFILE, "snapshot: empty input");
  const auto header = snap_split_ws(line);
  if (header.size() != 5 || header[0] != "emberline-snapshot" || header[1] != "v1")
    return set_err(EBL_EFILE, "snapshot: bad header '" + line + "'");
  int hh = 0, ww = 0;
  uint64_t st = 0;
  if (!snap_int(header[2], "height", &hh) || !snap_int(header[3], "width", &ww)) return EBL_EFILE;
  if (hh < 1 || ww < 1) return set_err(EBL_EFILE, "snapshot: dimensions must be positive");
  if (!snap_int(header[4], "step", &st)) return EBL_EFILE;
  const size_t need = static_cast<size_t>(hh) * ww;
  if (layer && layer_cap < need)
    return set_err(EBL_ERANGE, "ebl_snapshot_parse: the layer needs " + std::to_string(need) + " bytes");
  for (int row = hh - 1; row >= 0; --row) {
    if (!getline(line))
      return set_err(EBL_EFILE, "snapshot: expected " + std::to_string(hh) + " rows, input ended early");
    while (!line.empty() && (line.back() == '\r' || line.back() == ' ')) line.pop_back();
    if (static_cast<int>(line.size()) != ww)
      return set_err(EBL_EFILE, "snapshot: row has " + std::to_string(line.size()) + " cells, expected " +
                                    std::to_string(ww));
    for (int col = 0; col < ww; ++col) {
      const char c = line[col];
      const int v = c == 'U' ? 0 : c == 'B' ? 1 : c == 'X' ? 2 : -1;
      if (v < 0) return set_err(EBL_EFILE, std::string("snapshot: invalid fire-state character '") + c + "'");
      if (layer) layer[static_cast<size_t>(row) * ww + col] = static_cast<uint8_t>(v);
    }
  }
  bool agent = false;
  int32_t ar = 0, ac = 0, aw = 0;
  while (getline(line)) {
    const auto toks = snap_split_ws(line);
    if (toks.empty()) continue;
    if (toks[0] == "agent" && toks.size() == 4 && !agent) {
      if (!snap_int(toks[1], "agent row", &ar) || !snap_int(toks[2], "agent col", &ac) ||
          !snap_int(toks[3], "agent water", &aw))
        return EBL_EFILE;
      if (ar < 0 || ar >= hh || ac < 0 || ac >= ww) return set_err(EBL_EFILE, "snapshot: agent position out of bounds");
      if (aw < 0) return set_err(EBL_EFILE, "snapshot: negative agent water");
      agent = true;
      continue;
    }
    return set_err(EBL_EFILE, "snapshot: unexpected trailing line '" + line + "'");
  }
  *h = hh;
  *w = ww;
  *step = st;
  if (has_agent) *has_agent = agent ? 1 : 0;
  if (agent3 && agent) {
    agent3[0] = ar;
    agent3[1] = ac;
    agent3[2] = aw;
  }
  return EBL_OK;
}

// Host staging buffers for the host-buffer entry points: anonymous memory in 2 MiB transparent
// huge pages, faulted in, then page-locked and mapped (cudaHostRegister).  Huge pages make the
// DMA path robust: on the measured VM some 4 KiB-page pinned buffers copy at 14 GB/s instead of
// 54 GB/s; mapped, so ebl_batch_run writes results into them straight from the kernel.
namespace {
std::mutex g_host_mu;
std::unordered_map<void*, std::pair<void*, size_t>> g_host;  // user ptr -> (mapping, length)
}  // namespace

int ebl_host_alloc(size_t bytes, void** out) {
  if (!out || bytes == 0) return set_err(EBL_EINVAL, "ebl_host_alloc: bytes > 0 and an out pointer");
  constexpr size_t kHuge = size_t{2} << 20;
  const size_t len = (bytes + kHuge - 1) / kHuge * kHuge;
  void* base = mmap(nullptr, len + kHuge, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (base == MAP_FAILED) return set_err(EBL_ECUDA, "ebl_host_alloc: mmap failed");
  char* p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(base) + kHuge - 1) & ~(kHuge - 1));
  madvise(p, len, MADV_HUGEPAGE);  // a hint: 4 KiB pages when THP is off
  std::memset(p, 0, len);          // fault the pages in before they are pinned
  const cudaError_t e = cudaHostRegister(p, len, cudaHostRegisterPortable | cudaHostRegisterMapped);
  if (e != cudaSuccess) {
    munmap(base, len + kHuge);
    return set_err(EBL_ECUDA, std::string("ebl_host_alloc: ") + cudaGetErrorString(e));
  }
  {
    std::lock_guard<std::mutex> lk(g_host_mu);
    g_host[p] = {base, len + kHuge};
  }
  *out = p;
  return EBL_OK;
}

int ebl_host_free(void* p) {
  if (!p) return EBL_OK;
  std::pair<void*, size_t> m;
  {
    std::lock_guard<std::mutex> lk(g_host_mu);
    auto it = g_host.find(p);
    if (it == g_host.end()) return set_err(EBL_EINVAL, "ebl_host_free: not an ebl_host_alloc pointer");
    m = it->second;
    g_host.erase(it);
  }
  const cudaError_t e = cudaHostUnregister(p);
  munmap(m.first, m.second);
  if (e != cudaSuccess) return set_err(EBL_ECUDA, std::string("ebl_host_free: ") + cudaGetErrorString(e));
  return EBL_OK;
}

int ebl_device_rng_words(int n, const uint64_t* keys5, uint64_t* out) {
  if (n < 0 || (n > 0 && (!keys5 || !out))) return set_err(EBL_EINVAL, "bad arguments");
  if (n == 0) return EBL_OK;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return set_err(EBL_ECUDA, "no CUDA device available (the engine has no CPU path)");
  DeviceGuard guard(0);
  DevBuf<uint64_t> dk, dout;
  EBL_CUDA(dk.alloc(5 * static_cast<size_t>(n)));
  EBL_CUDA(dout.alloc(n));
  EBL_CUDA(cudaMemcpy(dk.p, keys5, 5 * sizeof(uint64_t) * n, cudaMemcpyHostToDevice));
  EBL_CUDA(ebl::launch_rng_probe(n, dk.p, dout.p, nullptr));
  EBL_CUDA(cudaMemcpy(out, dout.p, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost));
  return EBL_OK;
}

int ebl_batch_sync(ebl_batch* b) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b, true)) return e;
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  return EBL_OK;
}

// ---- one-shot reference signatures --------------------------------------------------
int ebl_run_stochastic(int h, int w, const uint8_t* initial, const double* speed, const double* dir,
                       const double* veg, const double* den, const double* slope8,
                       const ebl_sim_config* cfg, uint64_t seed, uint64_t step, uint64_t stream,
                       int steps, uint8_t* out) {
  if (steps < 0) return set_err(EBL_EINVAL, "steps must be >= 0");
  ebl_batch* b = nullptr;
  int rc = ebl_batch_create(&b, 0, 1, h, w, nullptr);
  if (rc) return rc;
  std::unique_ptr<ebl_batch, void (*)(ebl_batch*)> guard(b, ebl_batch_destroy);
  if ((rc = ebl_batch_set_config(b, cfg))) return rc;
  if ((rc = ebl_batch_set_grid(b, 1, speed, dir, veg, den, slope8))) return rc;
  if ((rc = ebl_batch_set_state(b, initial))) return rc;
  if ((rc = ebl_batch_set_key(b, seed, step, &stream, 0))) return rc;
  if ((rc = ebl_step_batch(b, steps))) return rc;
  return ebl_batch_get_state(b, out);
}

int ebl_step_stochastic(int h, int w, const uint8_t* fire, const double* speed, const double* dir,
                        const double* veg, const double* den, const double* slope8,
                        const ebl_sim_config* cfg, uint64_t seed, uint64_t step, uint64_t stream,
                        uint8_t* out) {
  return ebl_run_stochastic(h, w, fire, speed, dir, veg, den, slope8, cfg, seed, step, stream, 1, out);
}

// ---- RL ------------------------------------------------------------------------------
void ebl_env_default_preset(ebl_env_config* c) {  // rl_env.cpp:10-27
  *c = ebl_env_config{20, 20, 2, 30, 0.05, 120, 1, 1, 1.0, 0.0, 0.0, 0.0,
                      ebl_sim_config{0.06, 0.1, 0.2, 0.5, 1.0, 0.9, 200}};
}

void ebl_env_smoke10_preset(ebl_env_config* c) {  // rl_env.cpp:29-57
  *c = ebl_env_config{10, 10, 2, 60, 0.05, 100, 3, 0, 0.5, 0.0, 0.0, 0.0,
                      ebl_sim_config{0.03, 0.1, 0.2, 0.5, 1.0, 0.985, 200}};
}

int ebl_env_observation_size(const ebl_env_config* c) {
  const int side = 2 * c->window_radius + 1;
  return 3 * side * side + 3;
}

namespace {
int validate_env(const ebl_env_config* c) {  // rl_env.cpp:80-93
  if (c->height < 1 || c->width < 1) return set_err(EBL_EINVAL, "EnvConfig: dimensions must be at least 1x1");
  if (c->window_radius < 0) return set_err(EBL_EINVAL, "EnvConfig: negative window radius");
  if (c->water_capacity < 1) return set_err(EBL_EINVAL, "EnvConfig: water capacity must be >= 1");
  if (!(c->burn_penalty > 0.0)) return set_err(EBL_EINVAL, "EnvConfig: burn penalty must be > 0");
  if (c->max_episode_steps < 1) return set_err(EBL_EINVAL, "EnvConfig: max episode steps must be >= 1");
  if (c->ignition_count < 0 || c->ignition_count > c->height * c->width)
    return set_err(EBL_EINVAL, "EnvConfig: ignition count outside [0, cells]");
  return EBL_OK;
}

// Tanker step/rollout: the bit-plane kernel, or the byte kernel when EBL_KERNEL_TILED is
// selected (an independent implementation kept for cross-checking).
int tanker_launch(ebl_batch* b, ebl::RlArgs g) {
  if (b->kernel != EBL_KERNEL_TILED && ebl::rl_bits_fits(b->h, b->w) && b->kernel != EBL_KERNEL_RESIDENT &&
      ebl::rl_warp_smem_bytes(b->h, b->w) <= ebl::kResMaxSmem) {
    // the warp-local kernel (two barriers per step); its state stays bit-resident between launches
    const size_t words = static_cast<size_t>(b->n_envs) * 3 * b->h * ((b->w + 31) / 32);
    EBL_CUDA(b->rl_bits.alloc(words));
    g.bits = b->rl_bits.p;
    g.bits_in = b->rl_bits_valid ? 1 : 0;
    EBL_CUDA(ebl::launch_rl_tanker_warp(g, b->mode, b->stream));
    b->rl_bits_valid = b->rl_bits_truth = true;
    return EBL_OK;
  }
  if (int e = rl_sync_bytes(b)) return e;
  if (b->kernel != EBL_KERNEL_TILED && ebl::rl_bits_fits(b->h, b->w))
    EBL_CUDA(ebl::launch_rl_tanker_bits(g, b->mode, b->stream));  // pooled-list kernel (RESIDENT)
  else
    EBL_CUDA(ebl::launch_rl_tanker(g, b->mode, b->stream));
  return EBL_OK;
}

ebl::RlArgs rl_args(ebl_batch* b) {
  ebl::RlArgs g{};
  g.s = step_args(b);
  g.env = b->rl_env.p;
  g.state = b->state[b->cur].p;
  g.wet = b->wet.p;
  g.error = b->error.p;
  g.water_capacity = b->env_cfg.water_capacity;
  g.max_episode_steps = b->env_cfg.max_episode_steps;
  g.waste_water = b->env_cfg.waste_water;
  g.burn_penalty = b->env_cfg.burn_penalty;
  g.ignitions = b->tanker_ignitions;
  g.max_steps = b->tanker_max_steps;
  g.env_id0 = b->env_id0;
  g.seed = b->rl_seed;
  g.n_steps = 1;
  return g;
}
}  // namespace

int ebl_rl_configure(ebl_batch* b, int variant, const ebl_env_config* c, int tanker_ignitions,
                     int tanker_max_steps, uint32_t env_id0) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_sync(b)) return e;
  if (variant != EBL_RL_REFERENCE && variant != EBL_RL_TANKER) return set_err(EBL_EINVAL, "unknown RL variant");
  if (b->ncell > static_cast<size_t>(ebl::kRlMaxCells))
    return set_err(EBL_EINVAL, "RL envs must have at most 16384 cells (layer resident in shared memory)");
  EBL_CUDA(cudaSetDevice(b->device));
  if (variant == EBL_RL_REFERENCE) {
    if (!c) return set_err(EBL_EINVAL, "null env config");
    if (int e = validate_env(c)) return e;
    if (c->height != b->h || c->width != b->w) return set_err(EBL_EINVAL, "EnvConfig dims differ from the batch");
    b->env_cfg = *c;
    // flat terrain of the config (rl_env.cpp:99-105): one fuel class, zero elevation
    const uint8_t zero = 0;
    std::vector<uint8_t> cls(b->ncell, zero);
    std::vector<float> el(b->ncell, 0.f);
    const double veg = c->fuel_veg, den = c->fuel_den;
    if (int e = ebl_batch_set_terrain(b, 1, cls.data(), el.data(), 1, &veg, &den, 30.0)) return e;
    if (int e = ebl_batch_set_wind(b, 1, &c->wind_speed, &c->wind_direction)) return e;
    if (int e = ebl_batch_set_config(b, &c->spread)) return e;
  } else {
    if (b->mode == ebl::kStaticNone) return set_err(EBL_ESTATE, "tanker RL needs terrain set first");
    if (tanker_max_steps < 1 || tanker_ignitions < 0) return set_err(EBL_EINVAL, "bad tanker config");
    b->tanker_ignitions = tanker_ignitions;
    b->tanker_max_steps = tanker_max_steps;
    b->env_id0 = env_id0;
  }
  b->rl_variant = variant;
  const size_t n = b->n_envs;
  EBL_CUDA(b->rl_env.alloc(n));
  EBL_CUDA(b->wet.alloc(n * b->ncell));
  EBL_CUDA(cudaMemsetAsync(b->wet.p, 0, n * b->ncell, b->stream));
  EBL_CUDA(b->done.alloc(n));
  EBL_CUDA(b->reward.alloc(n));
  EBL_CUDA(b->reward_sum.alloc(n));
  EBL_CUDA(b->episodes.alloc(n));
  EBL_CUDA(b->actions.alloc(n));
  EBL_CUDA(b->mask.alloc(n));
  EBL_CUDA(b->error.alloc(1));
  EBL_CUDA(cudaMemsetAsync(b->error.p, 0, sizeof(int32_t), b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  return EBL_OK;
}

int ebl_rl_reset(ebl_batch* b, uint64_t seed, const uint64_t* streams, const uint8_t* mask) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_sync(b)) return e;
  if (b->rl_variant < 0) return set_err(EBL_ESTATE, "ebl_rl_configure first");
  if (int e = prepare(b)) return e;
  EBL_CUDA(cudaSetDevice(b->device));
  if (b->rl_variant == EBL_RL_REFERENCE) {
    // FireSuppressionEnv::reset is a short serial draw loop per env (rl_env.cpp:125-145);
    // it runs on the host and uploads the layers (once per episode, off the step path).
    const ebl_env_config& c = b->env_cfg;
    const uint64_t n = b->ncell;
    std::vector<uint8_t> st(n * b->n_envs);
    std::vector<ebl::RlEnv> ev(b->n_envs);
    EBL_CUDA(cudaMemcpyAsync(st.data(), b->state[b->cur].p, st.size(), cudaMemcpyDeviceToHost, b->stream));
    EBL_CUDA(cudaMemcpyAsync(ev.data(), b->rl_env.p, ev.size() * sizeof(ebl::RlEnv), cudaMemcpyDeviceToHost, b->stream));
    EBL_CUDA(cudaStreamSynchronize(b->stream));
    for (int e = 0; e < b->n_envs; ++e) {
      if (mask && !mask[e]) continue;
      const uint64_t stream = streams ? streams[e] : b->env_id0 + static_cast<uint64_t>(e);
      uint8_t* f = st.data() + e * n;
      std::memset(f, 0, n);
      uint64_t counter = 0;
      int burning = 0;
      for (int placed = 0; placed < c.ignition_count;) {
        const uint64_t cell = ebl::rng_below(seed, 0, stream, counter++, 1, n);
        if (f[cell] == 1) continue;
        f[cell] = 1;
        ++placed;
        ++burning;
      }
      const uint64_t a = ebl::rng_below(seed, 0, stream, counter++, 1, n);
      ebl::RlEnv& r = ev[e];
      r.row = static_cast<int32_t>(a / static_cast<uint64_t>(c.width));
      r.col = static_cast<int32_t>(a % static_cast<uint64_t>(c.width));
      r.water = c.water_capacity;
      r.step = 0;
      r.seed = seed;
      r.stream = stream;
      r.done = burning == 0;
      r.episode = 0;
    }
    EBL_CUDA(cudaMemcpyAsync(b->state[b->cur].p, st.data(), st.size(), cudaMemcpyHostToDevice, b->stream));
    EBL_CUDA(cudaMemcpyAsync(b->rl_env.p, ev.data(), ev.size() * sizeof(ebl::RlEnv), cudaMemcpyHostToDevice, b->stream));
    EBL_CUDA(cudaStreamSynchronize(b->stream));
  } else {
    b->rl_seed = seed;
    const uint8_t* dmask = nullptr;
    if (mask) {
      EBL_CUDA(cudaMemcpyAsync(b->mask.p, mask, b->n_envs, cudaMemcpyHostToDevice, b->stream));
      dmask = b->mask.p;
    }
    ebl::RlArgs g = rl_args(b);
    EBL_CUDA(ebl::launch_rl_tanker_reset(g, b->mode, dmask, b->stream));
    b->launches += 1;
  }
  b->counts_valid = false;
  return EBL_OK;
}

// The device address of a mapped pinned host buffer (ebl_host_alloc, cudaHostAlloc(Mapped)), or
// null for any other pointer.
void* mapped_device_ptr(const void* p, size_t align) {
  cudaPointerAttributes pa{};
  void* d = nullptr;
  if (p && cudaPointerGetAttributes(&pa, p) == cudaSuccess && pa.type == cudaMemoryTypeHost && pa.devicePointer &&
      (reinterpret_cast<uintptr_t>(pa.devicePointer) % align) == 0)
    d = pa.devicePointer;
  cudaGetLastError();
  return d;
}

int ebl_rl_step(ebl_batch* b, const int32_t* actions, double* reward, uint8_t* done, int device_io) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (b->rl_variant < 0) return set_err(EBL_ESTATE, "ebl_rl_configure first");
  if (int e = prepare(b)) return e;
  EBL_CUDA(cudaSetDevice(b->device));
  ebl::RlArgs g = rl_args(b);
  // tanker steps with host buffers in mapped pinned memory: the kernel reads the actions and writes
  // reward / done through the mapping (no copy launches around the step; EBL_RL_ZC=0 copies)
  static const int rl_zc = [] {  // 0: copies, 1: outputs and actions mapped, 2: outputs only
    const char* e = std::getenv("EBL_RL_ZC");
    return e ? std::atoi(e) : 2;
  }();
  const bool zc = rl_zc && !device_io && b->rl_variant != EBL_RL_REFERENCE;
  double* const zc_reward = zc && reward ? static_cast<double*>(mapped_device_ptr(reward, 8)) : nullptr;
  uint8_t* const zc_done = zc && done ? static_cast<uint8_t*>(mapped_device_ptr(done, 1)) : nullptr;
  if (actions) {
    const int32_t* zc_act = zc && rl_zc == 1 ? static_cast<const int32_t*>(mapped_device_ptr(actions, 4)) : nullptr;
    if (device_io) {
      g.actions = actions;
    } else if (zc_act) {
      g.actions = zc_act;
    } else {
      if (b->rl_variant == EBL_RL_REFERENCE)
        for (int e = 0; e < b->n_envs; ++e)
          if (actions[e] < 0 || actions[e] >= 10)
            return set_err(EBL_ERANGE, "action_from_index: index " + std::to_string(actions[e]) + " outside [0, 10)");
      EBL_CUDA(cudaMemcpyAsync(b->actions.p, actions, b->n_envs * sizeof(int32_t), cudaMemcpyHostToDevice, b->stream));
      g.actions = b->actions.p;
    }
  }
  g.reward = device_io && reward ? reward : zc_reward ? zc_reward : b->reward.p;
  g.done = device_io && done ? done : zc_done ? zc_done : b->done.p;
  if (b->rl_variant == EBL_RL_REFERENCE) {
    if (int e = rl_sync_bytes(b)) return e;
    EBL_CUDA(ebl::launch_rl_ref_step(g, b->mode, b->stream));
  } else {
    if (int e = tanker_launch(b, g)) return e;
  }
  b->launches += 1;
  b->steps_done += 1;
  b->counts_valid = false;
  if (!device_io) {
    if (reward && !zc_reward)
      EBL_CUDA(cudaMemcpyAsync(reward, b->reward.p, b->n_envs * sizeof(double), cudaMemcpyDeviceToHost, b->stream));
    if (done && !zc_done) EBL_CUDA(cudaMemcpyAsync(done, b->done.p, b->n_envs, cudaMemcpyDeviceToHost, b->stream));
  }
  if (b->rl_variant == EBL_RL_REFERENCE) {
    int32_t err = 0;
    EBL_CUDA(cudaMemcpyAsync(&err, b->error.p, sizeof err, cudaMemcpyDeviceToHost, b->stream));
    EBL_CUDA(cudaStreamSynchronize(b->stream));
    if (err) {
      EBL_CUDA(cudaMemsetAsync(b->error.p, 0, sizeof(int32_t), b->stream));
      return set_err(EBL_ELOGIC, "FireSuppressionEnv::step: episode already finished");
    }
  } else if (!device_io && (reward || done || (actions && g.actions != b->actions.p))) {
    // (host results, or host actions the kernel reads through the mapping: done before returning)
    EBL_CUDA(cudaStreamSynchronize(b->stream));
  }
  return EBL_OK;
}

int ebl_rl_rollout(ebl_batch* b, int n_steps, double* reward_sum, int32_t* episodes) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (b->rl_variant != EBL_RL_TANKER) return set_err(EBL_ESTATE, "rollout needs the tanker variant");
  if (n_steps < 1) return set_err(EBL_EINVAL, "n_steps must be >= 1");
  if (int e = prepare(b)) return e;
  EBL_CUDA(cudaSetDevice(b->device));
  EBL_CUDA(cudaMemsetAsync(b->reward_sum.p, 0, b->n_envs * sizeof(double), b->stream));
  EBL_CUDA(cudaMemsetAsync(b->episodes.p, 0, b->n_envs * sizeof(int32_t), b->stream));
  ebl::RlArgs g = rl_args(b);
  g.n_steps = n_steps;
  g.reward_sum = b->reward_sum.p;
  g.episodes = b->episodes.p;
  if (int e = tanker_launch(b, g)) return e;
  b->launches += 1;
  b->steps_done += n_steps;
  b->counts_valid = false;
  if (reward_sum) EBL_CUDA(cudaMemcpyAsync(reward_sum, b->reward_sum.p, b->n_envs * sizeof(double), cudaMemcpyDeviceToHost, b->stream));
  if (episodes) EBL_CUDA(cudaMemcpyAsync(episodes, b->episodes.p, b->n_envs * sizeof(int32_t), cudaMemcpyDeviceToHost, b->stream));
  if (reward_sum || episodes) EBL_CUDA(cudaStreamSynchronize(b->stream));
  return EBL_OK;
}

int ebl_rl_observe(ebl_batch* b, double* obs) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_sync(b)) return e;
  if (b->rl_variant != EBL_RL_REFERENCE) return set_err(EBL_ESTATE, "observe needs the reference variant");
  const int osz = ebl_env_observation_size(&b->env_cfg);
  const size_t total = static_cast<size_t>(b->n_envs) * osz;
  EBL_CUDA(b->obs.alloc(total));
  EBL_CUDA(ebl::launch_rl_observe(b->state[b->cur].p, b->rl_env.p, b->n_envs, b->h, b->w,
                                  b->env_cfg.window_radius, b->env_cfg.water_capacity, b->obs.p, b->stream));
  EBL_CUDA(cudaMemcpyAsync(obs, b->obs.p, total * sizeof(double), cudaMemcpyDeviceToHost, b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  return EBL_OK;
}

int ebl_rl_get_env_states(ebl_batch* b, ebl_env_state* out) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (b->rl_variant < 0) return set_err(EBL_ESTATE, "ebl_rl_configure first");
  std::vector<ebl::RlEnv> ev(b->n_envs);
  EBL_CUDA(cudaMemcpyAsync(ev.data(), b->rl_env.p, ev.size() * sizeof(ebl::RlEnv), cudaMemcpyDeviceToHost, b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  for (int e = 0; e < b->n_envs; ++e) {
    const ebl::RlEnv& r = ev[e];
    out[e] = ebl_env_state{r.row, r.col, r.water, r.step, r.seed, r.stream, r.done,
                           r.episode};
  }
  return EBL_OK;
}

int ebl_rl_set_env_states(ebl_batch* b, const ebl_env_state* in) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (b->rl_variant < 0) return set_err(EBL_ESTATE, "ebl_rl_configure first");
  std::vector<ebl::RlEnv> ev(b->n_envs);
  for (int e = 0; e < b->n_envs; ++e) {
    const ebl_env_state& s = in[e];
    ev[e] = ebl::RlEnv{s.agent_row, s.agent_col, s.water, s.step, s.seed, s.stream, s.done,
                       s.episode};
  }
  EBL_CUDA(cudaMemcpyAsync(b->rl_env.p, ev.data(), ev.size() * sizeof(ebl::RlEnv), cudaMemcpyHostToDevice, b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  return EBL_OK;
}

int ebl_rl_observe_device(ebl_batch* b, void* out_dev) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b, true)) return e;  // read-only: the bit-resident state stays valid
  if (b->rl_variant != EBL_RL_TANKER) return set_err(EBL_ESTATE, "observe_device needs the tanker variant");
  if (!out_dev) return set_err(EBL_EINVAL, "null out");
  EBL_CUDA(ebl::launch_rl_observe_planes(b->rl_bits_truth ? b->rl_bits.p : nullptr, b->state[b->cur].p, b->wet.p,
                                         static_cast<uint8_t*>(out_dev), b->n_envs, b->h, b->w, b->stream));
  b->launches += 1;
  return EBL_OK;
}

int ebl_rl_get_wet(ebl_batch* b, uint8_t* wet) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_sync(b)) return e;
  if (b->rl_variant < 0) return set_err(EBL_ESTATE, "ebl_rl_configure first");
  EBL_CUDA(cudaMemcpyAsync(wet, b->wet.p, b->ncell * b->n_envs, cudaMemcpyDeviceToHost, b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  return EBL_OK;
}

// ---- deterministic mode (engine.hpp:147-245) and its adjoint (C4) ---------------------------
#ifndef EBL_DET_FUSED  // one fused backward kernel per step (0: back1 + back2)
#define EBL_DET_FUSED 1
#endif
namespace {
int det_alloc(ebl_batch* b) {
  const size_t n = b->ncell * b->n_envs;
  for (auto& d : b->det) EBL_CUDA(d.alloc(n));
  return EBL_OK;
}

ebl::DetArgs det_args(ebl_batch* b) {
  ebl::DetArgs d{};
  d.s = step_args(b);
  const int c = b->det_cur * 3, o = (b->det_cur ^ 1) * 3;
  d.un = b->det[c].p;
  d.burn = b->det[c + 1].p;
  d.bd = b->det[c + 2].p;
  d.un_o = b->det[o].p;
  d.burn_o = b->det[o + 1].p;
  d.bd_o = b->det[o + 2].p;
  d.pot = b->det_pot.p;
  d.potT = b->det_potT.p;
  d.gam = b->det_gam.p;
  d.tab_stride = b->det_tables > 1 ? b->ncell : 0;
  d.pc = b->cfg.p_continue;
  d.V = b->det_V.p;
  d.align = b->det_align.p;
  d.wind_stride = b->n_winds > 1 ? 1 : 0;
  if (b->det_fac.p) {  // general form
    const size_t nt = b->ncell * b->det_tables;
    d.fac_F = b->det_fac.p;
    d.fac_pb = d.fac_F + nt;
    d.fac_V = d.fac_pb + nt * 8;
    d.fac_Va = d.fac_V + nt;
    d.fac_S = d.fac_Va + nt * 8;
  }
  return d;
}

// SpreadTables<double> for the deterministic mode, built on the host in the reference's
// arithmetic (ember_host.cpp) and uploaded; one table per env when grids or winds differ.
int det_tables(ebl_batch* b) {
  const ebl::Cfg6 c = cfg6(b->cfg);
  const bool general = b->mode == ebl::kStaticTables;
  const int T = general ? b->n_grids : ((b->n_grids > 1 || b->n_winds > 1) ? b->n_envs : 1);
  const size_t n = b->ncell;
  const bool dev_built = !general && b->det_dev_tables && std::abs(cfg6(b->cfg).alpha_s) < 325.0;
  std::vector<double> pot(dev_built ? 0 : n * 8 * T), gam(dev_built ? 0 : n * T);
  if (general) {  // per-cell layers: the SpreadTables plus the adjoint's derivative factors
    const size_t nt = n * T;
    ebl::build_tables(nt, b->g_speed.data(), b->g_dir.data(), b->g_veg.data(), b->g_den.data(),
                      b->g_slope.data(), c, pot.data(), gam.data());
    std::vector<double> fac(nt * 26);  // F | pb[8] | V | Va[8] | S[8]
    double* F = fac.data();
    double* pb = F + nt;
    double* V = pb + nt * 8;
    double* Va = V + nt;
    double* S = Va + nt * 8;
    ebl::build_det_factors(nt, b->g_speed.data(), b->g_dir.data(), b->g_veg.data(), b->g_den.data(),
                           b->g_slope.data(), c, F, pb, V, Va, S);
    EBL_CUDA(b->det_fac.alloc(fac.size()));
    EBL_CUDA(cudaMemcpyAsync(b->det_fac.p, fac.data(), fac.size() * sizeof(double), cudaMemcpyHostToDevice, b->stream));
  } else {
    if (b->h_terrain_stale) {  // terrain built on the device: fetch the host copy once
      const size_t m = n * b->n_grids;
      b->h_fuel.resize(m);
      b->h_elev.resize(m);
      EBL_CUDA(cudaMemcpyAsync(b->h_fuel.data(), b->fuel.p, m, cudaMemcpyDeviceToHost, b->stream));
      EBL_CUDA(cudaMemcpyAsync(b->h_elev.data(), b->elev.p, m * sizeof(float), cudaMemcpyDeviceToHost, b->stream));
      EBL_CUDA(cudaStreamSynchronize(b->stream));
      b->h_terrain_stale = false;
    }
    b->det_fac.reset();
    // on the device: pot = (source kappa_wind) exp(alpha_s S) with the cached fp64 slopes and the
    // restated libm exp, bit-identical to the host build (ember_det.cu); exact for |alpha_s S| < 512,
    // i.e. |alpha_s| < 325 (|S| < pi/2), else the host build.  gamma comes from the palette.
    if (dev_built) {
      if (!b->det_S_valid) {
        std::vector<double> S(n * 8 * b->n_grids);
        ebl::build_terrain_slopes64(b->n_grids, b->h, b->w, b->h_elev.data(), n, b->cellsize, S.data());
        EBL_CUDA(b->det_S.alloc(S.size()));
        EBL_CUDA(cudaMemcpyAsync(b->det_S.p, S.data(), S.size() * sizeof(double), cudaMemcpyHostToDevice, b->stream));
        EBL_CUDA(cudaStreamSynchronize(b->stream));
        b->det_S_valid = true;
      }
      EBL_CUDA(b->det_pot.alloc(n * 8 * T));
      EBL_CUDA(ebl::launch_det_tables_terrain(b->det_S.p, b->fuel.p, b->pal64.p, b->kw64.p, c.alpha_s, T, n,
                                              b->n_grids > 1 ? n : 0, b->n_winds > 1 ? 1 : 0, b->det_pot.p,
                                              b->stream));
    } else {
      ebl::build_terrain_tables(T, b->h, b->w, b->h_fuel.data(), b->h_elev.data(), b->n_grids > 1 ? n : 0,
                                b->pal_veg.data(), b->pal_den.data(), b->cellsize, b->wind_speed.data(),
                                b->wind_dir.data(), b->n_winds > 1 ? 1 : 0, c, pot.data(), gam.data());
    }
  }
  std::vector<double> V(b->n_winds), al(static_cast<size_t>(b->n_winds) * 8);
  for (int w = 0; w < b->n_winds; ++w) {  // kernel.hpp:24: cos(phi_k - theta) - 1
    V[w] = b->wind_speed[w];
    const double dir = ebl::wrap_angle(b->wind_dir[w]);
    for (int k = 0; k < 8; ++k) al[w * 8 + k] = std::cos(ebl::offset_angle(k) - dir) - 1.0;
  }
  if (!dev_built) {
    EBL_CUDA(b->det_pot.alloc(pot.size()));
    EBL_CUDA(b->det_gam.alloc(gam.size()));
    EBL_CUDA(cudaMemcpyAsync(b->det_pot.p, pot.data(), pot.size() * sizeof(double), cudaMemcpyHostToDevice, b->stream));
    EBL_CUDA(cudaMemcpyAsync(b->det_gam.p, gam.data(), gam.size() * sizeof(double), cudaMemcpyHostToDevice, b->stream));
  }
  static const bool pot_t = [] {
    const char* e = std::getenv("EBL_DET_POTT");
    return !e || std::atoi(e) != 0;
  }();
  if (pot_t) {  // the forward's target-ordered table (a permutation of the same fp64 values)
    EBL_CUDA(b->det_potT.alloc(n * 8 * T));
    EBL_CUDA(ebl::launch_pot_target(b->det_pot.p, b->det_potT.p, T, b->h, b->w, b->stream));
  } else {
    b->det_potT.reset();
  }
  EBL_CUDA(b->det_V.alloc(V.size()));
  EBL_CUDA(b->det_align.alloc(al.size()));
  EBL_CUDA(cudaMemcpyAsync(b->det_V.p, V.data(), V.size() * sizeof(double), cudaMemcpyHostToDevice, b->stream));
  EBL_CUDA(cudaMemcpyAsync(b->det_align.p, al.data(), al.size() * sizeof(double), cudaMemcpyHostToDevice, b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  b->det_tables = T;
  std::memcpy(&b->det_cfg, &b->cfg, sizeof b->cfg);
  b->det_tables_valid = true;
  return EBL_OK;
}
}  // namespace

int ebl_det_set_state(ebl_batch* b, const double* un, const double* burn, const double* bd) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (!un || !burn || !bd) return set_err(EBL_EINVAL, "null plane");
  EBL_CUDA(cudaSetDevice(b->device));
  if (int e = det_alloc(b)) return e;
  const size_t bytes = b->ncell * b->n_envs * sizeof(double);
  const int c = b->det_cur * 3;
  EBL_CUDA(cudaMemcpyAsync(b->det[c].p, un, bytes, cudaMemcpyHostToDevice, b->stream));
  EBL_CUDA(cudaMemcpyAsync(b->det[c + 1].p, burn, bytes, cudaMemcpyHostToDevice, b->stream));
  EBL_CUDA(cudaMemcpyAsync(b->det[c + 2].p, bd, bytes, cudaMemcpyHostToDevice, b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  b->det_ready = true;
  b->traj_steps = -1;
  return EBL_OK;
}

int ebl_det_set_state_from_fire(ebl_batch* b) {  // state_from_fire (engine.cpp:42-52)
  EBL_DEVICE_GUARD(b);
  if (int e = check_sync(b)) return e;
  EBL_CUDA(cudaSetDevice(b->device));
  if (int e = det_alloc(b)) return e;
  const int c = b->det_cur * 3;
  EBL_CUDA(ebl::launch_det_from_fire(b->state[b->cur].p, b->det[c].p, b->det[c + 1].p, b->det[c + 2].p,
                                     b->ncell * b->n_envs, b->stream));
  b->det_ready = true;
  b->traj_steps = -1;
  return EBL_OK;
}

int ebl_det_get_state(ebl_batch* b, double* un, double* burn, double* bd) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (!b->det_ready) return set_err(EBL_ESTATE, "ebl_det_set_state first");
  const size_t bytes = b->ncell * b->n_envs * sizeof(double);
  const int c = b->det_cur * 3;
  if (un) EBL_CUDA(cudaMemcpyAsync(un, b->det[c].p, bytes, cudaMemcpyDeviceToHost, b->stream));
  if (burn) EBL_CUDA(cudaMemcpyAsync(burn, b->det[c + 1].p, bytes, cudaMemcpyDeviceToHost, b->stream));
  if (bd) EBL_CUDA(cudaMemcpyAsync(bd, b->det[c + 2].p, bytes, cudaMemcpyDeviceToHost, b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  return EBL_OK;
}

int ebl_batch_set_det_tables(ebl_batch* b, int on_device) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  b->det_dev_tables = on_device != 0;
  b->det_tables_valid = false;
  return EBL_OK;
}

// EBL_DET_BD_DEFERRED=0: the recorded forward steps p_bd every step as the unrecorded one does
static bool det_bd_deferred() {
  static const bool on = [] {
    const char* e = std::getenv("EBL_DET_BD_DEFERRED");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

int ebl_det_forward(ebl_batch* b, int n_steps, int record) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (!b->det_ready) return set_err(EBL_ESTATE, "ebl_det_set_state first");
  if (b->mode == ebl::kStaticNone) return set_err(EBL_ESTATE, "no grid or terrain set on the batch");
  if (n_steps < 0) return set_err(EBL_EINVAL, "n_steps must be >= 0");
  if (int e = prepare(b)) return e;
  if (!b->det_tables_valid || std::memcmp(&b->det_cfg, &b->cfg, sizeof b->cfg) != 0)
    if (int e = det_tables(b)) return e;
  const size_t n = b->ncell * b->n_envs;
  if (record) EBL_CUDA(b->traj.alloc(3 * n * std::max(1, n_steps)));
  double* const tu = b->traj.p;
  double* const tbn = b->traj.p + n * std::max(1, n_steps);
  // record mode: p_bd is left out of the steps and accumulated after them (k_det_bd_run)
  const int cur0 = b->det_cur;
  for (int t = 0; t < n_steps; ++t) {
    ebl::DetArgs d = det_args(b);
    if (record && det_bd_deferred()) {
      d.bd = nullptr;
      d.bd_o = nullptr;
    }
    if (record) {
      // the trajectory slots are the states: step t reads slot t (step 0: the state buffers, which
      // it copies into slot 0) and writes slot t+1 (the last step: the state buffers); bd and the
      // output state ping-pong as without recording
      d.traj_lam = b->traj.p + 2 * n * n_steps;
      if (t == 0) {
        d.traj_un = tu;
        d.traj_burn = tbn;
      } else {
        d.un = tu + t * n;
        d.burn = tbn + t * n;
      }
      if (t + 1 < n_steps) {
        d.un_o = tu + (t + 1) * n;
        d.burn_o = tbn + (t + 1) * n;
      }
    }
    EBL_CUDA(ebl::launch_det_forward(d, t, b->stream));
    b->det_cur ^= 1;
    b->launches += 1;
  }
  if (record && det_bd_deferred() && n_steps > 0) {
    EBL_CUDA(ebl::launch_det_bd_run(b->det[cur0 * 3 + 2].p, b->det[b->det_cur * 3 + 2].p, tbn, n, n_steps,
                                    b->cfg.p_continue, b->stream));
    b->launches += 1;
  }
  b->traj_steps = record ? n_steps : -1;
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  return EBL_OK;
}

int ebl_det_set_mask(ebl_batch* b, const double* mask) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (!mask) return set_err(EBL_EINVAL, "mask is NULL");
  EBL_CUDA(cudaSetDevice(b->device));
  const size_t n = b->ncell * b->n_envs;
  EBL_CUDA(b->det_mask.alloc(n));
  EBL_CUDA(cudaMemcpyAsync(b->det_mask.p, mask, n * sizeof(double), cudaMemcpyHostToDevice, b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  b->det_mask_set = true;
  return EBL_OK;
}

int ebl_det_loss_grad(ebl_batch* b, const double* mask, double bce_w, double mse_w, int pool,
                      double* loss, double* grad6) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (b->traj_steps < 0 || !b->det_ready)
    return set_err(EBL_ESTATE, "ebl_det_loss_grad needs a recorded ebl_det_forward");
  if (pool < 1 || !(bce_w >= 0.0) || !(mse_w >= 0.0) || (bce_w == 0.0 && mse_w == 0.0))
    return set_err(EBL_EINVAL, "LossConfig: weights >= 0, one positive, pool_size >= 1");
  const size_t n = b->ncell * b->n_envs;
  const int bpe = std::max(static_cast<int>((b->ncell + 255) / 256), ebl::det_blocks_per_env(b->h, b->w));
  if (!mask && !b->det_mask_set) return set_err(EBL_ESTATE, "mask = NULL needs ebl_det_set_mask first");
  EBL_CUDA(b->det_mask.alloc(n));
  EBL_CUDA(b->adj.alloc(6 * n));
  EBL_CUDA(b->acc.alloc(static_cast<size_t>(b->n_envs) * bpe * 8));
  EBL_CUDA(b->det_loss.alloc(b->n_envs));
  EBL_CUDA(b->det_grad.alloc(static_cast<size_t>(b->n_envs) * 6));
  if (mask) {
    EBL_CUDA(cudaMemcpyAsync(b->det_mask.p, mask, n * sizeof(double), cudaMemcpyHostToDevice, b->stream));
    b->det_mask_set = false;  // a per-call mask replaces the resident one
  }
  EBL_CUDA(cudaMemsetAsync(b->acc.p, 0, static_cast<size_t>(b->n_envs) * bpe * 8 * sizeof(double), b->stream));
  ebl::DetArgs d = det_args(b);
  d.mask = b->det_mask.p;
  d.bce_w = bce_w;
  d.mse_w = mse_w;
  d.pool = pool;
  d.A_un = b->adj.p;
  d.A_burn = b->adj.p + n;
  d.A_bd = b->adj.p + 2 * n;
  d.a_lam = b->adj.p + 3 * n;
  d.acc = b->acc.p;
  d.loss = b->det_loss.p;
  d.grad = b->det_grad.p;
  d.traj_un = b->traj.p;
  d.traj_burn = b->traj.p + n * std::max(1, b->traj_steps);
  d.traj_lam = b->traj.p + 2 * n * std::max(1, b->traj_steps);
  d.inv_p_base = 1.0 / b->cfg.p_base;
  EBL_CUDA(ebl::launch_det_loss(d, b->stream));
#if EBL_DET_FUSED
  d.A_un_o = b->adj.p + 4 * n;  // fused backward: adjoints double-buffered
  d.A_burn_o = b->adj.p + 5 * n;
#endif
  for (int t = b->traj_steps - 1; t >= 0; --t) {
    EBL_CUDA(ebl::launch_det_backward(d, t, b->stream));
    if (d.A_un_o) {
      std::swap(d.A_un, d.A_un_o);
      std::swap(d.A_burn, d.A_burn_o);
    }
  }
  EBL_CUDA(ebl::launch_det_reduce(d, b->stream));
  b->launches += 2 + (d.A_un_o ? 1 : 2) * static_cast<uint64_t>(b->traj_steps);
  EBL_CUDA(cudaMemcpyAsync(loss, b->det_loss.p, b->n_envs * sizeof(double), cudaMemcpyDeviceToHost, b->stream));
  EBL_CUDA(cudaMemcpyAsync(grad6, b->det_grad.p, b->n_envs * 6 * sizeof(double), cudaMemcpyDeviceToHost, b->stream));
  EBL_CUDA(cudaStreamSynchronize(b->stream));
  return EBL_OK;
}

void ebl_default_calib_options(ebl_calib_options* o) {  // calibrate.hpp:158-166
  *o = ebl_calib_options{300, {0.12, 0.2, 0.4, 1.0, 1.0, 0.6}, {1, 1, 1, 1, 1, 1}, 1e-2, 2000};
}

// calibrate (calibrate.cpp:104-167) with every rollout, loss and gradient on the device.
int ebl_calibrate(ebl_batch* b, const double* p_un, const double* p_burn, const double* p_bd,
                  const double* mask, int horizon, double bce_w, double mse_w, int pool,
                  const ebl_calib_options* opt, double* loss_hist, double* theta_hist,
                  double* best_theta, double* best_loss) {
  EBL_DEVICE_GUARD(b);
  if (int e = check_batch(b)) return e;
  if (!opt || !p_un || !p_burn || !p_bd || !mask || !loss_hist || !theta_hist || !best_theta || !best_loss)
    return set_err(EBL_EINVAL, "null argument");
  const size_t n = b->ncell * b->n_envs;
  // validate_target / validate_loss_config / validate_state (calibrate.cpp:57-80, engine.cpp:54-72)
  for (int e = 0; e < b->n_envs; ++e) {
    bool any = false;
    for (size_t i = e * b->ncell; i < (e + 1) * b->ncell; ++i) {
      if (mask[i] != 0.0 && mask[i] != 1.0) return set_err(EBL_EINVAL, "CalibrationTarget: mask values must be 0 or 1");
      any |= mask[i] == 1.0;
    }
    if (!any) return set_err(EBL_EINVAL, "CalibrationTarget: mask has no burned cells");
  }
  if (horizon < 0) return set_err(EBL_EINVAL, "CalibrationTarget: negative horizon");
  if (!(bce_w >= 0.0) || !(mse_w >= 0.0)) return set_err(EBL_EINVAL, "LossConfig: weights must be >= 0");
  if (bce_w == 0.0 && mse_w == 0.0) return set_err(EBL_EINVAL, "LossConfig: at least one weight must be positive");
  if (pool < 1) return set_err(EBL_EINVAL, "LossConfig: pool_size must be >= 1");
  for (size_t i = 0; i < n; ++i) {
    if (!(p_un[i] >= 0.0) || !(p_burn[i] >= 0.0) || !(p_bd[i] >= 0.0))
      return set_err(EBL_EINVAL, "ContinuousState: negative or NaN component");
    if (std::abs(p_un[i] + p_burn[i] + p_bd[i] - 1.0) > 1e-9)
      return set_err(EBL_EINVAL, "ContinuousState: cell probabilities do not sum to 1");
  }
  if (opt->iterations < 0) return set_err(EBL_EINVAL, "calibrate: negative iteration count");
  if (horizon > opt->max_horizon) return set_err(EBL_EINVAL, "calibrate: horizon exceeds the configured maximum");
  // ThetaTransform::unconstrain (calibrate.cpp:35-55)
  double u[6];
  for (int i = 0; i < 6; ++i) u[i] = opt->init_theta[i];
  for (int i : {0, 4}) {
    const double y = opt->init_theta[i];
    if (!(y > 0.0)) return set_err(EBL_EINVAL, "inverse_softplus: argument must be > 0");
    u[i] = y > 20.0 ? y : std::log(std::expm1(y));
  }
  {
    const double p = opt->init_theta[5];
    if (!(p > 0.0 && p < 1.0)) return set_err(EBL_EINVAL, "logit: argument must be in (0, 1)");
    u[5] = std::log(p / (1.0 - p));
  }
  const double beta1 = 0.9, beta2 = 0.999, eps = 1e-8;  // AdamState defaults (calibrate.hpp:148-156)
  double m[6] = {0}, v[6] = {0};
  int t_adam = 0;
  *best_loss = std::numeric_limits<double>::infinity();
  const ebl_sim_config saved = b->cfg;
  std::vector<double> loss_e(b->n_envs), grad_e(static_cast<size_t>(b->n_envs) * 6);
  for (int iter = 0; iter <= opt->iterations; ++iter) {
    // ThetaTransform::constrain (calibrate.hpp:59-65): softplus / identity / logistic
    auto softplus = [](double x) { return x > 0.0 ? x + std::log(1.0 + std::exp(-x)) : std::log(1.0 + std::exp(x)); };
    auto logistic = [](double x) {
      if (x >= 0.0) return 1.0 / (1.0 + std::exp(-x));
      const double e = std::exp(x);
      return e / (1.0 + e);
    };
    const double th[6] = {softplus(u[0]), u[1], u[2], u[3], softplus(u[4]), logistic(u[5])};
    // d theta / d u: softplus' = logistic, logistic' = s (1 - s), identity elsewhere
    const double dth[6] = {logistic(u[0]), 1.0, 1.0, 1.0, logistic(u[4]), th[5] * (1.0 - th[5])};
    ebl_sim_config c = b->cfg;
    c.p_base = th[0], c.alpha_w1 = th[1], c.alpha_w2 = th[2], c.alpha_s = th[3], c.alpha_gamma = th[4],
    c.p_continue = th[5];
    if (int e = ebl_batch_set_config(b, &c)) return e;
    if (iter == 0) {  // initial state and target uploaded once, copied on the device afterwards
      if (int e = ebl_det_set_state(b, p_un, p_burn, p_bd)) return e;
      if (int e = ebl_det_set_mask(b, mask)) return e;
      EBL_CUDA(b->det_init.alloc(3 * n));
      for (int k = 0; k < 3; ++k)
        EBL_CUDA(cudaMemcpyAsync(b->det_init.p + k * n, b->det[b->det_cur * 3 + k].p, n * sizeof(double),
                                 cudaMemcpyDeviceToDevice, b->stream));
    } else {
      for (int k = 0; k < 3; ++k)
        EBL_CUDA(cudaMemcpyAsync(b->det[b->det_cur * 3 + k].p, b->det_init.p + k * n, n * sizeof(double),
                                 cudaMemcpyDeviceToDevice, b->stream));
    }
    if (int e = ebl_det_forward(b, horizon, 1)) return e;
    if (int e = ebl_det_loss_grad(b, nullptr, bce_w, mse_w, pool, loss_e.data(), grad_e.data())) return e;
    double l = 0.0, g[6] = {0};
    for (int e = 0; e < b->n_envs; ++e) {  // the batch's envs share theta: total loss
      l += loss_e[e];
      for (int k = 0; k < 6; ++k) g[k] += grad_e[e * 6 + k];
    }
    if (!std::isfinite(l))
      return set_err(EBL_ENUMERIC, "calibrate: loss became non-finite at iteration " + std::to_string(iter));
    loss_hist[iter] = l;
    for (int k = 0; k < 6; ++k) theta_hist[iter * 6 + k] = th[k];
    if (l < *best_loss) {
      *best_loss = l;
      for (int k = 0; k < 6; ++k) best_theta[k] = th[k];
    }
    if (iter == opt->iterations) break;
    // adam_step (calibrate.cpp:84-102) on d loss / d u
    double gu[6];
    for (int k = 0; k < 6; ++k) {
      gu[k] = opt->optimize[k] ? g[k] * dth[k] : 0.0;
      if (!std::isfinite(gu[k])) return set_err(EBL_ENUMERIC, "adam_step: non-finite gradient component");
    }
    t_adam += 1;
    const double bc1 = 1.0 - std::pow(beta1, t_adam), bc2 = 1.0 - std::pow(beta2, t_adam);
    for (int k = 0; k < 6; ++k) {
      m[k] = beta1 * m[k] + (1.0 - beta1) * gu[k];
      v[k] = beta2 * v[k] + (1.0 - beta2) * gu[k] * gu[k];
      const double m_hat = m[k] / bc1, v_hat = v[k] / bc2;
      u[k] = u[k] - opt->lr * m_hat / (std::sqrt(v_hat) + eps);
    }
  }
  return ebl_batch_set_config(b, &saved);
}

// ---- inputs ----------------------------------------------------------------------------
int ebl_synth_terrain(uint64_t seed, uint32_t env_id0, int n_envs, int h, int w, double elev_max,
                      double wind_max, uint8_t* fuel_class, float* elevation, double* wind_speed,
                      double* wind_direction) {
  if (n_envs < 1 || h < 2 || w < 2) return set_err(EBL_EINVAL, "synth_terrain: need n_envs >= 1, dims >= 2");
  if (!fuel_class || !elevation) return set_err(EBL_EINVAL, "null output");
  ebl::synth_terrain(seed, env_id0, n_envs, h, w, elev_max, wind_max, fuel_class, elevation,
                     wind_speed, wind_direction);
  return EBL_OK;
}

void ebl_worldcover_palette(int32_t* codes, double* veg, double* den) {
  ebl::worldcover_palette(codes, veg, den);
}

int ebl_synth_ignitions(uint64_t seed, uint32_t env_id0, int n_envs, int h, int w,
                        const uint8_t* fuel_class, const double* class_veg, const double* class_den,
                        int count, uint8_t* states) {
  if (n_envs < 1 || h < 1 || w < 1 || count < 0) return set_err(EBL_EINVAL, "synth_ignitions: bad sizes");
  return ebl::synth_ignitions(seed, env_id0, n_envs, h, w, fuel_class, class_veg, class_den, count,
                              states) >= 0
             ? EBL_OK
             : EBL_EINVAL;
}

}  // extern "C"
