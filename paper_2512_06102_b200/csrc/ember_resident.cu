// Fused env-resident multi-step kernel (the throughput path for batched envs,
// BASELINE C1).  One CTA owns one env for the whole launch: the env's fire layer
// is loaded once from HBM (uint8 [row][col]), converted to bit-planes in shared
// memory, advanced n_steps times, and written back once.  Per step:
//
//   P1 dense   (bit-sliced, 32 cells per op): for each 32-cell word,
//              any  = 8-neighbour dilation of the Burning plane,
//              cand = Unburned & any            (ignition candidates: the only
//                                                Unburned cells whose draw can matter),
//              act  = cand | Burning;           popc -> block-wide exclusive scan
//              -> compacted list of active cells (uint16 cell index).
//   P2 sparse  one thread per active cell (load-balanced): rng_word of the cell
//              (two mix64 rounds on the per-(env,step) prefix), Burning: survive
//              test on the integer threshold; candidate: the 8-bit neighbour mask
//              from the plane, lambda / p in fp32 with fp64 guard fallback
//              (ember_device.cuh).  Outcomes are OR-ed into IGN / OUT planes.
//   P3 dense   B = (B & ~OUT) | IGN;  X |= OUT.
//
// Every cell is updated every step (Burned and non-candidate Unburned cells by
// the bit-sliced identity in P3), so the dense count of cell-updates is the
// reference's (emberline_main.cpp:432-433).  The result is bit-identical to the
// tiled kernel and to engine.cpp:134-159 by construction (same per-cell rule,
// same keys).
#include <cuda_runtime.h>

#include <cstdint>

#include "ember_device.cuh"
#include "ember_kernels.h"
#include "ember_params.h"

namespace ebl {

namespace {

struct Planes {
  uint32_t* B;    // burning          [(H+2)][wpr], rows 0 and H+1 are zero padding
  uint32_t* X;    // burned
  uint32_t* IGN;  // ignited this step
  uint32_t* OUT;  // burned out this step
  uint32_t* ACT;  // active cells of the current step (unpadded [H][wpr])
  uint16_t* list;
  int wpr;
};

__device__ __forceinline__ uint32_t west_of(const uint32_t* row, int j, int wpr) {
  // bit c set iff cell c-1 (one column west) is set
  return (row[j] << 1) | (j > 0 ? row[j - 1] >> 31 : 0u);
  (void)wpr;
}

__device__ __forceinline__ uint32_t east_of(const uint32_t* row, int j, int wpr) {
  // bit c set iff cell c+1 is set
  return (row[j] >> 1) | (j + 1 < wpr ? row[j + 1] << 31 : 0u);
}

__device__ __forceinline__ uint32_t valid_mask(int j, int w) {
  const int rem = w - 32 * j;
  return rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
}

// Exclusive block scan of one int per thread; returns the total via *total.
__device__ __forceinline__ int block_exclusive_scan(int v, int* warp_tot, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    int t = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nw) warp_tot[lane] = t;  // inclusive warp prefix
    if (lane == nw - 1) *total = t;
  }
  __syncthreads();
  return (warp > 0 ? warp_tot[warp - 1] : 0) + x - v;
}

}  // namespace

template <int MODE>
__global__ void __launch_bounds__(kResThreads) k_step_resident(StepArgs a, int n_steps) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int warp_tot[32];
  __shared__ int s_total;
  __shared__ uint64_t s_prefix;
  __shared__ int32_t s_cnt[4];

  const int env = blockIdx.x;
  const int H = a.h, W = a.w;
  const int wpr = (W + 31) >> 5;
  const int nwords = H * wpr;
  const int pw = (H + 2) * wpr;  // padded plane words
  Planes p;
  p.wpr = wpr;
  p.B = reinterpret_cast<uint32_t*>(smem);
  p.X = p.B + pw;
  p.IGN = p.X + pw;
  p.OUT = p.IGN + pw;
  p.ACT = p.OUT + pw;
  p.list = reinterpret_cast<uint16_t*>(p.ACT + nwords);

  const size_t ncell = static_cast<size_t>(H) * W;
  const uint8_t* __restrict__ in = a.in + env * ncell;

  // ---- load: uint8 layer -> bit-planes --------------------------------------------
  for (int i = threadIdx.x; i < pw; i += blockDim.x) {
    p.B[i] = 0u;
    p.X[i] = 0u;
    p.IGN[i] = 0u;
    p.OUT[i] = 0u;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < nwords; idx += blockDim.x) {
    const int r = idx / wpr, j = idx - r * wpr;
    const int c0 = 32 * j;
    const int nc = min(32, W - c0);
    uint32_t b = 0u, x = 0u;
    const uint8_t* src = in + static_cast<size_t>(r) * W + c0;
    if (nc == 32 && (W & 15) == 0) {
      const uint4 q0 = __ldg(reinterpret_cast<const uint4*>(src));
      const uint4 q1 = __ldg(reinterpret_cast<const uint4*>(src) + 1);
      const uint32_t wds[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
      for (int q = 0; q < 8; ++q) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t v = (wds[q] >> (8 * k)) & 0xffu;
          b |= static_cast<uint32_t>(v == 1u) << (4 * q + k);
          x |= static_cast<uint32_t>(v == 2u) << (4 * q + k);
        }
      }
    } else {
      for (int k = 0; k < nc; ++k) {
        const uint8_t v = src[k];
        b |= static_cast<uint32_t>(v == 1) << k;
        x |= static_cast<uint32_t>(v == 2) << k;
      }
    }
    p.B[(r + 1) * wpr + j] = b;
    p.X[(r + 1) * wpr + j] = x;
  }
  if (threadIdx.x < 4) s_cnt[threadIdx.x] = 0;
  __syncthreads();

  const DiagCounters dg{a.diag};
  const uint64_t stream = a.streams[env];
  int32_t newly_last = 0;

  for (int t = 0; t < n_steps; ++t) {
    if (threadIdx.x == 0) s_prefix = key_prefix(a.seed, stream, a.step + static_cast<uint64_t>(t));
    // ---- P1: candidates + burning -> active count --------------------------------
    int cnt = 0;
    for (int idx = threadIdx.x; idx < nwords; idx += blockDim.x) {
      const int r = idx / wpr, j = idx - r * wpr;
      const uint32_t* up = p.B + (r + 2) * wpr;   // row r+1 (north)
      const uint32_t* mid = p.B + (r + 1) * wpr;
      const uint32_t* dn = p.B + r * wpr;         // row r-1 (south)
      const uint32_t hu = up[j] | west_of(up, j, wpr) | east_of(up, j, wpr);
      const uint32_t hd = dn[j] | west_of(dn, j, wpr) | east_of(dn, j, wpr);
      const uint32_t any = hu | hd | west_of(mid, j, wpr) | east_of(mid, j, wpr);
      const uint32_t b = mid[j];
      const uint32_t u = ~(b | p.X[(r + 1) * wpr + j]) & valid_mask(j, W);
      const uint32_t act = (u & any) | b;
      p.ACT[idx] = act;
      cnt += __popc(act);
    }
    int off = block_exclusive_scan(cnt, warp_tot, &s_total);
    for (int idx = threadIdx.x; idx < nwords; idx += blockDim.x) {
      uint32_t act = p.ACT[idx];
      const int r = idx / wpr, j = idx - r * wpr;
      const int base = r * W + 32 * j;
      while (act) {
        const int bit = __ffs(act) - 1;
        act &= act - 1;
        p.list[off++] = static_cast<uint16_t>(base + bit);
      }
    }
    __syncthreads();
    // ---- P2: sparse decisions ---------------------------------------------------
    const int total = s_total;
    const uint64_t prefix = s_prefix;
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
      const int cell = p.list[i];
      const int r = cell / W, c = cell - r * W;
      const int wi = (r + 1) * wpr + (c >> 5);
      const uint32_t bit = 1u << (c & 31);
      const uint64_t m = cell_bits53(prefix, static_cast<uint64_t>(cell), 0);
      if (p.B[wi] & bit) {
        if (m >= a.pc_thr) atomicOr(p.OUT + wi, bit);
      } else {
        uint32_t nb = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int ur = r - kDy[k], uc = c - kDx[k];
          if (uc < 0 || uc >= W) continue;  // row padding covers ur = -1 and ur = H
          nb |= ((p.B[(ur + 1) * wpr + (uc >> 5)] >> (uc & 31)) & 1u) << k;
        }
        if (ignite<MODE>(a, env, r, c, nb, m, dg)) atomicOr(p.IGN + wi, bit);
      }
    }
    __syncthreads();
    // ---- P3: apply ------------------------------------------------------------------
    int newly = 0;
    for (int idx = threadIdx.x; idx < nwords; idx += blockDim.x) {
      const int wi = (idx / wpr + 1) * wpr + idx % wpr;
      const uint32_t o = p.OUT[wi], g = p.IGN[wi];
      p.B[wi] = (p.B[wi] & ~o) | g;
      p.X[wi] |= o;
      p.OUT[wi] = 0u;
      p.IGN[wi] = 0u;
      newly += __popc(g);
    }
    newly_last = newly;
    __syncthreads();
  }

  // ---- store: bit-planes -> uint8 layer, counts -------------------------------------
  uint8_t* __restrict__ out = a.out + env * ncell;
  int32_t nB = 0, nX = 0;
  for (int idx = threadIdx.x; idx < nwords; idx += blockDim.x) {
    const int r = idx / wpr, j = idx - r * wpr;
    const uint32_t b = p.B[(r + 1) * wpr + j], x = p.X[(r + 1) * wpr + j];
    nB += __popc(b);
    nX += __popc(x);
    const int c0 = 32 * j;
    const int nc = min(32, W - c0);
    uint8_t* dst = out + static_cast<size_t>(r) * W + c0;
    if (nc == 32 && (W & 15) == 0) {
      uint32_t wds[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        uint32_t v = 0u;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int bit = 4 * q + k;
          v |= (((b >> bit) & 1u) | (((x >> bit) & 1u) << 1)) << (8 * k);
        }
        wds[q] = v;
      }
      reinterpret_cast<uint4*>(dst)[0] = make_uint4(wds[0], wds[1], wds[2], wds[3]);
      reinterpret_cast<uint4*>(dst)[1] = make_uint4(wds[4], wds[5], wds[6], wds[7]);
    } else {
      for (int k = 0; k < nc; ++k) dst[k] = static_cast<uint8_t>(((b >> k) & 1u) | (((x >> k) & 1u) << 1));
    }
  }
  if (a.counts) {
    atomicAdd(&s_cnt[1], nB);
    atomicAdd(&s_cnt[2], nX);
    atomicAdd(&s_cnt[3], newly_last);
    __syncthreads();
    if (threadIdx.x == 0) {
      a.counts[env * 4 + 0] = static_cast<int32_t>(ncell) - s_cnt[1] - s_cnt[2];
      a.counts[env * 4 + 1] = s_cnt[1];
      a.counts[env * 4 + 2] = s_cnt[2];
      a.counts[env * 4 + 3] = s_cnt[3];
    }
  }
}

size_t resident_smem_bytes(int h, int w) {
  const size_t wpr = (w + 31) / 32;
  const size_t planes = (4 * (static_cast<size_t>(h) + 2) + h) * wpr * sizeof(uint32_t);
  const size_t list = static_cast<size_t>(h) * w * sizeof(uint16_t);
  return planes + ((list + 15) & ~size_t(15));
}

bool resident_fits(int h, int w) {
  return static_cast<size_t>(h) * w <= 65536 && resident_smem_bytes(h, w) <= kResMaxSmem;
}

cudaError_t launch_step_resident(const StepArgs& a, int mode, int n_steps, cudaStream_t s) {
  const size_t sm = resident_smem_bytes(a.h, a.w);
  cudaError_t e;
  if (mode == kStaticTables) {
    e = cudaFuncSetAttribute(k_step_resident<kStaticTables>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sm));
    if (e != cudaSuccess) return e;
    k_step_resident<kStaticTables><<<a.n_envs, kResThreads, sm, s>>>(a, n_steps);
  } else {
    e = cudaFuncSetAttribute(k_step_resident<kStaticTerrain>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sm));
    if (e != cudaSuccess) return e;
    k_step_resident<kStaticTerrain><<<a.n_envs, kResThreads, sm, s>>>(a, n_steps);
  }
  return cudaGetLastError();
}

}  // namespace ebl
