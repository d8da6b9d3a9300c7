// Bit-plane helpers shared by the blocked CA kernel and the bit-plane RL kernel: one bit per
// cell, 32 cells of a row per word; row-major [rows][wpr] planes.
#pragma once
#include <cstdint>

namespace ebl {

__device__ __forceinline__ uint32_t west_of(const uint32_t* row, int j) {
  return (row[j] << 1) | (j > 0 ? row[j - 1] >> 31 : 0u);  // bit c <- cell c-1
}

__device__ __forceinline__ uint32_t east_of(const uint32_t* row, int j, int wpr) {
  return (row[j] >> 1) | (j + 1 < wpr ? row[j + 1] << 31 : 0u);  // bit c <- cell c+1
}

__device__ __forceinline__ uint32_t low_mask(int n) {
  return n >= 32 ? 0xffffffffu : (n <= 0 ? 0u : ((1u << n) - 1u));
}

// Iterates this thread's words idx = tid, tid+T, ... of an [rows][wpr] plane with the
// (row, word) pair maintained incrementally (no division in the loop).
struct WordIter {
  int idx, r, j, dr, dj, wpr, n;
  __device__ __forceinline__ WordIter(int wpr_, int n_) : wpr(wpr_), n(n_) {
    idx = threadIdx.x;
    r = idx / wpr;
    j = idx - r * wpr;
    dr = blockDim.x / wpr;
    dj = blockDim.x - dr * wpr;
  }
  __device__ __forceinline__ bool ok() const { return idx < n; }
  __device__ __forceinline__ void next() {
    idx += blockDim.x;
    r += dr;
    j += dj;
    if (j >= wpr) {
      j -= wpr;
      ++r;
    }
  }
};


// Bulk L2 prefetch (cp.async.bulk.prefetch, sm_90+): a hint, `bytes` a multiple of 16, 16-byte
// aligned address; no completion to wait for.
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uintptr_t lo = (a + 15) & ~uintptr_t(15);
  if (bytes < 32) return;
  const uint32_t n = (bytes - static_cast<uint32_t>(lo - a)) & ~15u;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"(n) : "memory");
}

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Row stride (words) of a bit-plane with wpr words per row: odd, so the 32 lanes of a warp
// each reading "its" row at the same column hit 32 distinct shared-memory banks.
__host__ __device__ __forceinline__ int plane_stride(int wpr) { return wpr | 1; }

// 32 uint8 cells (two 16-byte loads) -> Burning / Burned bits.  Bytes other than 1/2 act as
// Unburned exactly as in next_fire_cell (engine.cpp:15-25).
__device__ __forceinline__ void bytes_to_bits(const uint8_t* src, uint32_t& b, uint32_t& x) {
  const uint4 q0 = __ldg(reinterpret_cast<const uint4*>(src));
  const uint4 q1 = __ldg(reinterpret_cast<const uint4*>(src) + 1);
  const uint32_t wds[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
  b = 0u;
  x = 0u;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const uint32_t v = wds[q];
    const uint32_t z = v & 0xFCFCFCFCu;  // per byte: nonzero iff value >= 4
    const uint32_t small = ~((((z & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | z) >> 7) & 0x01010101u;
    const uint32_t b0 = v & 0x01010101u, b1 = (v >> 1) & 0x01010101u;
    const uint32_t lo = b0 & ~b1 & small;  // byte == 1
    const uint32_t hi = b1 & ~b0 & small;  // byte == 2
    b |= ((lo * 0x01020408u) >> 24 & 0xfu) << (4 * q);  // bytes' bit0 -> 4 contiguous bits
    x |= ((hi * 0x01020408u) >> 24 & 0xfu) << (4 * q);
  }
}

// Burning / Burned bits -> 32 uint8 cells (two 16-byte stores).
__device__ __forceinline__ void bits_to_bytes(uint32_t b, uint32_t x, uint8_t* dst) {
  uint32_t wds[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {  // spread 4 bits to 4 bytes: bit k -> bit 8k
    const uint32_t bs = (((b >> (4 * q)) & 0xfu) * 0x00204081u) & 0x01010101u;
    const uint32_t xs = (((x >> (4 * q)) & 0xfu) * 0x00204081u) & 0x01010101u;
    wds[q] = bs | (xs << 1);
  }
  reinterpret_cast<uint4*>(dst)[0] = make_uint4(wds[0], wds[1], wds[2], wds[3]);
  reinterpret_cast<uint4*>(dst)[1] = make_uint4(wds[4], wds[5], wds[6], wds[7]);
}

}  // namespace ebl
