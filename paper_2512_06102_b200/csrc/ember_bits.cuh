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

// The same, also ORing into `nc` a nonzero value when a byte is not a FireState (>= 3).
__device__ __forceinline__ void bytes_to_bits_nc(const uint8_t* src, uint32_t& b, uint32_t& x, uint32_t& nc) {
  const uint4 q0 = __ldg(reinterpret_cast<const uint4*>(src));
  const uint4 q1 = __ldg(reinterpret_cast<const uint4*>(src) + 1);
  const uint32_t wds[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
  b = 0u;
  x = 0u;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const uint32_t v = wds[q];
    const uint32_t z = v & 0xFCFCFCFCu;
    const uint32_t small = ~((((z & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | z) >> 7) & 0x01010101u;
    const uint32_t b0 = v & 0x01010101u, b1 = (v >> 1) & 0x01010101u;
    const uint32_t lo = b0 & ~b1 & small;
    const uint32_t hi = b1 & ~b0 & small;
    nc |= (~small & 0x01010101u) | (b0 & b1);  // byte >= 4, or byte == 3
    b |= ((lo * 0x01020408u) >> 24 & 0xfu) << (4 * q);
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


// Bit positions of the set bits of every byte value, 3 bits each (lowest first): the table of the
// n-th-set-bit search of the decide passes (read through the read-only cache; 1 KB).
__device__ const uint32_t kNthBitLut[256] = {0x000000u, 0x000000u, 0x000001u, 0x000008u, 0x000002u, 0x000010u, 0x000011u, 0x000088u, 0x000003u, 0x000018u, 0x000019u, 0x0000c8u, 0x00001au, 0x0000d0u, 0x0000d1u, 0x000688u, 0x000004u, 0x000020u, 0x000021u, 0x000108u, 0x000022u, 0x000110u, 0x000111u, 0x000888u, 0x000023u, 0x000118u, 0x000119u, 0x0008c8u, 0x00011au, 0x0008d0u, 0x0008d1u, 0x004688u, 0x000005u, 0x000028u, 0x000029u, 0x000148u, 0x00002au, 0x000150u, 0x000151u, 0x000a88u, 0x00002bu, 0x000158u, 0x000159u, 0x000ac8u, 0x00015au, 0x000ad0u, 0x000ad1u, 0x005688u, 0x00002cu, 0x000160u, 0x000161u, 0x000b08u, 0x000162u, 0x000b10u, 0x000b11u, 0x005888u, 0x000163u, 0x000b18u, 0x000b19u, 0x0058c8u, 0x000b1au, 0x0058d0u, 0x0058d1u, 0x02c688u, 0x000006u, 0x000030u, 0x000031u, 0x000188u, 0x000032u, 0x000190u, 0x000191u, 0x000c88u, 0x000033u, 0x000198u, 0x000199u, 0x000cc8u, 0x00019au, 0x000cd0u, 0x000cd1u, 0x006688u, 0x000034u, 0x0001a0u, 0x0001a1u, 0x000d08u, 0x0001a2u, 0x000d10u, 0x000d11u, 0x006888u, 0x0001a3u, 0x000d18u, 0x000d19u, 0x0068c8u, 0x000d1au, 0x0068d0u, 0x0068d1u, 0x034688u, 0x000035u, 0x0001a8u, 0x0001a9u, 0x000d48u, 0x0001aau, 0x000d50u, 0x000d51u, 0x006a88u, 0x0001abu, 0x000d58u, 0x000d59u, 0x006ac8u, 0x000d5au, 0x006ad0u, 0x006ad1u, 0x035688u, 0x0001acu, 0x000d60u, 0x000d61u, 0x006b08u, 0x000d62u, 0x006b10u, 0x006b11u, 0x035888u, 0x000d63u, 0x006b18u, 0x006b19u, 0x0358c8u, 0x006b1au, 0x0358d0u, 0x0358d1u, 0x1ac688u, 0x000007u, 0x000038u, 0x000039u, 0x0001c8u, 0x00003au, 0x0001d0u, 0x0001d1u, 0x000e88u, 0x00003bu, 0x0001d8u, 0x0001d9u, 0x000ec8u, 0x0001dau, 0x000ed0u, 0x000ed1u, 0x007688u, 0x00003cu, 0x0001e0u, 0x0001e1u, 0x000f08u, 0x0001e2u, 0x000f10u, 0x000f11u, 0x007888u, 0x0001e3u, 0x000f18u, 0x000f19u, 0x0078c8u, 0x000f1au, 0x0078d0u, 0x0078d1u, 0x03c688u, 0x00003du, 0x0001e8u, 0x0001e9u, 0x000f48u, 0x0001eau, 0x000f50u, 0x000f51u, 0x007a88u, 0x0001ebu, 0x000f58u, 0x000f59u, 0x007ac8u, 0x000f5au, 0x007ad0u, 0x007ad1u, 0x03d688u, 0x0001ecu, 0x000f60u, 0x000f61u, 0x007b08u, 0x000f62u, 0x007b10u, 0x007b11u, 0x03d888u, 0x000f63u, 0x007b18u, 0x007b19u, 0x03d8c8u, 0x007b1au, 0x03d8d0u, 0x03d8d1u, 0x1ec688u, 0x00003eu, 0x0001f0u, 0x0001f1u, 0x000f88u, 0x0001f2u, 0x000f90u, 0x000f91u, 0x007c88u, 0x0001f3u, 0x000f98u, 0x000f99u, 0x007cc8u, 0x000f9au, 0x007cd0u, 0x007cd1u, 0x03e688u, 0x0001f4u, 0x000fa0u, 0x000fa1u, 0x007d08u, 0x000fa2u, 0x007d10u, 0x007d11u, 0x03e888u, 0x000fa3u, 0x007d18u, 0x007d19u, 0x03e8c8u, 0x007d1au, 0x03e8d0u, 0x03e8d1u, 0x1f4688u, 0x0001f5u, 0x000fa8u, 0x000fa9u, 0x007d48u, 0x000faau, 0x007d50u, 0x007d51u, 0x03ea88u, 0x000fabu, 0x007d58u, 0x007d59u, 0x03eac8u, 0x007d5au, 0x03ead0u, 0x03ead1u, 0x1f5688u, 0x000facu, 0x007d60u, 0x007d61u, 0x03eb08u, 0x007d62u, 0x03eb10u, 0x03eb11u, 0x1f5888u, 0x007d63u, 0x03eb18u, 0x03eb19u, 0x1f58c8u, 0x03eb1au, 0x1f58d0u, 0x1f58d1u, 0xfac688u};
}  // namespace ebl
