// exp(x) bit-identical to the reference's libm (glibc 2.39, x86-64 FMA variant of
// sysdeps/ieee754/dbl-64/e_exp.c): the same table (ember_exp_table.h, generated and checked by
// scripts/gen_exp_table.py), constants and operation sequence -- every product-sum the FMA build
// contracts is an explicit fma here, so device and host evaluate the identical IEEE operations.
//   x = k ln2/128 + r,  exp(x) = 2^(k/128) exp(r) = scale (1 + tail) exp(r)
//   tmp = tail + r + r^2 (C2 + r C3) + r^4 (C4 + r C5),  exp(x) = scale + scale tmp
// Valid (bit-exact) for 2^-54 <= |x| < 512 and, as glibc, 1 + x below; `exact` is cleared outside
// (callers fall back to their own exp there).  Pinned against the live libm by
// tests/test_exp_glibc.py (CPU) and the device path by tests/test_det_gpu.py.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>

#include "ember_exp_table.h"

namespace ebl {

__host__ __device__ __forceinline__ double u64_as_f64(uint64_t v) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double(static_cast<long long>(v));
#else
  double d;
  std::memcpy(&d, &v, sizeof d);
  return d;
#endif
}
__host__ __device__ __forceinline__ uint64_t f64_as_u64(double d) {
#ifdef __CUDA_ARCH__
  return static_cast<uint64_t>(__double_as_longlong(d));
#else
  uint64_t v;
  std::memcpy(&v, &d, sizeof v);
  return v;
#endif
}

// tab: the EBL_EXP_TAB_INIT table (256 entries) in any memory space (shared memory on the device)
__host__ __device__ __forceinline__ double exp_glibc(double x, const uint64_t* tab, bool* exact) {
  const uint32_t abstop = static_cast<uint32_t>(f64_as_u64(x) >> 52) & 0x7ffu;
  if (abstop - 0x3c9u > 0x3eu) {
    if (static_cast<int32_t>(abstop - 0x3c9u) < 0) return 1.0 + x;  // |x| < 2^-54: 1 + x (as glibc)
    *exact = false;  // |x| >= 512, inf, nan: outside the domain restated here
    return exp(x);
  }
  const double kd0 = fma(x, u64_as_f64(kExpC0), u64_as_f64(kExpC1));  // x N/ln2 + shift
  const uint64_t ki = f64_as_u64(kd0);
  const double kd = kd0 - u64_as_f64(kExpC1);
  double r = fma(kd, u64_as_f64(kExpC2), x);  // x - kd ln2/N (hi)
  r = fma(kd, u64_as_f64(kExpC3), r);         //            (lo)
  const uint32_t idx = 2u * static_cast<uint32_t>(ki & 127u);
  const uint64_t top = ki << 45;
  const double p23 = fma(r, u64_as_f64(kExpC5), u64_as_f64(kExpC4));  // C2 + r C3
  const double tr = r + u64_as_f64(tab[idx]);                                    // tail + r
  const uint64_t sbits = tab[idx + 1] + top;
  const double r2 = r * r;
  const double p45 = fma(r, u64_as_f64(kExpC7), u64_as_f64(kExpC6));  // C4 + r C5
  const double t1 = fma(p23, r2, tr);
  const double r4 = r2 * r2;
  const double tmp = fma(r4, p45, t1);
  const double scale = u64_as_f64(sbits);
  return fma(scale, tmp, scale);
}

}  // namespace ebl
